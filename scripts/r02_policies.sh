#!/bin/bash
# ARM policy comparison with per-second timelines (RAPID vs hybrid-2048 on the same trace), + ncu census variants
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02b}
mkdir -p $out
summ() { python -c "import json,sys; d=json.load(open('$1')); c=d.get('comparator') or {}; print(round(d['value']), 'win', round(d['device_window']['tokens_per_s']), 'p99', d['p99_itl_ms'], 'ttft50', d['p50_ttft_ms'], 'B', round(d['device_window']['mean_decode_batch'] or 0), '| hyb', round(c.get('value',0)), c.get('p99_itl_ms'))" 2>&1 | tail -1; }
for pol in adaptive feedback balanced; do
  timeout 600 python bench.py --arm-policy $pol --no-cpu-baseline --timeline $out/tl_$pol > $out/$pol.json 2> $out/$pol.err
  echo "$pol: $(summ $out/$pol.json)"
done
bash scripts/ncu_census.sh

#!/bin/bash
# cfg 5: Qwen2.5-14B 8192/128, RAPID (measured ARM) vs same-engine hybrid-2048 / hybrid-512, same trace
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02v}
mkdir -p $out
summ() { python -c "import json,sys; d=json.load(open('$1')); c=d.get('comparator') or {}; print(round(d['value']), 'unconstr', round(d['tokens_per_s_unconstrained']), 'p99', d['p99_itl_ms'], 'ttft50', round(d['p50_ttft_ms']), d.get('arm_decisions'), 'clk', d['clocks'].get('sm_mhz'), '|', c.get('engine'), round(c.get('value',0)), round(c.get('tokens_per_s_unconstrained',0)), c.get('p99_itl_ms'), 'slo', c.get('slo_met'))" 2>&1 | tail -1; }
for cmp in hybrid-2048 hybrid-512; do
  timeout 900 python bench.py --model qwen2.5-14b --prompt 8192 --output 128 --qps 3.5 --compare $cmp --no-cpu-baseline > $out/q14_$cmp.json 2> $out/q14_$cmp.err
  echo "cfg5 rapid vs $cmp: $(summ $out/q14_$cmp.json)"
done

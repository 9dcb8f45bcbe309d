#!/bin/bash
# After a kernel change: all GPU tests, re-measured ARM tables, default bench (+ hybrid comparator)
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02n}
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu.log
P=$out/llama3.1-8b_ctx1152_chunk1023.json
timeout 1200 python -m paper_2601_11822_b200.profiler --model llama3.1-8b --ctx 1152 --chunk 1023 --out $P > $out/prof.log 2>&1; echo "prof rc=$?"; tail -14 $out/prof.log | cut -c1-200
summ() { python -c "import json,sys; d=json.load(open('$1')); c=d.get('comparator') or {}; print(round(d['value']), 'win', round(d['device_window']['tokens_per_s'] or 0), 'p99', d['p99_itl_ms'], 'ttft50', d['p50_ttft_ms'], 'B', round(d['device_window']['mean_decode_batch'] or 0), d.get('arm_decisions'), 'roof', round(d['roofline']['frac'],3), '| hyb', round(c.get('value',0)), c.get('p99_itl_ms'))" 2>&1 | tail -1; }
for pol in balanced feedback; do
  timeout 600 python bench.py --arm-profile $P --arm-policy $pol --no-cpu-baseline --timeline $out/tl_$pol > $out/$pol.json 2> $out/$pol.err
  echo "$pol: $(summ $out/$pol.json)"
done

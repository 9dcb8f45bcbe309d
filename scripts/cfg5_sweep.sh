#!/bin/bash
# cfg 5: Qwen2.5-14B prefill-heavy long context (in 8192 / out 128), RAPID (adaptive ARM) vs the
# same engine's chunked-prefill hybrid mode, QPS sweep; plus the cfg-2/3 8B engine comparison.
# Usage: bash scripts/cfg5_sweep.sh <outdir>
out=${1:-gpurun_out/sweep}
mkdir -p $out
for q in ${QPS14:-1.5 2.5 3.5}; do
  for e in rapid hybrid-2048 hybrid-512; do
    extra="--engine $e"; [ $e = rapid ] && extra="--arm"
    timeout 400 python bench.py --model qwen2.5-14b --prompt 8192 --output 128 --qps $q --steps 300 --warmup 20 \
      --no-cpu-baseline $extra > $out/q14_${e}_${q}.json 2> $out/q14_${e}_${q}.err
    echo "14b $e qps=$q: $(python -c "import json,sys; d=json.load(open('$out/q14_${e}_${q}.json')); print(round(d['value']), 'tok/s p99', round(d['p99_itl_ms'],1), 'ms ttft50', round(d['p50_ttft_ms']), 'ms run', round(d['run_tokens_per_s']), d['arm_decisions'])" 2>&1 | tail -1)"
  done
done

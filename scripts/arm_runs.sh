#!/bin/bash
# Measured ARM tables (profiler) for 8B (cfg 2/3 mix) and Qwen-14B (cfg 5 mix), then benches with them.
out=${1:-gpurun_out/arm}
mkdir -p $out profiles/arm
timeout 900 python -m paper_2601_11822_b200.profiler --model llama3.1-8b --ctx 1152 --out profiles/arm/llama3.1-8b_ctx1152.json 2>&1 | tail -20 > $out/prof8b.log
timeout 1200 python -m paper_2601_11822_b200.profiler --model qwen2.5-14b --ctx 8256 --out profiles/arm/qwen2.5-14b_ctx8256.json 2>&1 | tail -20 > $out/prof14b.log
summ() { python -c "import json,sys; d=json.load(open('$1')); print(round(d['value']), 'tok/s p99', round(d['p99_itl_ms'],1), 'ms ttft50', round(d['p50_ttft_ms']), 'ms run', round(d['run_tokens_per_s']), 'B', round(d['mean_decode_batch'] or 0), d['arm_decisions'])" 2>&1 | tail -1; }
for q in 40 56; do
  timeout 400 python bench.py --qps $q --arm-profile profiles/arm/llama3.1-8b_ctx1152.json --no-cpu-baseline > $out/8b_bal_$q.json 2> $out/8b_bal_$q.err
  echo "8b balanced qps=$q: $(summ $out/8b_bal_$q.json)"
done
for q in 2.5 3.5; do
  timeout 400 python bench.py --model qwen2.5-14b --prompt 8192 --output 128 --qps $q --steps 300 --warmup 20 \
    --arm-profile profiles/arm/qwen2.5-14b_ctx8256.json --no-cpu-baseline > $out/14b_bal_$q.json 2> $out/14b_bal_$q.err
  echo "14b balanced qps=$q: $(summ $out/14b_bal_$q.json)"
done

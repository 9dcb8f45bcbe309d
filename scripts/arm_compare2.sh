#!/bin/bash
out=${1:-gpurun_out/armc2}
mkdir -p $out
prof=profiles/arm/llama3.1-8b_ctx1152_chunk1023.json
summ() { python -c "import json,sys; d=json.load(open('$1')); print(round(d['value']), 'tok/s p99', round(d['p99_itl_ms'],1), 'slo_met', d['slo_met'], 'ttft50', round(d['p50_ttft_ms']), 'B', round(d['mean_decode_batch'] or 0), d['arm_decisions'])" 2>&1 | tail -1; }
for slo in 50 25; do
  timeout 300 python bench.py --qps 56 --slo-ms $slo --arm-profile $prof --arm-policy adaptive --no-cpu-baseline > $out/adaptive$slo.json 2> $out/adaptive$slo.err
  echo "adaptive q56 slo$slo: $(summ $out/adaptive$slo.json)"
done
timeout 300 python bench.py --qps 56 --slo-ms 50 --arm-profile $prof --arm-policy adaptive --no-cpu-baseline > $out/adaptive50b.json 2> $out/adaptive50b.err
echo "adaptive q56 slo50 (repeat): $(summ $out/adaptive50b.json)"
timeout 400 python bench.py --model qwen2.5-14b --prompt 8192 --output 128 --qps 3.5 --steps 300 --warmup 20 --arm-profile profiles/arm/qwen2.5-14b_ctx8256.json --arm-policy adaptive --no-cpu-baseline > $out/q14_adaptive.json 2> $out/q14_adaptive.err
echo "14b adaptive q3.5: $(summ $out/q14_adaptive.json)"

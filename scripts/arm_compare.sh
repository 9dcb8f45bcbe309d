#!/bin/bash
out=${1:-gpurun_out/armc}
mkdir -p $out
prof=profiles/arm/llama3.1-8b_ctx1152_chunk1023.json
summ() { python -c "import json,sys; d=json.load(open('$1')); print(round(d['value']), 'tok/s p99', round(d['p99_itl_ms'],1), 'slo_met', d['slo_met'], 'ttft50', round(d['p50_ttft_ms']), 'B', round(d['mean_decode_batch'] or 0), d['arm_decisions'])" 2>&1 | tail -1; }
timeout 500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python scripts/step_bench.py --B 128,256 --pdl 1
for pol in adaptive balanced; do
  timeout 300 python bench.py --qps 56 --arm-profile $prof --arm-policy $pol --no-cpu-baseline > $out/$pol.json 2> $out/$pol.err
  echo "$pol q56 slo50: $(summ $out/$pol.json)"
done
timeout 300 python bench.py --qps 56 --slo-ms 25 --arm-profile $prof --arm-policy adaptive --no-cpu-baseline > $out/adaptive25.json 2> $out/adaptive25.err
echo "adaptive q56 slo25: $(summ $out/adaptive25.json)"
timeout 300 python bench.py --qps 48 --engine hybrid-2048 --no-cpu-baseline > $out/hybrid-2048.json 2> $out/hybrid-2048.err
echo "hybrid-2048 q48: $(summ $out/hybrid-2048.json)"

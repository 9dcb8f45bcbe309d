#!/bin/bash
# RAPID (measured ARM, balanced) vs same-engine hybrid at two ITL SLOs (Llama-3.1-8B, 1024/256).
out=${1:-gpurun_out/slo}
mkdir -p $out
prof=$out/llama3.1-8b_ctx1152_chunk1023.json
timeout 500 python -m paper_2601_11822_b200.profiler --model llama3.1-8b --ctx 1152 --chunk 1023 --out $prof > $out/prof.log 2>&1
summ() { python -c "import json,sys; d=json.load(open('$1')); print(round(d['value']), 'tok/s p99', round(d['p99_itl_ms'],1), 'slo_met', d['slo_met'], 'ttft50', round(d['p50_ttft_ms']), 'B', round(d['mean_decode_batch'] or 0), d['arm_decisions'])" 2>&1 | tail -1; }
for slo in 50 25; do
  timeout 300 python bench.py --qps 56 --slo-ms $slo --arm-profile $prof --no-cpu-baseline > $out/rapid_$slo.json 2> $out/rapid_$slo.err
  echo "slo $slo rapid-balanced q56: $(summ $out/rapid_$slo.json)"
done
for e in hybrid-2048 hybrid-1024 hybrid-512; do
  timeout 300 python bench.py --qps 48 --slo-ms 25 --engine $e --no-cpu-baseline > $out/$e.json 2> $out/$e.err
  echo "$e q48: $(summ $out/$e.json)"
done

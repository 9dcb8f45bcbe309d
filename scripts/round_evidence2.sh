#!/bin/bash
out=${1:-gpurun_out/ev2}
mkdir -p $out
timeout 600 python -m paper_2601_11822_b200.profiler --model llama3.1-8b --ctx 1152 --chunk 1023 --out $out/llama3.1-8b_ctx1152_chunk1023.json > $out/prof8b.log 2>&1
summ() { python -c "import json,sys; d=json.load(open('$1')); print(round(d['value']), 'tok/s p99', round(d['p99_itl_ms'],1), 'slo_met', d['slo_met'], 'ttft50', round(d['p50_ttft_ms']), 'B', round(d['mean_decode_batch'] or 0), 'frac', round(d['roofline']['frac'],3), d['arm_decisions'])" 2>&1 | tail -1; }
P8=$out/llama3.1-8b_ctx1152_chunk1023.json
for i in 1 2 3; do
  timeout 400 python bench.py --arm-profile $P8 > $out/default$i.json 2> $out/default$i.err; echo "default (adaptive ARM) q56 #$i: $(summ $out/default$i.json)"
done
for e in hybrid-2048; do
  timeout 400 python bench.py --qps 48 --engine $e --no-cpu-baseline > $out/$e.json 2> $out/$e.err; echo "$e q48: $(summ $out/$e.json)"
done
timeout 400 python bench.py --decode-sms 72 --qps 40 --no-cpu-baseline > $out/cfg2.json 2> $out/cfg2.err; echo "cfg2 static 72/76 q40: $(summ $out/cfg2.json)"

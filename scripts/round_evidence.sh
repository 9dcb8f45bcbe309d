#!/bin/bash
# Re-profile the measured ARM tables on the current kernels, then the engine comparison.
out=${1:-gpurun_out/ev}
mkdir -p $out
timeout 600 python -m paper_2601_11822_b200.profiler --model llama3.1-8b --ctx 1152 --chunk 1023 --out $out/llama3.1-8b_ctx1152_chunk1023.json > $out/prof8b.log 2>&1
timeout 900 python -m paper_2601_11822_b200.profiler --model qwen2.5-14b --ctx 8256 --chunk 2048 --out $out/qwen2.5-14b_ctx8256.json > $out/prof14b.log 2>&1
summ() { python -c "import json,sys; d=json.load(open('$1')); print(round(d['value']), 'tok/s p99', round(d['p99_itl_ms'],1), 'slo_met', d['slo_met'], 'ttft50', round(d['p50_ttft_ms']), 'B', round(d['mean_decode_batch'] or 0), 'frac', round(d['roofline']['frac'],3), d['arm_decisions'])" 2>&1 | tail -1; }
P8=$out/llama3.1-8b_ctx1152_chunk1023.json
P14=$out/qwen2.5-14b_ctx8256.json
for i in 1 2; do
  timeout 400 python bench.py --arm-profile $P8 > $out/default$i.json 2> $out/default$i.err; echo "default (adaptive ARM) q56 #$i: $(summ $out/default$i.json)"
done
timeout 400 python bench.py --decode-sms 72 --qps 40 --no-cpu-baseline > $out/cfg2.json 2> $out/cfg2.err; echo "cfg2 static 72/76 q40: $(summ $out/cfg2.json)"
timeout 400 python bench.py --arm --qps 48 --no-cpu-baseline > $out/refarm.json 2> $out/refarm.err; echo "reference allocate() q48: $(summ $out/refarm.json)"
for e in hybrid-2048 hybrid-1024 hybrid-512; do
  timeout 400 python bench.py --qps 48 --engine $e --no-cpu-baseline > $out/$e.json 2> $out/$e.err; echo "$e q48: $(summ $out/$e.json)"
done
for q in 3.5; do
  timeout 500 python bench.py --model qwen2.5-14b --prompt 8192 --output 128 --qps $q --steps 300 --warmup 20 --arm-profile $P14 --no-cpu-baseline > $out/q14_rapid_$q.json 2> $out/q14_rapid_$q.err; echo "14b rapid adaptive q$q: $(summ $out/q14_rapid_$q.json)"
  for e in hybrid-2048 hybrid-512; do
    timeout 500 python bench.py --model qwen2.5-14b --prompt 8192 --output 128 --qps $q --steps 300 --warmup 20 --engine $e --no-cpu-baseline > $out/q14_${e}_$q.json 2> $out/q14_${e}_$q.err; echo "14b $e q$q: $(summ $out/q14_${e}_$q.json)"
  done
done

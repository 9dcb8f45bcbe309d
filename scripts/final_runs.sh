#!/bin/bash
# Round-end evidence: ncu capture of the bench's dominant kernel, launch list of the bench
# command, and the engine comparison on the current build.
out=${1:-gpurun_out/final}
mkdir -p $out
timeout 300 ncu --set full --import-source on --clock-control none -k regex:decode_attn_tc -s 3 -c 1 \
  -o $out/dattn72_B128 python scripts/attn_bench.py --sms 72 --B 128 --reps 4 > $out/ncu_dattn.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 6000 -c 1500 --csv \
  --log-file $out/launches_bench.csv python bench.py --steps 30 --warmup 3 --duration 10 --no-cpu-baseline \
  > $out/bench_under_ncu.log 2>&1
summ() { python -c "import json,sys; d=json.load(open('$1')); print(round(d['value']), 'tok/s p99', round(d['p99_itl_ms'],1), 'ms ttft50', round(d['p50_ttft_ms']), 'ms B', round(d['mean_decode_batch'] or 0), 'duty', d.get('stream_duty'), d['arm_decisions'])" 2>&1 | tail -1; }
timeout 400 python bench.py > $out/bench_default.json 2> $out/bench_default.err; echo "default cfg2: $(summ $out/bench_default.json)"
timeout 400 python bench.py --qps 56 --arm-profile profiles/arm/llama3.1-8b_ctx1152.json --no-cpu-baseline > $out/arm56.json 2> $out/arm56.err; echo "measured ARM q56: $(summ $out/arm56.json)"
timeout 400 python bench.py --qps 48 --arm --no-cpu-baseline > $out/refarm48.json 2> $out/refarm48.err; echo "reference ARM q48: $(summ $out/refarm48.json)"
for e in hybrid-2048 hybrid-512; do
  timeout 400 python bench.py --qps 48 --engine $e --no-cpu-baseline > $out/$e.json 2> $out/$e.err; echo "$e q48: $(summ $out/$e.json)"
done
timeout 300 python bench.py --impl reference > $out/bench_reference.json 2> $out/bench_reference.err; cat $out/bench_reference.json

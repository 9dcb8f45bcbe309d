#!/bin/bash
# ncu evidence for the round: full captures of the top kernels + the default bench command's launch list.
out=${1:-gpurun_out/ncu_final}
mkdir -p $out
timeout 300 ncu --set full --import-source on --clock-control none -k regex:decode_attn_tc -s 3 -c 1 \
  -o $out/dattn64_B192 python scripts/attn_bench.py --sms 64 --B 192 --reps 4 > $out/dattn.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:prefill_attn_tc -s 2 -c 1 \
  -o $out/pattn_T1023 python scripts/pattn_bench.py > $out/pattn.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_bf16 -s 16 -c 1 \
  -o $out/gemm_gateup_B192 python scripts/gemm_chain.py --sms 64 --batches 192 --shapes gate_up --n 8 > $out/gemm.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_bf16 -s 42 -c 1 \
  -o $out/gemm_prefill_gateup python scripts/prefill_variant.py > $out/gemm_prefill.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 20000 -c 2000 --csv \
  --log-file $out/launches_default_bench.csv python bench.py --steps 40 --warmup 3 --duration 14 --no-cpu-baseline \
  > $out/bench_under_ncu.log 2>&1
ls -la $out

#!/bin/bash
# ncu full capture of the decode QKV GEMM (B=128, 64-SM grid, full-device stream) and the O GEMM.
O=gpurun_out/gemm_ncu; mkdir -p $O
timeout 120 python scripts/gemm_chain.py --sms 64 --no-green --batches 128 --shapes qkv,o > $O/chain_nogreen.jsonl 2>&1
for sh in qkv o; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_bf16 --launch-skip 12 --launch-count 1 \
    -o $O/${sh}_B128_64sms python scripts/gemm_chain.py --sms 64 --no-green --batches 128 --shapes $sh --n 4 > $O/ncu_$sh.log 2>&1
done

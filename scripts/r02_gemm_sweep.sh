#!/bin/bash
# Decode QKV / O GEMM schedules on decode partitions (debug knobs of gemm_bf16_launch):
# variant -1 = default (stream-K), 0 = data-parallel whole tiles, 1 = two A sub-tiles,
# 3 = two sub-tiles + stream-K; pair -1 auto, 0 single-CTA tiles, 1 CTA pairs.
O=gpurun_out/gemm_sweep; mkdir -p $O
for sms in 32 48 64; do
  for v in -1 0 1 3; do
    for pr in -1 0 1; do
      timeout 200 python scripts/gemm_chain.py --sms $sms --batches 64,128,256 --shapes qkv,o --variant $v --pair $pr \
        2>>$O/err.log | sed "s/^{/{\"variant\": $v, \"pair\": $pr, /" >> $O/sweep.jsonl
    done
  done
done

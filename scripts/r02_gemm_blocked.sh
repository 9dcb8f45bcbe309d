#!/bin/bash
# Decode GEMMs with block-packed weights (one contiguous 16 KB TMA box per 128 x 64 k-block) vs row-major.
O=gpurun_out/gemm_blocked; mkdir -p $O
for sms in 32 48 64 148; do
  timeout 300 python scripts/gemm_chain.py --sms $sms --batches 64,128,256 > $O/plain_$sms.jsonl 2>> $O/err.log
  timeout 300 python scripts/gemm_chain.py --sms $sms --batches 64,128,256 --blocked > $O/blocked_$sms.jsonl 2>> $O/err.log
done

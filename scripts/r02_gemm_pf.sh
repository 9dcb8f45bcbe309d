#!/bin/bash
# Decode GEMM weight L2 lookahead: chains per projection on decode partitions, pf sweep.
set -x
O=gpurun_out/gemm_pf; mkdir -p $O
for sms in 32 48 64; do
  timeout 400 python scripts/gemm_chain.py --sms $sms --batches 64,128,256 --pf 0,4,8,16 > $O/chain_$sms.jsonl 2> $O/chain_$sms.err
done

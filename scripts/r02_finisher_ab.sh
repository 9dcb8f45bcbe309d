#!/bin/bash
# A/B of the stream-K finisher with the next chunk's partial requested one chunk ahead:
# GEMM parity tests, decode GEMM chains and traces, new build vs the previous one (RB_LIB).
O=gpurun_out/fin_ab; mkdir -p $O
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "linear" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python scripts/gemm_determinism.py --sms 32,64 > $O/det_new.jsonl 2>&1
for sms in 32 48 64; do
  timeout 300 python scripts/gemm_chain.py --sms $sms --batches 64,128,256 > $O/new_$sms.jsonl 2>> $O/err.log
  RB_LIB=paper_2601_11822_b200/_lib_ab/librapid_head.so timeout 300 python scripts/gemm_chain.py --sms $sms --batches 64,128,256 > $O/old_$sms.jsonl 2>> $O/err.log
done
timeout 120 python scripts/gemm_chain_trace.py --shape qkv --sms 64 --B 256 --n 4 > $O/trace_qkv_64_256_new.txt 2>&1

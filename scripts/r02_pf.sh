#!/bin/bash
# Decode attention L2 lookahead: parity, isolated sweep over partitions, beside a prefill GEMM.
# NOTE: measured a decode-attention L2 lookahead knob (--pf) that was reverted after this sweep
# (profiles/r02/dattn/dead_ends/l2_lookahead_*); kept as the record of how those files were made.
set -x
O=gpurun_out/pf; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "decode_attention" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python scripts/attn_bench.py --sms 32,48,64,96,148 --B 256 --pf 0,2,4,8,16 > $O/attn_bench.jsonl 2> $O/attn_bench.err
timeout 600 python scripts/contention_probe.py --sms 32,48,64 --B 256 --cases alone,gemm --pf 0,4,8 > $O/contention.jsonl 2> $O/contention.err

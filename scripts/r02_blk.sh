#!/bin/bash
# K3b (block-wide half-page stages) vs the per-warp kernel: parity, isolated partitions, beside a prefill GEMM.
# NOTE: shapes 5 / 6 (block-wide K3b, dims-split) were reverted after this run (diff and data:
# profiles/r02/dattn/dead_ends/blockwide/); kept as the record of how those files were made.
set -x
O=gpurun_out/blk2; mkdir -p $O
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k "decode_attention" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python scripts/attn_bench.py --sms 24,32,40,48,56,64,96,148 --B 128,256 --shapes 0,5,6 > $O/attn_bench.jsonl 2> $O/attn_bench.err
timeout 300 python scripts/contention_probe.py --sms 32,48 --B 256 --cases alone,gemm --pf -1 > $O/contention_base.jsonl 2> $O/contention.err

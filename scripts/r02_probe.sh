#!/bin/bash
# ncu env probe, K2 tile modes (+ parity), contention probe
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02d}
mkdir -p $out
timeout 120 ncu --metrics gpu__time_duration.sum -c 1 python -c "import torch,os; torch.zeros(1,device='cuda'); print('ENV', sorted(k for k in os.environ if 'INJ' in k or 'NV' in k or 'PRELOAD' in k or 'CUDA' in k))" > $out/ncu_env.log 2>&1; grep ENV $out/ncu_env.log
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k prefill_attention > $out/pattn_tests.log 2>&1; echo "pattn tests rc=$?"; tail -2 $out/pattn_tests.log
timeout 300 python scripts/pattn_bench.py > $out/pattn_bench.jsonl 2>&1; cat $out/pattn_bench.jsonl
timeout 600 python scripts/contention_probe.py --sms 56,88 > $out/contention.jsonl 2>&1; cat $out/contention.jsonl

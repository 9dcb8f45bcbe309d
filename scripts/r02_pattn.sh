#!/bin/bash
# K2 parity + timing + one ncu --set full capture at T=2048 after a 6144 prefix
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02f}
mkdir -p $out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k prefill_attention > $out/pattn_tests.log 2>&1; echo "pattn tests rc=$?"; tail -2 $out/pattn_tests.log
timeout 300 python scripts/pattn_bench.py --tiles 0 > $out/pattn_bench.jsonl 2>&1; cat $out/pattn_bench.jsonl
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_attn --launch-skip 2 -c 1 \
  -o $out/pattn_2048_6144 python scripts/pattn_bench.py --tiles 0 --cases 2048:6144 > $out/ncu.log 2>&1; echo "ncu rc=$?"
fi

#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02x}
mkdir -p $out
timeout 600 python -m pytest tests/test_realshape_gpu.py -q -x -k ksplit > $out/ksplit_tests.log 2>&1; echo "ksplit tests rc=$?"; tail -3 $out/ksplit_tests.log
for s in 48 72; do
  timeout 300 python scripts/step_bench.py --B 128,256 --decode-sms $s --pdl 1 --ksplit 0,1 --reps 3 >> $out/step.jsonl 2>&1
done
cat $out/step.jsonl
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "all gpu rc=$?"; tail -2 $out/pytest_gpu.log

#!/bin/bash
# Round-2 GPU evidence: gpu tests, smoke, default bench (RAPID + hybrid-2048 comparator),
# the kernel census of smoke() under ncu, reference arm.
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02}
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $out/smoke.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_ncu.log 2>&1
echo "ncu census rc=$? rb_launches=$(grep -c 'rb::' $out/smoke_launches.csv)"
timeout 900 python bench.py > $out/bench_default.json 2> $out/bench_default.err; echo "bench rc=$?"; tail -c 3000 $out/bench_default.json
timeout 600 python bench.py --steps 20 --warmup 5 > $out/bench_s20.json 2> $out/bench_s20.err; echo "bench20 rc=$?"; tail -c 1500 $out/bench_s20.json

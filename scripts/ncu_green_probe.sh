#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out/greenprobe
for v in plain memset memcpy ctx_sync ctx_cudafree event graph; do
  timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv \
    --log-file gpurun_out/greenprobe/$v.csv python scripts/green_ncu_probe.py $v > gpurun_out/greenprobe/$v.log 2>&1
  echo "$v rc=$? rmsnorm_rows=$(grep -c rmsnorm gpurun_out/greenprobe/$v.csv) $(grep -h 'ERROR' gpurun_out/greenprobe/$v.log gpurun_out/greenprobe/$v.csv | head -1)"
done
# skip-based: is it only the first green launch that fails?
timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -s 5 -c 20 --csv \
  --log-file gpurun_out/greenprobe/skip5.csv python scripts/green_ncu_probe.py plain > gpurun_out/greenprobe/skip5.log 2>&1
echo "skip5 rc=$? rmsnorm_rows=$(grep -c rmsnorm gpurun_out/greenprobe/skip5.csv)"

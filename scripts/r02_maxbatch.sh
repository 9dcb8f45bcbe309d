#!/bin/bash
# ncu census of smoke() (profiler-aware split), re-measured ARM tables (both sides strictly under load,
# batches to 384), balanced policy at max_batch 256 and 384, hybrid-2048 at max_batch 384.
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02c}
mkdir -p $out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_ncu.log 2>&1
echo "ncu census rc=$? rb_launches=$(grep -c 'rb::' $out/smoke_launches.csv)"; tail -2 $out/smoke_ncu.log
P=$out/llama3.1-8b_ctx1152_chunk1023_b384.json
timeout 1200 python -m paper_2601_11822_b200.profiler --model llama3.1-8b --ctx 1152 --chunk 1023 \
  --batches 1,2,4,8,16,32,48,64,96,128,160,192,224,256,288,320,352,384 --out $P > $out/prof.log 2>&1; echo "prof rc=$?"; tail -14 $out/prof.log
summ() { python -c "import json,sys; d=json.load(open('$1')); c=d.get('comparator') or {}; print(round(d['value']), 'win', round(d['device_window']['tokens_per_s'] or 0), 'p99', d['p99_itl_ms'], 'ttft50', d['p50_ttft_ms'], 'B', round(d['device_window']['mean_decode_batch'] or 0), d.get('arm_decisions'), '| hyb', round(c.get('value',0)), c.get('p99_itl_ms'))" 2>&1 | tail -1; }
for mb in 256 384; do
  timeout 600 python bench.py --arm-profile $P --arm-policy balanced --max-batch $mb --no-cpu-baseline --timeline $out/tl_bal$mb > $out/bal$mb.json 2> $out/bal$mb.err
  echo "balanced mb=$mb: $(summ $out/bal$mb.json)"
done
timeout 600 python bench.py --engine hybrid-2048 --max-batch 384 --compare none --no-cpu-baseline > $out/hyb384.json 2> $out/hyb384.err
echo "hybrid-2048 mb=384: $(summ $out/hyb384.json)"

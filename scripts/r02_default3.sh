#!/bin/bash
# The driver's default bench, three times on one box (variance of the headline), then the reference arm
# and the replica path at N=2 on the same GPU.
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02ai}
mkdir -p $out
summ() { python -c "import json,sys; d=json.load(open('$1')); c=d.get('comparator') or {}; print(round(d['value']), 'p99', d['p99_itl_ms'], 'ttft50', round(d['p50_ttft_ms']), 'roof', round(d['roofline']['frac'],3), 'clk', d['clocks'].get('sm_mhz'), 'W', d['clocks'].get('power_w'), 'host', d['host_loop']['decode_completion_to_next_launch']['median_us'], 'duty', d['stream_duty'], '| hyb', round(c.get('value',0)), c.get('p99_itl_ms'), 'ratio', round(d.get('vs_comparator') or 0, 4))" 2>&1 | tail -1; }
for i in 1 2 3; do
  timeout 700 python bench.py > $out/default$i.json 2> $out/default$i.err
  echo "default #$i: $(summ $out/default$i.json)"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $out/reference.json 2> $out/reference.err; echo "reference rc=$?"; tail -c 400 $out/reference.json
bash scripts/r02_replicas2.sh $out

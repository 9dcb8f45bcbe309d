#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02p}
mkdir -p $out
summ() { python -c "import json,sys; d=json.load(open('$1')); c=d.get('comparator') or {}; print(round(d['value']), 'win', round(d['device_window']['tokens_per_s'] or 0), 'p99', d['p99_itl_ms'], 'ttft50', round(d['p50_ttft_ms']), 'B', round(d['device_window']['mean_decode_batch'] or 0), 'duty', d['stream_duty'], 'host', d['host_loop'], 'clk', d['clocks'].get('sm_mhz'), '| hyb', round(c.get('value',0)), c.get('p99_itl_ms'), (c.get('clocks') or {}).get('sm_mhz'))" 2>&1 | tail -1; }
for ps in 0 50; do
  timeout 600 python bench.py --poll-sleep-us $ps --no-cpu-baseline > $out/bal_ps$ps.json 2> $out/bal_ps$ps.err
  echo "balanced poll_sleep=$ps: $(summ $out/bal_ps$ps.json)"
done
timeout 600 python bench.py --arm-policy feedback --no-cpu-baseline > $out/fb.json 2> $out/fb.err
echo "feedback: $(summ $out/fb.json)"

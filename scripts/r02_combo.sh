#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02q}
mkdir -p $out
NCU=0 bash scripts/r02_pattn.sh $out/pattn
bash scripts/r02_tp.sh $out/tp
summ() { python -c "import json,sys; d=json.load(open('$1')); c=d.get('comparator') or {}; print(round(d['value']), 'win', round(d['device_window']['tokens_per_s'] or 0), 'p99', d['p99_itl_ms'], 'ttft50', round(d['p50_ttft_ms']), 'B', round(d['device_window']['mean_decode_batch'] or 0), 'duty', d['stream_duty'], 'host', d['host_loop']['decode_completion_to_next_launch'], 'clk', d['clocks'].get('sm_mhz'), '| hyb', round(c.get('value',0)), c.get('p99_itl_ms'), (c.get('clocks') or {}).get('sm_mhz'))" 2>&1 | tail -1; }
timeout 600 python bench.py --no-cpu-baseline > $out/bal.json 2> $out/bal.err
echo "balanced: $(summ $out/bal.json)"

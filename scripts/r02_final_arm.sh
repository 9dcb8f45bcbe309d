#!/bin/bash
# Final kernels: re-measured ARM tables (batches to 320), then RAPID (feedback / balanced, max_batch
# 256 and 320) against hybrid-2048 on the same trace, with clocks and board power.
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02ag}
mkdir -p $out
P=$out/llama3.1-8b_ctx1152_chunk1023.json
timeout 1500 python -m paper_2601_11822_b200.profiler --model llama3.1-8b --ctx 1152 --chunk 1023 \
  --batches 1,2,4,8,16,32,48,64,96,128,160,192,224,256,288,320 --out $P > $out/prof.log 2>&1; echo "prof rc=$?"
summ() { python -c "import json,sys; d=json.load(open('$1')); c=d.get('comparator') or {}; print(round(d['value']), 'p99', d['p99_itl_ms'], 'ttft50', round(d['p50_ttft_ms']), 'B', round(d['device_window']['mean_decode_batch'] or 0), 'clk', d['clocks'].get('sm_mhz'), 'W', d['clocks'].get('power_w'), 'tpj', d.get('tokens_per_joule'), d.get('arm_decisions',{}).get('decode_sms') if d.get('arm_decisions') else None, '| hyb', round(c.get('value',0)), c.get('p99_itl_ms'), (c.get('clocks') or {}).get('sm_mhz'), (c.get('clocks') or {}).get('power_w'), c.get('tokens_per_joule'))" 2>&1 | tail -1; }
for cfg in "feedback 256" "balanced 256" "feedback 320"; do
  set -- $cfg
  timeout 700 python bench.py --arm-profile $P --arm-policy $1 --max-batch $2 --no-cpu-baseline > $out/$1_$2.json 2> $out/$1_$2.err
  echo "$1 mb=$2: $(summ $out/$1_$2.json)"
done

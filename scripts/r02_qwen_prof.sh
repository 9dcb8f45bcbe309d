#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02ap}
mkdir -p $out
P=$out/qwen2.5-14b_ctx8256.json
timeout 2400 python -m paper_2601_11822_b200.profiler --model qwen2.5-14b --ctx 8256 --chunk 2048 --out $P > $out/prof.log 2>&1; echo "prof rc=$?"; tail -3 $out/prof.log | cut -c1-150
summ() { python -c "import json,sys; d=json.load(open('$1')); c=d.get('comparator') or {}; print(round(d['value']), 'p99', d['p99_itl_ms'], d.get('arm_decisions'), '|', c.get('engine'), round(c.get('value',0)), c.get('p99_itl_ms'))" 2>&1 | tail -1; }
timeout 900 python bench.py --model qwen2.5-14b --prompt 8192 --output 128 --qps 3.5 --arm-profile $P --compare hybrid-512 --no-cpu-baseline > $out/q14.json 2> $out/q14.err
echo "cfg5 new tables: $(summ $out/q14.json)"

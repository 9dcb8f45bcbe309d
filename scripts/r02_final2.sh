#!/bin/bash
# cfg 5 on the final kernels; the default bench at the driver's short settings (--steps 20 --warmup 5)
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02an}
mkdir -p $out
bash scripts/r02_cfg5.sh $out
timeout 700 python bench.py --steps 20 --warmup 5 > $out/default_s20.json 2> $out/default_s20.err
python -c "import json; d=json.load(open('$out/default_s20.json')); print('s20', round(d['value']), 'hyb', round(d['comparator']['value']), d['p99_itl_ms'], d['ms_per_step'])"

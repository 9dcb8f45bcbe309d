#!/bin/bash
# cfg 5 under the BASELINE metric as defined (max over QPS of the run-level tokens/s at p99 ITL <= 50 ms):
# Qwen2.5-14B 8192/128, RAPID (measured ARM, default policy) and hybrid-512 / hybrid-1024 on the same trace per QPS.
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/cfg5_sweep}
mkdir -p $out
for q in 2.5 3.0 3.5 4.0 4.5; do
  for cmp in hybrid-512 hybrid-1024; do
    timeout 900 python bench.py --model qwen2.5-14b --prompt 8192 --output 128 --qps $q --compare $cmp --no-cpu-baseline \
      > $out/q${q}_$cmp.json 2> $out/q${q}_$cmp.err
    python -c "import json; d=json.load(open('$out/q${q}_$cmp.json')); c=d['comparator']; print('qps $q', 'rapid', round(d['value']), round(d['tokens_per_s_unconstrained']), 'p99', d['p99_itl_ms'], '|', c['engine'], round(c['value']), round(c['tokens_per_s_unconstrained']), 'p99', c['p99_itl_ms'])"
  done
done

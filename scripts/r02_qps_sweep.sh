#!/bin/bash
# BASELINE metric as defined (max over a QPS sweep of the run-level tokens/s subject to p99 ITL <= 50 ms):
# RAPID (default policy) with hybrid-2048 on the same trace at each QPS.
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02ax}
mkdir -p $out
for q in 24 32 40 48 56 64; do
  timeout 700 python bench.py --qps $q --steps 200 --warmup 20 --no-cpu-baseline > $out/q$q.json 2> $out/q$q.err
  python -c "import json; d=json.load(open('$out/q$q.json')); c=d['comparator']; print('qps $q', 'rapid', round(d['value']), round(d['tokens_per_s_unconstrained']), 'p99', d['p99_itl_ms'], 'ttft50', round(d['p50_ttft_ms']), 'goodput', round(d['goodput_req_s'],2), '| hyb', round(c['value']), round(c['tokens_per_s_unconstrained']), 'p99', c['p99_itl_ms'], 'ttft50', round(c['p50_ttft_ms']), 'goodput', round(c['goodput_req_s'],2))"
done

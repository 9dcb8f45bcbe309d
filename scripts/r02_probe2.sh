#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02e}
mkdir -p $out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_ncu.log 2>&1
echo "ncu census rc=$? rb_launches=$(grep -c 'rb::' $out/smoke_launches.csv)"; tail -2 $out/smoke_ncu.log
timeout 300 python scripts/pattn_bench.py --tiles 0 > $out/pattn_bench.jsonl 2>&1; cat $out/pattn_bench.jsonl
timeout 600 python scripts/contention_probe.py --sms 56,88 > $out/contention.jsonl 2>&1; cat $out/contention.jsonl

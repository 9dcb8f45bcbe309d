#!/bin/bash
# ncu evidence on the final kernels: launch lists of one decode step (B=256, ctx 1152, 48-SM grids) and one
# prefill chunk (T=1023, 100-SM grids) - cold, serialised: shares, not absolutes - and full captures of
# decode attention (48-SM grid) and prefill attention (2048 after 6144).
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02ak}
mkdir -p $out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_decode_B256_48sms.csv \
  python scripts/profile_step.py --B 256 --ctx 1152 --decode-sms 48 --what decode --reps 2 --no-green > $out/ls_dec.log 2>&1; echo "dec rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_prefill_T1023_100sms.csv \
  python scripts/profile_step.py --B 8 --T 1023 --decode-sms 48 --what prefill --reps 2 --no-green > $out/ls_pre.log 2>&1; echo "pre rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_attn_tc --launch-skip 3 -c 1 \
  -o $out/dattn48_B224 python scripts/attn_bench.py --sms 48 --B 224 --no-green --reps 2 > $out/dattn.log 2>&1; echo "dattn rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_attn --launch-skip 2 -c 1 \
  -o $out/pattn_2048_6144 python scripts/pattn_bench.py --tiles 0 --cases 2048:6144 > $out/pattn.log 2>&1; echo "pattn rc=$?"

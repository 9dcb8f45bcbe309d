#!/bin/bash
# cfg-4 serving path at world 2 on ONE GPU (two processes time-sliced on one device, peer-memory
# all-reduce): the code the 8-GPU run takes with --tp-ar nccl, validated for lockstep, no
# deadlock and the reference invariants. Tiny model: every all-reduce round trip crosses a
# context switch here, so the 8B model would take hours.
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02q}
mkdir -p $out
for ar in ${ARS:-peer push}; do
RB_WATCHDOG_S=${WD:-150} RB_DEBUG_WARMUP=1 RB_DEBUG_TP=1 timeout ${TPT:-300} python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
  bench.py --tp 2 --tp-ar $ar --model ${TPMODEL:-tiny} --qps 2 --duration 8 --steps 12 --warmup 3 --prompt 96 --output 24 \
  --max-batch 16 --kv-memory-fraction 0.3 --decode-sms 72 --no-cpu-baseline > $out/tp2_$ar.json 2> $out/tp2_$ar.err
echo "tp2 $ar rc=$?"; tail -c 1500 $out/tp2_$ar.json; grep -h "tp_rank\|Error\|error" $out/tp2_$ar.err | tail -5
done

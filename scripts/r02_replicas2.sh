#!/bin/bash
# Replica path (cfg 3 at N=2) on ONE GPU: two ranks share the device (gloo), each serves requests
# i mod 2 with its own engine, pool and green contexts; pooled run-level stats, max-over-ranks window.
cd "$(dirname "$0")/.." || exit 1
out=${1:-gpurun_out/r02ah}
mkdir -p $out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 \
  bench.py --gpus 2 --qps 20 --steps 100 --warmup 10 --kv-memory-fraction 0.4 --compare none --no-cpu-baseline \
  > $out/replicas2.json 2> $out/replicas2.err
echo "replicas2 rc=$?"; tail -c 800 $out/replicas2.json; grep -i "error" $out/replicas2.err | tail -3

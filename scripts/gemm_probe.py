"""Focused GEMM experiments: split-K on/off, tile counts, host overhead per call."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402
from scripts.kbench import timeit  # noqa: E402

dev = "cuda"
sc = ops.GemmScratch(dev)
flush = torch.empty(256 << 20, dtype=torch.int8, device=dev)
for (T, O, K, mode) in [(256, 6144, 4096, 2), (64, 6144, 4096, 2), (1024, 4096, 4096, 1), (1024, 6144, 4096, 1),
                        (2048, 4096, 4096, 1)]:
    x = torch.randn(T, K, device=dev).bfloat16()
    w = (torch.randn(O, K, device=dev) * 0.02).bfloat16()
    y = torch.empty(T, O, device=dev, dtype=torch.bfloat16)
    for use in (True, False):
        ms = timeit(lambda: ops.linear(x, w, out=y, mode=mode, scratch=sc if use else None), flush=flush)
        print(json.dumps(dict(T=T, O=O, K=K, mode=mode, splitk=use, us=ms * 1e3,
                              tflops=2 * T * O * K / ms / 1e9)), flush=True)
    for _ in range(5):
        ops.linear(x, w, out=y, mode=mode, scratch=sc)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 50
    for _ in range(n):
        ops.linear(x, w, out=y, mode=mode, scratch=sc)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(json.dumps(dict(T=T, host_us_per_call=(t1 - t0) / n * 1e6, wall_us_per_call=(t2 - t0) / n * 1e6)),
          flush=True)

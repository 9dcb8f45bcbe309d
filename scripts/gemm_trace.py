"""Timeline of one GEMM launch from in-kernel globaltimer stamps."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402

dev = "cuda"
lib = ops.load()
for (T, O, K, mode, split) in [(256, 6144, 4096, 2, False), (256, 6144, 4096, 2, True), (64, 6144, 4096, 2, False),
                               (1024, 4096, 4096, 1, False), (2048, 28672, 4096, 1, False)]:
    x = torch.randn(T, K, device=dev).bfloat16()
    w = (torch.randn(O, K, device=dev) * 0.02).bfloat16()
    y = torch.empty(T, O, device=dev, dtype=torch.bfloat16)
    sc = ops.GemmScratch(dev) if split else None
    tr = torch.zeros(148 * 8, dtype=torch.int64, device=dev)
    for _ in range(3):
        ops.linear(x, w, out=y, mode=mode, scratch=sc)
    torch.cuda.synchronize()
    lib.rb_debug_gemm_trace(tr.data_ptr())
    ops.linear(x, w, out=y, mode=mode, scratch=sc)
    torch.cuda.synchronize()
    lib.rb_debug_gemm_trace(None)
    t = tr.view(148, 8).cpu()
    used = t[:, 0] > 0
    t = t[used]
    t0 = t[:, 0].min()
    rel = (t - t0).float() / 1000.0  # us
    print(f"T={T} O={O} K={K} mode={mode} split={split} ctas={int(used.sum())}")
    names = ["start", "setup", "mma_first_full", "mma_last_full", "epi_tfull", "epi_done", "end"]
    for i, nm in enumerate(names):
        col = rel[:, i]
        print(f"  {nm:16s} min {col.min():8.2f} med {col.median():8.2f} max {col.max():8.2f} us")

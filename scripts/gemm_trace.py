"""Timeline of one GEMM launch from in-kernel globaltimer stamps."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402

dev = "cuda"
lib = ops.load()
sc = ops.GemmScratch(dev)
shapes = [(128, 6144, 4096, 2, 72), (128, 28672, 4096, 2, 72), (128, 4096, 14336, 2, 72), (1023, 28672, 4096, 1, 76)]
if len(sys.argv) > 1:
    shapes = [tuple(map(int, sys.argv[1:6]))]
for (T, O, K, mode, sms) in shapes:
    x = torch.randn(T, K, device=dev).bfloat16()
    w = (torch.randn(O, K, device=dev) * 0.02).bfloat16()
    y = torch.empty(T, O, device=dev, dtype=torch.bfloat16)
    tr = torch.zeros(16 * 148 * 16, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.int8, device=dev)
    for _ in range(3):
        ops.linear(x, w, out=y, mode=mode, num_sms=sms, scratch=sc)
    flush.zero_()
    torch.cuda.synchronize()
    lib.rb_debug_gemm_trace(tr.data_ptr())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    ops.linear(x, w, out=y, mode=mode, num_sms=sms, scratch=sc)
    ev1.record()
    torch.cuda.synchronize()
    print(f"  event-timed launch: {ev0.elapsed_time(ev1) * 1e3:.2f} us")
    lib.rb_debug_gemm_trace(None)
    t = tr[: 148 * 16].view(148, 16).cpu()
    used = t[:, 0] > 0
    t = t[used]
    t0 = t[:, 0].min()
    rel = (t - t0).float() / 1000.0  # us
    print(f"T={T} O={O} K={K} mode={mode} sms={sms} ctas={int(used.sum())}")
    names = ["start", "setup", "mma_first_full", "mma_last_full", "epi_tfull", "epi_done", "end", "c_stored", "c_published", "f_in", "f_done"]
    for i, nm in enumerate(names):
        col = rel[:, i]
        ok = col[t[:, i] > 0] if i in (2, 3) else col
        if ok.numel() == 0:
            continue
        print(f"  {nm:16s} min {ok.min():8.2f} med {ok.median():8.2f} max {ok.max():8.2f} us")

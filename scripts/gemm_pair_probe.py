"""Pair (cta_group::2) vs single-CTA GEMM: correctness + graph-timed speed."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa
from scripts.kbench import timeit  # noqa
lib = ops.load()
dev = "cuda"
sc = ops.GemmScratch(dev)
flush = torch.empty(256 << 20, dtype=torch.int8, device=dev)
shapes = [(1024, 6144, 4096, 1, 148), (1024, 4096, 4096, 1, 148), (1024, 28672, 4096, 1, 148), (1024, 4096, 14336, 1, 148),
          (2048, 28672, 4096, 1, 148), (1023, 28672, 4096, 1, 76), (1023, 6144, 4096, 1, 76),
          (128, 6144, 4096, 2, 72), (128, 4096, 4096, 2, 72), (128, 28672, 4096, 2, 72), (128, 4096, 14336, 2, 72),
          (64, 6144, 4096, 2, 72), (256, 6144, 4096, 2, 148), (8, 4096, 4096, 2, 72)]
for (T, O, K, mode, sms) in shapes:
    x = torch.randn(T, K, device=dev).bfloat16()
    w = (torch.randn(O, K, device=dev) * 0.02).bfloat16()
    ref = (x.float() @ w.float().T)
    row = dict(T=T, O=O, K=K, mode=mode, sms=sms)
    for pm in (0, 1):
        lib.rb_debug_gemm_pair_mode(pm)
        y = torch.empty(T, O, device=dev, dtype=torch.bfloat16)
        ops.linear(x, w, out=y, mode=mode, num_sms=sms, scratch=sc)
        torch.cuda.synchronize()
        err = float((y.float() - ref).norm() / ref.norm())
        ms = timeit(lambda: ops.linear(x, w, out=y, mode=mode, num_sms=sms, scratch=sc), flush=flush if mode == 2 else None)
        row[f"{'pair' if pm else 'single'}_us"] = round(ms * 1e3, 2)
        row[f"{'pair' if pm else 'single'}_err"] = err
        if mode == 1:
            row[f"{'pair' if pm else 'single'}_tflops"] = round(2 * T * O * K / ms / 1e9, 1)
        else:
            row[f"{'pair' if pm else 'single'}_wgbs"] = round(O * K * 2 / ms / 1e6, 1)
    lib.rb_debug_gemm_pair_mode(-1)
    print(json.dumps(row), flush=True)

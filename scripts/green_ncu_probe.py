"""Which first operation on a green context lets ncu profile the kernels launched there?
(driver census failure probe: ncu 2025.2 fails "Failed to prepare kernel for profiling" on
the first kernel launched in a green context, rc 9)

    ncu ... python scripts/green_ncu_probe.py <variant>
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402

v = sys.argv[1]
lib = ops.load()
torch.cuda.set_device(0)
x = torch.randn(64, 1024, device="cuda").bfloat16()
w = torch.ones(1024, device="cuda").bfloat16()
y = torch.empty_like(x)
gs = ops.GreenSplit(72)
ds = gs.streams[0]
cudart = ctypes.CDLL("libcudart.so.12")
cuda = ctypes.CDLL("libcuda.so.1")
if v == "memset":
    assert cudart.cudaMemsetAsync(ctypes.c_void_p(y.data_ptr()), 0, 1024, ctypes.c_void_p(ds.cuda_stream)) == 0
    ds.synchronize()
if v == "memcpy":
    h = torch.zeros(1024, dtype=torch.uint8, pin_memory=True)
    assert cudart.cudaMemcpyAsync(ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(h.data_ptr()), 1024, 1,
                                  ctypes.c_void_p(ds.cuda_stream)) == 0
    ds.synchronize()
if v == "ctx_sync":
    ops._check(lib.rb_debug_green_ctx_push(gs.handle, 0), "push")
    assert cuda.cuCtxSynchronize() == 0
    ops._check(lib.rb_debug_ctx_pop(), "pop")
if v == "ctx_cudafree":
    ops._check(lib.rb_debug_green_ctx_push(gs.handle, 0), "push")
    cudart.cudaFree(ctypes.c_void_p(0))
    ops._check(lib.rb_debug_ctx_pop(), "pop")
if v == "event":
    e = torch.cuda.Event()
    e.record(ds)
    e.synchronize()
if v == "graph":
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=ds):
        ops.rmsnorm(x, w, y, 1e-5, stream=ds)
    g.replay()
    ds.synchronize()
for _ in range(3):
    ops.rmsnorm(x, w, y, 1e-5, stream=ds)
torch.cuda.synchronize()
print("probe", v, "ok", float(y.float().abs().mean()))

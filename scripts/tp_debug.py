"""Standalone checks of the TP collectives on one GPU (two in-process ranks)."""
import ctypes
import faulthandler
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402
from paper_2601_11822_b200.tp import _vp_array, nccl_unique_id  # noqa: E402

faulthandler.dump_traceback_later(40, exit=True)
lib = ops.load()
what = sys.argv[1] if len(sys.argv) > 1 else "peer"
if what == "nccl":
    print("nccl available", lib.rb_tp_nccl_available(), flush=True)
    uid = nccl_unique_id()
    print("uid ok", flush=True)
    comm = ctypes.c_void_p()
    ops._check(lib.rb_tp_nccl_comm_init(uid, 1, 0, ctypes.byref(comm)), "init")
    print("comm ok", flush=True)
    keys = torch.zeros(8, dtype=torch.int64, device="cuda")
    h = ctypes.c_void_p()
    ops._check(lib.rb_tp_create(1, 0, 1, comm.value, None, None, _vp_array([keys.data_ptr()]), None, None, 0,
                                ctypes.byref(h)), "create")
    x = torch.randn(4096, device="cuda").bfloat16()
    y = x.clone()
    ops._check(lib.rb_tp_allreduce(h.value, y.data_ptr(), 4096, torch.cuda.current_stream().cuda_stream), "ar")
    torch.cuda.synchronize()
    print("nccl world1 identity:", torch.equal(x, y), flush=True)
    sys.exit(0)
world = 2
n = 8192 * 16
gs = ops.GreenSplit(74)
words = lib.rb_tp_flag_words()
part = [[torch.zeros(n, dtype=torch.bfloat16, device="cuda") for _ in range(world)] for _ in range(2)]
keys = [torch.zeros(8, dtype=torch.int64, device="cuda") for _ in range(world)]
flags = [torch.zeros(words, dtype=torch.int32, device="cuda") for _ in range(world)]
epochs = [torch.zeros(128, dtype=torch.int32, device="cuda") for _ in range(world)]
hs = []
for r in range(world):
    h = ctypes.c_void_p()
    ops._check(lib.rb_tp_create(world, r, 2, None, _vp_array([t.data_ptr() for t in part[0]]),
                                _vp_array([t.data_ptr() for t in part[1]]), _vp_array([t.data_ptr() for t in keys]),
                                _vp_array([t.data_ptr() for t in flags]), epochs[r].data_ptr(), n,
                                ctypes.byref(h)), "create")
    hs.append(h.value)
xs = [torch.randn(n, device="cuda").bfloat16() for _ in range(world)]
want = (xs[0].float() + xs[1].float())
torch.cuda.synchronize()
for it in range(3):
    ys = [x.clone() for x in xs]
    torch.cuda.synchronize()
    for r in range(world):
        ops._check(lib.rb_tp_allreduce(hs[r], ys[r].data_ptr(), n, gs.stream_handles[r]), "ar")
    print("launched", it, flush=True)
    torch.cuda.synchronize()
    print("iter", it, "rank0 err", float((ys[0].float() - want).abs().max()), "ranks equal", torch.equal(ys[0], ys[1]),
          flush=True)

"""Tensor parallelism for the decoder (cfg 4: Llama-3.1-70B, TP=8).

The reference folds tp into one aggregate GPU (GpuSpec.aggregate, pkg/src/pdsim/core.py:
147-165) and prices no collective; here the shards are physical:

  * QKV, gate|up: column-parallel (rank r owns q heads [r*Hq/w, ...), kv heads
    [r*Hkv/w, ...), intermediate rows [r*I/w, ...));
  * O, down: row-parallel (the matching input columns); their GEMM writes a partial and
    one all-reduce per GEMM (2 per layer) restores the replicated residual stream;
  * lm_head: vocab-parallel (rows [r*V/w, ...)); greedy sampling max-reduces packed
    (logit, -index) keys, so ties resolve to the lowest global id as torch.argmax does;
  * embedding, norms: replicated. KV cache: each rank holds its kv heads only.

Collectives (csrc/tp.cu): NCCL (mode 1, one communicator per phase stream) or the
one-shot peer-memory all-reduce with the residual add fused (mode 2). `IpcPeerGroup` wires
mode 2 for one rank per process through cudaIpc handles — on a real node across GPUs, in
the single-GPU tests across two processes sharing the device (the same code path; ranks in
ONE process are not supported: a rank's spinning all-reduce would block the other rank's
kernels queued behind it on a shared hardware queue).
"""

from __future__ import annotations

import ctypes
import dataclasses

import torch

from paper_2601_11822_b200 import ops
from paper_2601_11822_b200.specs import ArchConfig

ID_BYTES = 128
AR_FLAG_SLOTS = 128


def local_arch(arch: ArchConfig, world: int) -> ArchConfig:
    """This rank's shard shape (heads, intermediate and vocab divided by `world`)."""
    for what, n in (("q_heads", arch.q_heads), ("kv_heads", arch.kv_heads), ("intermediate", arch.intermediate),
                    ("vocab", arch.vocab)):
        if n % world:
            raise ValueError(f"tp: {what}={n} is not divisible by world={world}")
    if (arch.intermediate // world) % 16:
        raise ValueError("tp: the intermediate shard must be a multiple of 16 (SwiGLU row blocks)")
    return dataclasses.replace(arch, q_heads=arch.q_heads // world, kv_heads=arch.kv_heads // world,
                               intermediate=arch.intermediate // world, vocab=arch.vocab // world,
                               tie_embeddings=False)


def shard_state(arch: ArchConfig, state: dict, rank: int, world: int) -> dict:
    """Rank `rank`'s slice of an oracle-named fp32 state dict (oracle/llama_fp32.py)."""
    la = local_arch(arch, world)
    D = arch.head_dim
    q0, q1 = rank * la.q_heads * D, (rank + 1) * la.q_heads * D
    k0, k1 = rank * la.kv_heads * D, (rank + 1) * la.kv_heads * D
    i0, i1 = rank * la.intermediate, (rank + 1) * la.intermediate
    v0, v1 = rank * la.vocab, (rank + 1) * la.vocab
    out = {"embed": state["embed"], "norm": state["norm"],
           "lm_head": state.get("lm_head", state["embed"])[v0:v1]}
    for i in range(arch.layers):
        p = f"layers.{i}."
        out[p + "ln1"] = state[p + "ln1"]
        out[p + "ln2"] = state[p + "ln2"]
        out[p + "q"] = state[p + "q"][q0:q1]
        out[p + "k"] = state[p + "k"][k0:k1]
        out[p + "v"] = state[p + "v"][k0:k1]
        if arch.qkv_bias:
            out[p + "bq"] = state[p + "bq"][q0:q1]
            out[p + "bk"] = state[p + "bk"][k0:k1]
            out[p + "bv"] = state[p + "bv"][k0:k1]
        out[p + "o"] = state[p + "o"][:, q0:q1]
        out[p + "gate"] = state[p + "gate"][i0:i1]
        out[p + "up"] = state[p + "up"][i0:i1]
        out[p + "down"] = state[p + "down"][:, i0:i1]
    return out


def reference_tp_forward(arch: ArchConfig, state: dict, world: int, ids: torch.Tensor) -> torch.Tensor:
    """fp32 CPU restatement of the sharded math (test helper): the full-vocab logits of a
    prompt computed shard by shard, partials summed where the GPU all-reduces."""
    from oracle.llama_fp32 import Oracle

    orc = Oracle(arch, state)
    return orc.forward_tp(ids.long(), [shard_state(arch, state, r, world) for r in range(world)], local_arch(arch,
                                                                                                               world))


class TpContext:
    """One phase's TP handle (rb_tp_create) plus the device buffers it points at."""

    def __init__(self, handle: int, keep: list):
        self.handle = handle
        self._keep = keep

    def close(self) -> None:
        if self.handle:
            ops.load().rb_tp_destroy(self.handle)
            self.handle = 0


def _vp_array(ptrs):
    return (ctypes.c_void_p * len(ptrs))(*ptrs)


class _PhaseBuffers:
    """One rank's mode-2 buffers for one phase: two staging buffers [rows, H] bf16, argmax
    keys [rows] uint64, a zeroed flag array and zeroed per-CTA round counters."""

    def __init__(self, rows: int, H: int, device, slots: int = 1):
        words = ops.load().rb_tp_flag_words()
        # mode 2: this rank's partial; mode 3: one receive slot per sender rank
        self.part = [torch.zeros(slots * rows, H, dtype=torch.bfloat16, device=device) for _ in range(2)]
        self.keys = torch.zeros(rows, dtype=torch.int64, device=device)
        self.flags = torch.zeros(words, dtype=torch.int32, device=device)
        self.epoch = torch.zeros(AR_FLAG_SLOTS, dtype=torch.int32, device=device)

    def shared(self) -> list[torch.Tensor]:
        return [self.part[0], self.part[1], self.keys, self.flags]


def _ipc_handle(t: torch.Tensor):
    """cudaIpc handle of a tensor's storage (torch's own CUDA IPC export)."""
    return (t.untyped_storage()._share_cuda_(), t.storage_offset(), t.numel(), t.dtype)


def _ipc_open(h, device) -> torch.Tensor:
    storage = torch.UntypedStorage._new_shared_cuda(*h[0])
    out = torch.empty(0, dtype=h[3], device=device)
    out.set_(storage, h[1], (h[2],))
    return out


class IpcPeerGroup:
    """Peer-memory contexts for one rank per process (the multi-GPU layout).

    Every rank allocates its buffers, exports cudaIpc handles through `pg` (a
    torch.distributed group, gloo or NCCL) and maps its peers' buffers (NVLink P2P across
    GPUs; the same device across processes in the tests). mode 2: the one-shot all-reduce
    kernel reads the peers' staging buffers; mode 3: the row-parallel GEMM's epilogue pushes
    its tiles into the peers' receive slots and the reduce reads only local memory."""

    def __init__(self, runner, rank: int, world: int, pg=None, device="cuda", mode: int = 2):
        import torch.distributed as dist

        if mode not in (2, 3):
            raise ValueError("IpcPeerGroup: mode 2 (pull all-reduce) or 3 (GEMM push)")
        lib = ops.load()
        self.contexts: dict[str, TpContext] = {}
        self._keep = []
        for phase in ("pre", "dec"):
            buf = getattr(runner, phase)
            rows, H = buf.x.shape
            mine = _PhaseBuffers(rows, H, device, slots=world if mode == 3 else 1)
            handles = [None] * world
            dist.all_gather_object(handles, [_ipc_handle(t) for t in mine.shared()], group=pg)
            views = []
            for j in range(world):
                views.append(mine.shared() if j == rank else [_ipc_open(h, device) for h in handles[j]])
            ptr = [[v[k].data_ptr() for v in views] for k in range(4)]
            h = ctypes.c_void_p()
            ops._check(lib.rb_tp_create(world, rank, mode, None, _vp_array(ptr[0]), _vp_array(ptr[1]),
                                        _vp_array(ptr[2]), _vp_array(ptr[3]), mine.epoch.data_ptr(), rows * H,
                                        ctypes.byref(h)), "rb_tp_create")
            ctx = TpContext(h.value, [mine, views])
            buf.tp = ctx
            self.contexts[phase] = ctx


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(ID_BYTES)
    ops._check(ops.load().rb_tp_nccl_unique_id(buf), "rb_tp_nccl_unique_id")
    return buf.raw


class NcclPhaseComms:
    """Mode-1 contexts for one rank: one NCCL communicator per phase.

    `ids` = {"pre": 128-byte unique id, "dec": ...}, identical on every rank (rank 0
    creates them with nccl_unique_id() and broadcasts them)."""

    def __init__(self, runner, rank: int, world: int, ids: dict, device="cuda"):
        lib = ops.load()
        if not lib.rb_tp_nccl_available():
            raise RuntimeError("tp: libnccl.so.2 is not loadable")
        self.comms = {}
        for phase in ("pre", "dec"):
            comm = ctypes.c_void_p()
            ops._check(lib.rb_tp_nccl_comm_init(ids[phase], world, rank, ctypes.byref(comm)), "rb_tp_nccl_comm_init")
            self.comms[phase] = comm.value
            buf = getattr(runner, phase)
            keys = torch.zeros(buf.x.shape[0], dtype=torch.int64, device=device)
            key_ptrs = [0] * world
            key_ptrs[rank] = keys.data_ptr()
            h = ctypes.c_void_p()
            ops._check(lib.rb_tp_create(world, rank, 1, comm.value, None, None, _vp_array(key_ptrs), None, None, 0,
                                        ctypes.byref(h)), "rb_tp_create")
            buf.tp = TpContext(h.value, [keys])

    def close(self) -> None:
        lib = ops.load()
        for c in self.comms.values():
            lib.rb_tp_nccl_comm_destroy(c)
        self.comms = {}

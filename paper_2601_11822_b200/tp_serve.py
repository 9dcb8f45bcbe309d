"""cfg 4 end to end: the RAPID engine over a tensor-parallel B200 executor, one process per GPU.

The reference folds TP into one aggregate GPU (GpuSpec.aggregate, pkg/src/pdsim/core.py:147-165)
and prices no collective. Here every rank holds its shard (tp.local_arch: q/kv heads,
intermediate rows and lm_head vocab rows divided by the world; embedding and norms replicated)
and its slice of the paged KV cache; rank 0 runs RapidEngine + its B200Executor and every
worker rank replays rank 0's device commands (tp_engine.CommandChannel: fixed-size int32
frames over a host gloo group) on its shard, in the same order, on the same green-context
split. The row-parallel O / down projections all-reduce inside the forward (tp.py / csrc/tp.cu:
NCCL, one communicator per phase stream, or the peer-memory all-reduce), so collectives line
up across ranks by construction; the vocab-parallel argmax is a max-reduce, so sampled ids are
identical on every rank and only rank 0 reads them back.

    build_tp_executor(arch, rank, world, host_group, ar="nccl", ...) -> B200Executor (attached)
    rank 0:  attach_leader(ex, channel); ... drive RapidEngine ...; stop_workers(channel)
    rank r:  ex.warmup(...same splits as rank 0...); serve_worker(ex, channel)
"""

from __future__ import annotations

import torch

from paper_2601_11822_b200.executor_b200 import B200Executor
from paper_2601_11822_b200.model import DecoderWeights
from paper_2601_11822_b200.specs import ArchConfig
from paper_2601_11822_b200.tp import IpcPeerGroup, NcclPhaseComms, local_arch, nccl_unique_id
from paper_2601_11822_b200.traffic import prompt_token_ids

AR_MODES = {"nccl": 1, "peer": 2, "push": 3}


def agreed_num_blocks(local_blocks: int, host_group) -> int:
    """Every rank's cache must hold every page id rank 0's pool hands out: the pool is the
    smallest cache over the ranks."""
    import torch.distributed as dist

    t = torch.tensor([local_blocks], dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=host_group)
    return int(t.item())


def build_tp_executor(arch: ArchConfig, rank: int, world: int, host_group, *, ar: str = "nccl",
                      device: str = "cuda", state: dict | None = None, **executor_kw) -> B200Executor:
    """This rank's sharded executor with its collectives attached (see the module docstring).

    `state`: a full-model fp32 state dict to shard (default: random weights of the real shapes).
    `ar`: "nccl" (mode 1; NVLink / NVSwitch across GPUs), "peer" (mode 2: one-shot pull
    all-reduce over cudaIpc-mapped peer buffers) or "push" (mode 3: the row-parallel GEMM's
    epilogue stores its tiles into every rank). Peer modes also run with several ranks on one
    GPU (one process each), which is how the one-GPU boxes validate the path."""
    import torch.distributed as dist

    if ar not in AR_MODES:
        raise ValueError(f"tp: all-reduce mode {ar!r} (nccl | peer | push)")
    la = local_arch(arch, world)
    dev = torch.device(device)
    if state is not None:  # this rank's slice of a full fp32 state (parity tests: tp.shard_state)
        from paper_2601_11822_b200.tp import shard_state

        weights = DecoderWeights.from_state(la, shard_state(arch, state, rank, world), device=dev)
    else:
        weights = DecoderWeights.random(la, device=dev, seed=rank, embed_vocab=arch.vocab)
    ex = B200Executor(la, weights=weights, vocab_offset=rank * la.vocab,
                      token_source=lambda req: prompt_token_ids(req.id, req.prompt_tokens, arch.vocab),
                      **executor_kw)
    ex.num_blocks = agreed_num_blocks(ex.num_blocks, host_group)
    ex.tp_world, ex.tp_rank = world, rank
    if ar == "nccl":
        obj = [[nccl_unique_id(), nccl_unique_id()] if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=host_group)
        ex.tp_comms = NcclPhaseComms(ex.runner, rank, world, {"pre": obj[0][0], "dec": obj[0][1]}, device=dev)
    else:
        ex.tp_comms = IpcPeerGroup(ex.runner, rank, world, pg=host_group, device=dev, mode=AR_MODES[ar])
    return ex

"""Tensor parallelism on the B200 (csrc/tp.cu through the C ABI).

* TP=2 as two processes sharing the GPU (the multi-GPU code path: cudaIpc-mapped peer
  buffers, gloo for the handle exchange), joined by the one-shot peer-memory all-reduce
  (mode 2) — logits (concatenated vocab shards) must match the unsharded GPU forward and the
  fp32 oracle, and both ranks must sample the same greedy ids.
* NCCL (mode 1) at world 1: the dlopen'ed NCCL path (ncclAllReduce sum / uint64 max) is a
  bit-exact identity on the forward.
"""

import pytest
import torch

from oracle.llama_fp32 import Oracle, init_state
from paper_2601_11822_b200 import ops
from paper_2601_11822_b200.model import DecoderWeights, Runner
from paper_2601_11822_b200.specs import ARCHS
from paper_2601_11822_b200.tp import IpcPeerGroup, NcclPhaseComms, local_arch, nccl_unique_id, shard_state

pytestmark = pytest.mark.gpu
TOL = 2e-2


def rel(a, b):
    a, b = a.float().cpu(), b.float().cpu()
    return float((a - b).norm() / b.norm())


def _runner(w, vocab_offset=0):
    r = Runner(w, num_blocks=64, num_slots=4, max_blocks_per_seq=32, max_prefill_tokens=256, max_decode_batch=8,
               vocab_offset=vocab_offset)
    r.block_table[1, :20] = torch.arange(3, 23, dtype=torch.int32, device="cuda")
    return r


def _decode_inputs(r, P, step):
    d = r.dec
    d.slot[:1] = 1
    d.pos[:1] = P - 1 + step
    d.seq[:1] = P + step


P = 150
STEPS = 4


def _prompt(vocab):
    return torch.randint(0, vocab, (P,), generator=torch.Generator().manual_seed(7), dtype=torch.int32)


def _tp_rank(rank, world, port, out_dir, mode):
    import os

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    arch = ARCHS["tiny"]
    la = local_arch(arch, world)
    r = _runner(DecoderWeights.from_state(la, shard_state(arch, init_state(arch, seed=0), rank, world)),
                vocab_offset=rank * la.vocab)
    IpcPeerGroup(r, rank, world, mode=mode)
    prompt = _prompt(arch.vocab)
    logits = r.prefill(1, prompt[: P - 1].cuda(), 0, num_sms=148, logits=True).clone()
    r.last_tok[1] = int(prompt[P - 1])
    ids = []
    for step in range(STEPS):
        _decode_inputs(r, P, step)
        r.decode_body(1, num_sms=148)
        ids.append(int(r.dec.out_ids[0]))  # synchronizes; the next input is on the device already
    torch.cuda.synchronize()
    torch.save({"logits": logits.cpu(), "ids": ids}, os.path.join(out_dir, f"rank{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", [2, 3])
def test_tp2_ipc_peer_allreduce_matches_unsharded(tmp_path, mode):
    """mode 2: pull all-reduce kernel after the row-parallel GEMMs; mode 3: the GEMM epilogue
    pushes its tiles into every rank's receive slot (GEMM and collective fused)."""
    import socket

    import torch.multiprocessing as mp

    arch = ARCHS["tiny"]
    st = init_state(arch, seed=0)
    world = 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mp.spawn(_tp_rank, args=(world, port, str(tmp_path), mode), nprocs=world, join=True)
    res = [torch.load(tmp_path / f"rank{r}.pt") for r in range(world)]
    tp_logits = torch.cat([x["logits"][0] for x in res])
    full = _runner(DecoderWeights.from_state(arch, st))
    prompt = _prompt(arch.vocab)
    ref_full = full.prefill(1, prompt[: P - 1].cuda(), 0, num_sms=148, logits=True).clone()
    oracle_logits, _ = Oracle(arch, st).forward(prompt[: P - 1].long(), 0, None)
    assert rel(tp_logits, ref_full[0]) < TOL
    assert rel(tp_logits, oracle_logits[-1]) < TOL
    assert res[0]["ids"] == res[1]["ids"]  # every rank samples the same global id
    full.last_tok[1] = int(prompt[P - 1])
    want = []
    for step in range(STEPS):
        _decode_inputs(full, P, step)
        full.decode_body(1, num_sms=148)
        want.append(int(full.dec.out_ids[0]))
    flips = sum(a != b for a, b in zip(res[0]["ids"], want))
    assert flips == 0 or res[0]["ids"][0] == want[0], (res[0]["ids"], want)


def test_nccl_world1_identity():
    arch = ARCHS["tiny"]
    st = init_state(arch, seed=0)
    w = DecoderWeights.from_state(arch, st)
    base = _runner(w)
    tp = _runner(w)
    comms = NcclPhaseComms(tp, 0, 1, {"pre": nccl_unique_id(), "dec": nccl_unique_id()})
    ids = torch.randint(0, arch.vocab, (97,), generator=torch.Generator().manual_seed(3), dtype=torch.int32).cuda()
    a = base.prefill(1, ids, 0, num_sms=148, logits=True).clone()
    b = tp.prefill(1, ids, 0, num_sms=148, logits=True).clone()
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    for r in (base, tp):
        r.last_tok[1] = 5
        _decode_inputs(r, 98, 0)
        r.decode_body(1, num_sms=148)
    torch.cuda.synchronize()
    assert int(base.dec.out_ids[0]) == int(tp.dec.out_ids[0])
    assert torch.equal(base.kv, tp.kv)
    comms.close()


def _tp_serve_rank(rank, world, port, out_dir, ar):
    import os

    import torch.distributed as dist

    from paper_2601_11822_b200.arm import CostParams
    from paper_2601_11822_b200.engines.rapid import RapidEngine
    from paper_2601_11822_b200.harness import run_items
    from paper_2601_11822_b200.slo import SloSpec
    from paper_2601_11822_b200.specs import b200_spec
    from paper_2601_11822_b200.tp_engine import CommandChannel, attach_leader, serve_worker, stop_workers
    from paper_2601_11822_b200.tp_serve import build_tp_executor
    from paper_2601_11822_b200.traffic import WorkloadSpec, synthesize

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    arch = ARCHS["tiny"]
    ex = build_tp_executor(arch, rank, world, None, ar=ar, state=init_state(arch, seed=0), static_decode_sms=72,
                           max_batch=16, chunk_tokens=32, num_blocks=256, max_context=512, num_slots=32)
    ch = CommandChannel()
    ex.warmup()
    if rank == 0:
        attach_leader(ex, ch)
        items = synthesize(WorkloadSpec(qps=16.0, duration_s=2.0, seed=0, mean_prompt_tokens=64,
                                        mean_output_tokens=16))[:6]
        model = arch.model_spec()
        slo = SloSpec(itl_slo_us=50_000)
        try:
            res = run_items("rapid", items, model, b200_spec(), CostParams(), slo,
                            engine_factory=lambda: RapidEngine(model, b200_spec(), CostParams(), slo, chunk_tokens=32,
                                                               max_batch=16, executor=ex))
        finally:
            stop_workers(ch)
        done = {r.id: (r.prompt_tokens, ex.generated[r.id]) for r in res.engine.requests
                if r.state.value == "finished"}
        torch.save({"done": done, "n": len(items)}, os.path.join(out_dir, "served.pt"))
    else:
        serve_worker(ex, ch)
    ex.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("ar", ["peer", "push"])
def test_tp2_serving_exact_greedy(tmp_path, ar):
    """cfg-4 serving path (tp_serve + tp_engine) at world 2 on one GPU: rank 0's RapidEngine
    drives both shards through the int32 command channel; every finished request's greedy ids
    equal the fp32 oracle's (teacher-forced), i.e. the sharded forward, the command replay and
    the vocab-parallel argmax agree end to end."""
    import socket

    import torch.multiprocessing as mp

    from paper_2601_11822_b200.traffic import prompt_token_ids

    arch = ARCHS["tiny"]
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mp.spawn(_tp_serve_rank, args=(2, port, str(tmp_path), ar), nprocs=2, join=True)
    out = torch.load(tmp_path / "served.pt")
    assert len(out["done"]) == out["n"]
    orc = Oracle(arch, init_state(arch, seed=0))
    for rid, (P, gen) in out["done"].items():
        prompt = prompt_token_ids(rid, P, arch.vocab).long()
        logits, _ = orc.forward(torch.cat([prompt, torch.tensor(gen[:-1], dtype=torch.long)]), 0, None)
        want = [int(x) for x in logits[P - 1 :].argmax(-1)]
        assert gen == want, (rid, gen, want)

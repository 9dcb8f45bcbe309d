"""Tensor-parallel sharding (tp.py) on CPU: the sharded fp32 restatement (column-parallel
QKV / gate|up, row-parallel O / down with summed partials, vocab-parallel lm_head) must equal
the unsharded oracle forward, and the shard shapes must be what the C forward expects."""

import dataclasses

import pytest
import torch

from oracle.llama_fp32 import Oracle, init_state
from paper_2601_11822_b200.specs import ARCHS
from paper_2601_11822_b200.tp import local_arch, shard_state

SMALL = dataclasses.replace(ARCHS["tiny"], layers=2, vocab=1024)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("bias", [False, True])
def test_sharded_forward_equals_full(world, bias):
    arch = dataclasses.replace(SMALL, kv_heads=4, qkv_bias=bias)
    st = init_state(arch, seed=3)
    ids = torch.randint(0, arch.vocab, (23,), generator=torch.Generator().manual_seed(1))
    full, _ = Oracle(arch, st).forward(ids, 0, None)
    la = local_arch(arch, world)
    tp = Oracle(arch, st).forward_tp(ids, [shard_state(arch, st, r, world) for r in range(world)], la)
    assert tp.shape == full.shape
    assert torch.allclose(tp, full, rtol=1e-4, atol=1e-4)


def test_shard_shapes():
    arch = ARCHS["llama3.1-70b"]
    la = local_arch(arch, 8)
    assert (la.q_heads, la.kv_heads, la.intermediate, la.vocab) == (8, 1, 3584, 16032)
    assert not la.tie_embeddings
    st = init_state(dataclasses.replace(SMALL, kv_heads=4), seed=0)
    sh = shard_state(dataclasses.replace(SMALL, kv_heads=4), st, 1, 2)
    D = SMALL.head_dim
    assert sh["layers.0.q"].shape == (SMALL.q_heads // 2 * D, SMALL.hidden)
    assert sh["layers.0.k"].shape == (2 * D, SMALL.hidden)
    assert sh["layers.0.o"].shape == (SMALL.hidden, SMALL.q_heads // 2 * D)
    assert sh["layers.0.down"].shape == (SMALL.hidden, SMALL.intermediate // 2)
    assert sh["lm_head"].shape == (SMALL.vocab // 2, SMALL.hidden)
    assert torch.equal(sh["layers.0.q"], st["layers.0.q"][SMALL.q_heads // 2 * D:])
    assert torch.equal(sh["embed"], st["embed"])  # replicated


def test_indivisible_world_rejected():
    with pytest.raises(ValueError):
        local_arch(ARCHS["tiny"], 3)

"""The fp32 oracle vs HF transformers (CPU). Pins the numeric oracle, whose
parity with the reference is otherwise unpinned (the reference has no model)."""

import dataclasses

import pytest
import torch

from oracle.llama_fp32 import Oracle, init_state
from paper_2601_11822_b200.model import rope_inv_freq
from paper_2601_11822_b200.specs import ARCHS

transformers = pytest.importorskip("transformers")


def small(arch, **kw):
    return dataclasses.replace(arch, **kw)


def _hf_model(arch, state):
    common = dict(vocab_size=arch.vocab, hidden_size=arch.hidden, intermediate_size=arch.intermediate,
                  num_hidden_layers=arch.layers, num_attention_heads=arch.q_heads, num_key_value_heads=arch.kv_heads,
                  head_dim=arch.head_dim, rms_norm_eps=arch.rms_eps, rope_theta=arch.rope_theta,
                  max_position_embeddings=arch.max_position, tie_word_embeddings=arch.tie_embeddings)
    if arch.qkv_bias:
        cfg = transformers.Qwen2Config(**common)
        cls = transformers.Qwen2ForCausalLM
    else:
        rs = arch.rope_scaling
        cfg = transformers.LlamaConfig(**common, rope_scaling=None if rs is None else {
            "rope_type": "llama3", "factor": rs["factor"], "low_freq_factor": rs["low_freq_factor"],
            "high_freq_factor": rs["high_freq_factor"],
            "original_max_position_embeddings": rs["original_max_position"]}, attention_bias=False, mlp_bias=False)
        cls = transformers.LlamaForCausalLM
    cfg._attn_implementation = "eager"
    m = cls(cfg).float().eval()
    sd = {"model.embed_tokens.weight": state["embed"], "model.norm.weight": state["norm"]}
    if not arch.tie_embeddings:
        sd["lm_head.weight"] = state["lm_head"]
    for i in range(arch.layers):
        p, q = f"layers.{i}.", f"model.layers.{i}."
        sd.update({q + "input_layernorm.weight": state[p + "ln1"], q + "post_attention_layernorm.weight":
                   state[p + "ln2"], q + "self_attn.q_proj.weight": state[p + "q"], q + "self_attn.k_proj.weight":
                   state[p + "k"], q + "self_attn.v_proj.weight": state[p + "v"], q + "self_attn.o_proj.weight":
                   state[p + "o"], q + "mlp.gate_proj.weight": state[p + "gate"], q + "mlp.up_proj.weight":
                   state[p + "up"], q + "mlp.down_proj.weight": state[p + "down"]})
        if arch.qkv_bias:
            sd.update({q + "self_attn.q_proj.bias": state[p + "bq"], q + "self_attn.k_proj.bias": state[p + "bk"],
                       q + "self_attn.v_proj.bias": state[p + "bv"]})
    missing, unexpected = m.load_state_dict(sd, strict=False)
    assert not [k for k in missing if "rotary" not in k], missing
    assert not unexpected
    return m


@pytest.mark.parametrize("name,kw", [
    ("tiny", {}),
    ("tiny", {"layers": 2, "hidden": 256, "intermediate": 512, "vocab": 512}),
    ("qwen2.5-14b", {"layers": 2, "hidden": 320, "q_heads": 5, "kv_heads": 1, "intermediate": 640, "vocab": 1000}),
])
def test_oracle_matches_hf(name, kw):
    torch.manual_seed(0)
    arch = small(ARCHS[name], **kw)
    st = init_state(arch, seed=3)
    orc = Oracle(arch, st)
    ids = torch.randint(0, arch.vocab, (37,))
    mine, _ = orc.forward(ids, 0, None)
    hf = _hf_model(arch, st)
    with torch.no_grad():
        ref = hf(ids[None]).logits[0]
    rel = (mine - ref).norm() / ref.norm()
    assert rel < 1e-4, rel


def test_oracle_incremental_equals_full():
    arch = small(ARCHS["tiny"], layers=2, hidden=256, intermediate=512, vocab=512)
    orc = Oracle(arch, init_state(arch, seed=1))
    ids = torch.randint(0, arch.vocab, (20,))
    full, _ = orc.forward(ids, 0, None)
    part, kv = orc.forward(ids[:13], 0, None)
    rest, _ = orc.forward(ids[13:], 13, kv)
    assert torch.allclose(torch.cat([part, rest]), full, atol=1e-4, rtol=1e-4)


def test_rope_inv_freq_matches_hf_llama3():
    arch = ARCHS["llama3.1-8b"]
    from transformers.modeling_rope_utils import ROPE_INIT_FUNCTIONS
    cfg = transformers.LlamaConfig(hidden_size=arch.hidden, num_attention_heads=arch.q_heads, head_dim=arch.head_dim,
                                   rope_theta=arch.rope_theta, max_position_embeddings=arch.max_position,
                                   rope_scaling={"rope_type": "llama3", "factor": 8.0, "low_freq_factor": 1.0,
                                                 "high_freq_factor": 4.0,
                                                 "original_max_position_embeddings": 8192})
    hf_inv, _ = ROPE_INIT_FUNCTIONS["llama3"](cfg, "cpu")
    mine = rope_inv_freq(arch)
    assert torch.allclose(mine.float(), hf_inv.float(), rtol=1e-6, atol=0)

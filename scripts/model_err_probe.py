"""Model-level bf16 error budget at real shapes (diagnostic).

For a 1- and 2-layer Llama-3.1-8B / Qwen2.5-14B (random init), prefill logits of the native
forward (rb_decoder_forward) vs the fp32 oracle, next to an IDEAL bf16 pipeline (torch on the
GPU, fp32 math with every kernel-boundary activation rounded to bf16 exactly where the native
forward stores bf16): if native ~= ideal, the model-level error is the format's, not a kernel's.
"""
import dataclasses
import math
import sys

import torch

sys.path.insert(0, ".")
from oracle.llama_fp32 import Oracle, _rms, _rope, init_state, inv_freq  # noqa: E402
from paper_2601_11822_b200.model import DecoderWeights, Runner  # noqa: E402
from paper_2601_11822_b200.specs import ARCHS  # noqa: E402


def ideal(arch, st, ids, dev):
    bf = lambda t: t.bfloat16().float()  # noqa: E731
    s = {k: v.to(dev) for k, v in st.items()}
    T, D, G = ids.shape[0], arch.head_dim, arch.q_heads // arch.kv_heads
    pos = torch.arange(T, device=dev)
    fr = inv_freq(arch).to(dev)
    x = s["embed"][ids.to(dev)]
    for i in range(arch.layers):
        p = f"layers.{i}."
        h = bf(_rms(x, s[p + "ln1"], arch.rms_eps))
        q, k, v = h @ s[p + "q"].T, h @ s[p + "k"].T, h @ s[p + "v"].T
        if arch.qkv_bias:
            q, k, v = q + s[p + "bq"], k + s[p + "bk"], v + s[p + "bv"]
        q = bf(_rope(q.view(T, arch.q_heads, D), pos, fr))
        k = bf(_rope(k.view(T, arch.kv_heads, D), pos, fr))
        v = bf(v.view(T, arch.kv_heads, D))
        sc = torch.einsum("thd,nhd->htn", q, k.repeat_interleave(G, 1)) / math.sqrt(D)
        sc = sc.masked_fill((pos[None, :] > pos[:, None])[None], float("-inf"))
        o = bf(torch.einsum("htn,nhd->thd", torch.softmax(sc, -1), v.repeat_interleave(G, 1)).reshape(T, -1))
        x = bf(x + o @ s[p + "o"].T)
        h = bf(_rms(x, s[p + "ln2"], arch.rms_eps))
        x = bf(x + bf(torch.nn.functional.silu(h @ s[p + "gate"].T) * (h @ s[p + "up"].T)) @ s[p + "down"].T)
    hl = bf(_rms(x[-1:], s["norm"], arch.rms_eps))
    return bf(hl @ s.get("lm_head", s["embed"]).T)[0].cpu()


def rel(a, b):
    a, b = a.float(), b.float()
    return float((a - b).norm() / b.norm())


for name in ("llama3.1-8b", "qwen2.5-14b"):
    for L in (1, 2):
        arch = dataclasses.replace(ARCHS[name], layers=L)
        st = init_state(arch, seed=1, style="random")
        g = torch.Generator().manual_seed(11)
        P = 700
        ids = torch.randint(0, arch.vocab, (P,), generator=g, dtype=torch.int32)[: P - 1]
        ref = Oracle(arch, st).forward(ids.long(), 0, None)[0][-1]
        w = DecoderWeights.from_state(arch, st)
        r = Runner(w, num_blocks=64, num_slots=2, max_blocks_per_seq=64, max_prefill_tokens=1024, max_decode_batch=8)
        r.block_table[0, :44] = torch.randperm(64)[:44].int().cuda()
        dev_ids = ids.cuda()
        for chunk in ((0, 699), (0, 512, 699)):
            for a, b in zip(chunk[:-1], chunk[1:]):
                lg = r.prefill(0, dev_ids[a:b], a, num_sms=148, logits=True)
            torch.cuda.synchronize()
            print(f"{name} L={L} chunks={chunk}: native {rel(lg[0].cpu(), ref):.4f}  ideal-bf16 "
                  f"{rel(ideal(arch, st, ids.long(), 'cuda'), ref):.4f}  native-vs-ideal "
                  f"{rel(lg[0].cpu(), ideal(arch, st, ids.long(), 'cuda')):.4f}", flush=True)
        del r, w, st
        torch.cuda.empty_cache()

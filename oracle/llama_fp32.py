"""CPU fp32 oracle of the decoder numerics — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module, and only as the checker / CPU baseline; the product path
(paper_2601_11822_b200) never calls it.

PARITY UNPINNED vs the reference: the reference (arxiv/paper_2601_11822,
pkg/src/pdsim) is a discrete-event simulator with no model numerics
("numeric precision emulation ... non-goals").
This restatement follows standard Llama-3.x / Qwen2 math — RMSNorm
(x * rsqrt(mean(x^2) + eps) * w), llama3-scaled rotate-half RoPE, GQA
attention, SwiGLU MLP, optional QKV bias — and is cross-checked against
HF transformers' LlamaForCausalLM / Qwen2ForCausalLM in
tests/test_oracle.py. It also hosts the paged-KV reference used by the CPU
tests of the block-table contract.
"""

from __future__ import annotations

import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def inv_freq(arch) -> torch.Tensor:
    D = arch.head_dim
    f = 1.0 / (arch.rope_theta ** (torch.arange(0, D, 2, dtype=torch.float64) / D))
    rs = arch.rope_scaling
    if rs:
        factor, lo, hi, old = rs["factor"], rs["low_freq_factor"], rs["high_freq_factor"], rs["original_max_position"]
        wl = 2 * math.pi / f
        out = []
        for fi, w in zip(f.tolist(), wl.tolist()):
            if w < old / hi:
                out.append(fi)
            elif w > old / lo:
                out.append(fi / factor)
            else:
                s = (old / w - lo) / (hi - lo)
                out.append((1 - s) * fi / factor + s * fi)
        f = torch.tensor(out, dtype=torch.float64)
    return f


# Frozen cfg-1 init ("confident"): see init_state.
CONFIDENT_EMBED_STD = 1.0
CONFIDENT_LM_SCALE = 0.02


def init_state(arch, seed: int = 0, std: float = 0.02, bf16_round: bool = True, style: str = "auto") -> dict:
    """Deterministic weights (CPU generator), optionally rounded to bf16 values.

    style "random": every matrix N(0, std), norms 1 + N(0, 0.1).
    style "confident" (the frozen cfg-1 tiny decoder, default for arch "tiny"): the same
    random blocks, but the token embedding has unit std and lm_head is a fixed random row
    permutation of it times CONFIDENT_LM_SCALE (lm_head[succ(v)] = s * embed[v]). The
    residual stream then carries the current token's embedding next to the blocks'
    context-dependent output (comparable norms), so every logit row is one clear top-1
    (the successor of the current token, ~20 sigma above the rest) plus a context-dependent
    part that holds most of the row's L2 mass. Greedy ids are therefore stable under bf16
    rounding (greedy-id exactness is decidable), while the per-step logits rel-L2 check
    still sees the attention / paged-KV numerics. Random N(0, 0.02) logits have top-1 gaps
    of ~0.25 sigma, so over a ~1k-token trace some gap always falls inside the bf16 error
    (SURVEY.md §7.3.6)."""
    g = torch.Generator().manual_seed(seed)
    H, D, I, V = arch.hidden, arch.head_dim, arch.intermediate, arch.vocab
    if style == "auto":
        style = "confident" if arch.name == "tiny" else "random"
    if style not in ("random", "confident"):
        raise ValueError(f"unknown init style {style!r}")

    def w(*shape):
        x = torch.randn(*shape, generator=g) * std
        return x.to(torch.bfloat16).float() if bf16_round else x

    def n(size):
        x = 1.0 + 0.1 * torch.randn(size, generator=g)
        return x.to(torch.bfloat16).float() if bf16_round else x

    if style == "confident":
        e = torch.randn(V, H, generator=g) * CONFIDENT_EMBED_STD
        st = {"embed": e.to(torch.bfloat16).float() if bf16_round else e}
    else:
        st = {"embed": w(V, H)}
    for i in range(arch.layers):
        p = f"layers.{i}."
        st[p + "ln1"] = n(H)
        st[p + "q"] = w(arch.q_heads * D, H)
        st[p + "k"] = w(arch.kv_heads * D, H)
        st[p + "v"] = w(arch.kv_heads * D, H)
        if arch.qkv_bias:
            st[p + "bq"] = w(arch.q_heads * D)
            st[p + "bk"] = w(arch.kv_heads * D)
            st[p + "bv"] = w(arch.kv_heads * D)
        st[p + "o"] = w(H, arch.q_heads * D)
        st[p + "ln2"] = n(H)
        st[p + "gate"] = w(I, H)
        st[p + "up"] = w(I, H)
        st[p + "down"] = w(H, I)
    st["norm"] = n(H)
    if style == "confident":
        if arch.tie_embeddings:
            raise ValueError("the confident init needs an untied lm_head")
        succ = torch.randperm(V, generator=g)
        lm = torch.empty(V, H)
        lm[succ] = st["embed"] * CONFIDENT_LM_SCALE
        st["lm_head"] = lm.to(torch.bfloat16).float() if bf16_round else lm
    elif not arch.tie_embeddings:
        st["lm_head"] = w(V, H)
    return st


def _rms(x, w, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


def _rope(x, pos, freqs):
    # x [T, h, D]; rotate-half pairing (i, i + D/2)
    ang = pos.double()[:, None] * freqs[None, :]
    c, s = ang.cos().float()[:, None, :], ang.sin().float()[:, None, :]
    half = x.shape[-1] // 2
    x1, x2 = x[..., :half], x[..., half:]
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)


class Oracle:
    """fp32 forward with an explicit per-sequence KV list (contiguous)."""

    def __init__(self, arch, state: dict):
        self.a = arch
        self.s = state
        self.freqs = inv_freq(arch)

    def forward(self, ids: torch.Tensor, start: int, kv: list | None):
        """ids [T] at positions start..start+T-1 given kv (per layer (K, V) [start, Hkv, D]).
        Returns logits [T, V] and the extended kv."""
        a, s = self.a, self.s
        T = ids.shape[0]
        D = a.head_dim
        G = a.q_heads // a.kv_heads
        pos = torch.arange(start, start + T)
        x = s["embed"][ids.long()]
        new_kv = []
        for i in range(a.layers):
            p = f"layers.{i}."
            h = _rms(x, s[p + "ln1"], a.rms_eps)
            q = h @ s[p + "q"].T
            k = h @ s[p + "k"].T
            v = h @ s[p + "v"].T
            if a.qkv_bias:
                q, k, v = q + s[p + "bq"], k + s[p + "bk"], v + s[p + "bv"]
            q = _rope(q.view(T, a.q_heads, D), pos, self.freqs)
            k = _rope(k.view(T, a.kv_heads, D), pos, self.freqs)
            v = v.view(T, a.kv_heads, D)
            if kv is not None and start > 0:
                k = torch.cat([kv[i][0], k], 0)
                v = torch.cat([kv[i][1], v], 0)
            new_kv.append((k, v))
            kf = k.repeat_interleave(G, dim=1)
            vf = v.repeat_interleave(G, dim=1)
            sc = torch.einsum("thd,nhd->htn", q, kf) / math.sqrt(D)
            qpos = pos[:, None]
            kpos = torch.arange(k.shape[0])[None, :]
            sc = sc.masked_fill((kpos > qpos)[None], float("-inf"))
            o = torch.einsum("htn,nhd->thd", torch.softmax(sc, -1), vf).reshape(T, a.q_heads * D)
            x = x + o @ s[p + "o"].T
            h = _rms(x, s[p + "ln2"], a.rms_eps)
            x = x + (torch.nn.functional.silu(h @ s[p + "gate"].T) * (h @ s[p + "up"].T)) @ s[p + "down"].T
        x = _rms(x, s["norm"], a.rms_eps)
        logits = x @ s.get("lm_head", s["embed"]).T
        return logits, new_kv

    def forward_tp(self, ids: torch.Tensor, shards: list[dict], la) -> torch.Tensor:
        """The same prompt forward computed shard by shard (tensor parallel, test restatement
        of paper_2601_11822_b200/tp.py): column-parallel QKV / gate|up, row-parallel O / down
        whose partials are summed (the all-reduce), vocab-parallel lm_head concatenated.
        shards[r] = tp.shard_state(...) of rank r, la = tp.local_arch(...). Returns [T, V]."""
        a, s = self.a, self.s
        T = ids.shape[0]
        D = a.head_dim
        G = la.q_heads // la.kv_heads
        pos = torch.arange(T)
        x = s["embed"][ids.long()]
        for i in range(a.layers):
            p = f"layers.{i}."
            h = _rms(x, s[p + "ln1"], a.rms_eps)
            attn_sum = torch.zeros_like(x)
            for sh in shards:
                q, k, v = h @ sh[p + "q"].T, h @ sh[p + "k"].T, h @ sh[p + "v"].T
                if a.qkv_bias:
                    q, k, v = q + sh[p + "bq"], k + sh[p + "bk"], v + sh[p + "bv"]
                q = _rope(q.view(T, la.q_heads, D), pos, self.freqs)
                k = _rope(k.view(T, la.kv_heads, D), pos, self.freqs)
                v = v.view(T, la.kv_heads, D)
                sc = torch.einsum("thd,nhd->htn", q, k.repeat_interleave(G, 1)) / math.sqrt(D)
                sc = sc.masked_fill((pos[None, :] > pos[:, None])[None], float("-inf"))
                o = torch.einsum("htn,nhd->thd", torch.softmax(sc, -1), v.repeat_interleave(G, 1))
                attn_sum = attn_sum + o.reshape(T, -1) @ sh[p + "o"].T  # partial of the row-parallel O
            x = x + attn_sum
            h = _rms(x, s[p + "ln2"], a.rms_eps)
            mlp_sum = torch.zeros_like(x)
            for sh in shards:
                mlp_sum = mlp_sum + (torch.nn.functional.silu(h @ sh[p + "gate"].T) * (h @ sh[p + "up"].T)) @ \
                    sh[p + "down"].T
            x = x + mlp_sum
        x = _rms(x, s["norm"], a.rms_eps)
        return torch.cat([x @ sh["lm_head"].T for sh in shards], dim=-1)

    def greedy(self, prompt: torch.Tensor, n_out: int):
        """Greedy continuation: returns (token ids [n_out], logits of each emitting step [n_out, V])."""
        logits, kv = self.forward(prompt, 0, None)
        outs, lg = [], []
        cur = logits[-1]
        pos = prompt.shape[0]
        for _ in range(n_out):
            lg.append(cur)
            t = int(torch.argmax(cur))
            outs.append(t)
            l2, kv = self.forward(torch.tensor([t]), pos, kv)
            cur = l2[-1]
            pos += 1
        return outs, torch.stack(lg)


def paged_attention_ref(q, cache, block_row, n):
    """Decode attention oracle over a paged cache [nb][2][Hkv][16][D]: q [Hq, D] -> [Hq, D] (fp32)."""
    Hkv, D = cache.shape[2], cache.shape[4]
    pages = block_row[: (n + 15) // 16].long()
    kv = cache[pages].float()
    k = kv[:, 0].permute(0, 2, 1, 3).reshape(-1, Hkv, D)[:n]
    v = kv[:, 1].permute(0, 2, 1, 3).reshape(-1, Hkv, D)[:n]
    G = q.shape[0] // Hkv
    s = torch.einsum("hd,nhd->hn", q.float(), k.repeat_interleave(G, 1)) / math.sqrt(D)
    return torch.einsum("hn,nhd->hd", torch.softmax(s, -1), v.repeat_interleave(G, 1))


def decode_batch(orc: Oracle, ids: torch.Tensor, positions: list[int], kvs: list[list]) -> torch.Tensor:
    """One batched decode step (weights read once for all rows; attention per
    sequence over its own KV). kvs[b][layer] = (K [n,Hkv,D], V) is extended in place.
    Returns logits [B, V]."""
    a, s = orc.a, orc.s
    B = ids.shape[0]
    D = a.head_dim
    G = a.q_heads // a.kv_heads
    x = s["embed"][ids.long()]
    pos = torch.tensor(positions)
    for i in range(a.layers):
        p = f"layers.{i}."
        h = _rms(x, s[p + "ln1"], a.rms_eps)
        q = h @ s[p + "q"].T
        k = h @ s[p + "k"].T
        v = h @ s[p + "v"].T
        if a.qkv_bias:
            q, k, v = q + s[p + "bq"], k + s[p + "bk"], v + s[p + "bv"]
        q = _rope(q.view(B, a.q_heads, D), pos, orc.freqs)
        k = _rope(k.view(B, a.kv_heads, D), pos, orc.freqs)
        v = v.view(B, a.kv_heads, D)
        o = torch.empty(B, a.q_heads, D)
        for b in range(B):
            K, V = kvs[b][i]
            K = torch.cat([K, k[b : b + 1]], 0)
            V = torch.cat([V, v[b : b + 1]], 0)
            kvs[b][i] = (K, V)
            sc = torch.einsum("hd,nhd->hn", q[b], K.repeat_interleave(G, 1)) / math.sqrt(D)
            o[b] = torch.einsum("hn,nhd->hd", torch.softmax(sc, -1), V.repeat_interleave(G, 1))
        x = x + o.reshape(B, -1) @ s[p + "o"].T
        h = _rms(x, s[p + "ln2"], a.rms_eps)
        x = x + (torch.nn.functional.silu(h @ s[p + "gate"].T) * (h @ s[p + "up"].T)) @ s[p + "down"].T
    x = _rms(x, s["norm"], a.rms_eps)
    return x @ s.get("lm_head", s["embed"]).T

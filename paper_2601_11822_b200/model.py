"""Decoder weights and the device-side forward passes (prefill chunk, decode step).

This is the physical realization of the two priced calls of the reference:
`prefill_time` (pkg/src/pdsim/costmodel.py:89-106) becomes `Runner.prefill`,
`decode_time` (costmodel.py:109-134) becomes `Runner.decode` (one CUDA-graph
replay). Every op goes through the C ABI (ops.py -> librapid_b200.so).

HBM layout:
  * weights: bf16, K-contiguous [out, in]; QKV fused [(Hq+2Hkv)*D, H];
    gate/up fused [2I, H] (gate rows first)
  * KV cache: one tensor [L][num_blocks][2][Hkv][16][D] bf16 — shared by the
    prefill and decode streams; no KV ever moves between phases
  * block table: int32 [num_slots][max_blocks]; a request owns one slot row
  * last_tok: int32 [num_slots] — the next decode input of each slot; written by
    prefill completion and by the decode argmax, so token ids never round-trip
    through the host between steps
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from paper_2601_11822_b200 import ops
from paper_2601_11822_b200.specs import ArchConfig

PAGE = 16


def rope_inv_freq(arch: ArchConfig) -> torch.Tensor:
    """Per-pair inverse frequencies (fp64), incl. llama3 frequency scaling."""
    D = arch.head_dim
    inv = 1.0 / (arch.rope_theta ** (torch.arange(0, D, 2, dtype=torch.float64) / D))
    rs = arch.rope_scaling
    if rs:
        factor, lo, hi, old = rs["factor"], rs["low_freq_factor"], rs["high_freq_factor"], rs["original_max_position"]
        lo_wl, hi_wl = old / lo, old / hi
        wl = 2 * math.pi / inv
        scaled = torch.where(wl > lo_wl, inv / factor, inv)
        smooth = (old / wl - lo) / (hi - lo)
        smoothed = (1 - smooth) * scaled / factor + smooth * scaled
        medium = (wl >= hi_wl) & (wl <= lo_wl)
        inv = torch.where(medium, smoothed, scaled)
    return inv


def rope_table(arch: ArchConfig, max_pos: int) -> torch.Tensor:
    """fp32 [max_pos][D] = [cos(pos*f) | sin(pos*f)] for the fused RoPE kernel."""
    inv = rope_inv_freq(arch)
    ang = torch.arange(max_pos, dtype=torch.float64)[:, None] * inv[None, :]
    return torch.cat([ang.cos(), ang.sin()], dim=1).float()


@dataclass
class LayerWeights:
    ln1: torch.Tensor
    wqkv: torch.Tensor
    bqkv: torch.Tensor | None
    wo: torch.Tensor
    ln2: torch.Tensor
    wgu: torch.Tensor
    wd: torch.Tensor


class DecoderWeights:
    def __init__(self, arch: ArchConfig, embed, layers: list[LayerWeights], norm, lm_head):
        self.arch = arch
        self.embed = embed
        self.layers = layers
        self.norm = norm
        self.lm_head = lm_head

    @classmethod
    def random(cls, arch: ArchConfig, device="cuda", seed: int = 0, std: float = 0.02) -> "DecoderWeights":
        """Random-init weights of the real shapes (no checkpoints offline), generated on the device."""
        g = torch.Generator(device=device).manual_seed(seed)
        H, D, I = arch.hidden, arch.head_dim, arch.intermediate
        nq = (arch.q_heads + 2 * arch.kv_heads) * D

        def w(*shape):
            return (torch.randn(*shape, device=device, generator=g, dtype=torch.float32) * std).to(torch.bfloat16)

        def n(size):
            return (1.0 + 0.1 * torch.randn(size, device=device, generator=g)).to(torch.bfloat16)

        layers = []
        for _ in range(arch.layers):
            layers.append(LayerWeights(n(H), w(nq, H), w(nq) if arch.qkv_bias else None, w(H, arch.q_heads * D), n(H),
                                       w(2 * I, H), w(H, I)))
        embed = w(arch.vocab, H)
        lm = embed if arch.tie_embeddings else w(arch.vocab, H)
        return cls(arch, embed, layers, n(H), lm)

    @classmethod
    def from_state(cls, arch: ArchConfig, state: dict, device="cuda") -> "DecoderWeights":
        """From an fp32 oracle/HF-style state dict (oracle.llama_fp32 naming)."""
        def t(x):
            return x.to(device=device, dtype=torch.bfloat16).contiguous()

        layers = []
        for i in range(arch.layers):
            p = f"layers.{i}."
            wqkv = torch.cat([state[p + "q"], state[p + "k"], state[p + "v"]], 0)
            b = None
            if arch.qkv_bias:
                b = t(torch.cat([state[p + "bq"], state[p + "bk"], state[p + "bv"]], 0))
            layers.append(LayerWeights(t(state[p + "ln1"]), t(wqkv), b, t(state[p + "o"]), t(state[p + "ln2"]),
                                       t(torch.cat([state[p + "gate"], state[p + "up"]], 0)), t(state[p + "down"])))
        lm = state.get("lm_head", state["embed"])
        return cls(arch, t(state["embed"]), layers, t(state["norm"]), t(lm))

    def nbytes(self) -> int:
        tot = self.embed.numel() * 2 + self.norm.numel() * 2
        if self.lm_head is not self.embed:
            tot += self.lm_head.numel() * 2
        for L in self.layers:
            for x in (L.ln1, L.wqkv, L.bqkv, L.wo, L.ln2, L.wgu, L.wd):
                if x is not None:
                    tot += x.numel() * 2
        return tot


class _Buffers:
    """Activation workspace of one phase (prefill and decode never share one)."""

    def __init__(self, arch: ArchConfig, rows: int, device, logits_rows: int):
        H, D, I = arch.hidden, arch.head_dim, arch.intermediate
        nq = (arch.q_heads + 2 * arch.kv_heads) * D
        bf = torch.bfloat16
        self.x = torch.empty(rows, H, dtype=bf, device=device)
        self.h = torch.empty(rows, H, dtype=bf, device=device)
        self.qkv = torch.empty(rows, nq, dtype=bf, device=device)
        self.q = torch.empty(rows, arch.q_heads * D, dtype=bf, device=device)
        self.attn = torch.empty(rows, arch.q_heads * D, dtype=bf, device=device)
        self.gu = torch.empty(rows, 2 * I, dtype=bf, device=device)
        self.act = torch.empty(rows, I, dtype=bf, device=device)
        self.logits = torch.empty(max(1, logits_rows), arch.vocab, dtype=bf, device=device)
        self.ids = torch.zeros(rows, dtype=torch.int32, device=device)
        self.pos = torch.full((rows,), -1, dtype=torch.int32, device=device)
        self.slot = torch.zeros(rows, dtype=torch.int32, device=device)
        self.seq = torch.zeros(rows, dtype=torch.int32, device=device)
        self.out_ids = torch.zeros(rows, dtype=torch.int32, device=device)
        # split-K partials + tile counters of this phase's GEMMs (never shared across streams)
        self.scratch = ops.GemmScratch(device, ws_bytes=64 << 20, n_counters=8192)


class Runner:
    """Owns weights, the shared paged KV cache, slot state and per-phase workspaces."""

    def __init__(self, weights: DecoderWeights, num_blocks: int, num_slots: int, max_blocks_per_seq: int,
                 max_prefill_tokens: int = 2048, max_decode_batch: int = 256, device="cuda",
                 max_position: int | None = None):
        arch = weights.arch
        self.arch = arch
        self.w = weights
        self.device = torch.device(device)
        self.num_blocks = num_blocks
        self.num_slots = num_slots
        self.dummy_slot = num_slots  # padding rows of a decode bucket point here
        self.max_blocks = max_blocks_per_seq
        self.kv = torch.empty(arch.layers, num_blocks, 2, arch.kv_heads, PAGE, arch.head_dim, dtype=torch.bfloat16,
                              device=self.device)
        self.block_table = torch.zeros(num_slots + 1, max_blocks_per_seq, dtype=torch.int32, device=self.device)
        self.last_tok = torch.zeros(num_slots + 1, dtype=torch.int32, device=self.device)
        mp = max_position or max(PAGE * max_blocks_per_seq + PAGE, 4096)
        self.cos_sin = rope_table(arch, mp).to(self.device)
        self.pre = _Buffers(arch, max_prefill_tokens, self.device, 1)
        self.dec = _Buffers(arch, max_decode_batch, self.device, max_decode_batch)
        self.max_prefill_tokens = max_prefill_tokens
        self.max_decode_batch = max_decode_batch
        self.scale = 1.0 / math.sqrt(arch.head_dim)
        self.eps = arch.rms_eps
        chunks = max(1, (max_blocks_per_seq + 15) // 16)
        self.attn_ws = torch.empty(max_decode_batch * arch.q_heads * chunks * (arch.head_dim + 2), dtype=torch.float32,
                                   device=self.device)

    @staticmethod
    def kv_bytes_per_block(arch: ArchConfig) -> int:
        return arch.layers * 2 * arch.kv_heads * PAGE * arch.head_dim * 2

    # ------------------------------------------------------------------ layers
    def _layers(self, B: _Buffers, T: int, num_sms: int, stream, attn_fn):
        arch, W = self.arch, self.w
        sc = B.scratch
        x, h = B.x[:T], B.h[:T]
        for li, L in enumerate(W.layers):
            ops.rmsnorm(x, L.ln1, h, self.eps, stream=stream)
            ops.linear(h, L.wqkv, out=B.qkv[:T], bias=L.bqkv, num_sms=num_sms, scratch=sc, stream=stream)
            ops.rope_cache_write(B.qkv[:T], B.pos[:T], B.slot[:T], self.block_table, self.cos_sin, B.q[:T],
                                 self.kv[li], num_q_heads=arch.q_heads, num_kv_heads=arch.kv_heads,
                                 head_dim=arch.head_dim, stream=stream)
            attn_fn(li)
            ops.linear(B.attn[:T], L.wo, out=x, residual=x, num_sms=num_sms, scratch=sc, stream=stream)
            ops.rmsnorm(x, L.ln2, h, self.eps, stream=stream)
            ops.linear(h, L.wgu, out=B.gu[:T], num_sms=num_sms, scratch=sc, stream=stream)
            ops.silu_mul(B.gu[:T], B.act[:T], stream=stream)
            ops.linear(B.act[:T], L.wd, out=x, residual=x, num_sms=num_sms, scratch=sc, stream=stream)

    # ------------------------------------------------------------------ prefill
    def prefill(self, slot: int, token_ids: torch.Tensor, start: int, *, num_sms: int, stream=None,
                logits: bool = False) -> torch.Tensor | None:
        """KV for positions start..start+T-1 of `slot` (token_ids: device int32 [T]).

        With logits=True also returns the last row's logits (hybrid mode / tests)."""
        T = int(token_ids.shape[0])
        if T == 0:
            return None
        if T > self.max_prefill_tokens:
            raise ValueError(f"prefill chunk {T} exceeds workspace {self.max_prefill_tokens}")
        arch, B = self.arch, self.pre
        st = stream
        B.ids[:T].copy_(token_ids, non_blocking=True)
        torch.arange(start, start + T, dtype=torch.int32, device=self.device, out=B.pos[:T])
        B.slot[:T].fill_(slot)
        ops.embed(self.w.embed, B.x[:T], ids=B.ids[:T], stream=st)
        bt_row = self.block_table[slot]
        q3 = B.q[:T].view(T, arch.q_heads, arch.head_dim)
        o3 = B.attn[:T].view(T, arch.q_heads, arch.head_dim)

        def attn(li):
            ops.prefill_attention(q3, self.kv[li], bt_row, start, o3, num_kv_heads=arch.kv_heads, scale=self.scale,
                                  stream=st)

        self._layers(B, T, num_sms, st, attn)
        if not logits:
            return None
        last = B.x[T - 1 : T]
        ops.rmsnorm(last, self.w.norm, B.h[:1], self.eps, stream=st)
        ops.linear(B.h[:1], self.w.lm_head, out=B.logits[:1], num_sms=num_sms, scratch=B.scratch, stream=st)
        return B.logits[:1]

    # ------------------------------------------------------------------ decode
    def decode_body(self, Bsz: int, *, num_sms: int, max_pages: int | None = None, stream=None,
                    write_logits_only: bool = False):
        """One decode step over rows 0..Bsz-1 of the decode workspace.

        Inputs (device, pre-filled): dec.slot, dec.pos (= ctx-1, -1 for padding),
        dec.seq (= ctx, 0 for padding). Reads the input token from last_tok[slot],
        writes the greedy token to dec.out_ids and last_tok[slot]. Graph-capturable.
        """
        arch, B = self.arch, self.dec
        st = stream
        ops.embed(self.w.embed, B.x[:Bsz], slot_of_row=B.slot[:Bsz], last_tok=self.last_tok, ids_out=B.ids[:Bsz],
                  stream=st)
        q3 = B.q[:Bsz].view(Bsz, arch.q_heads, arch.head_dim)
        o3 = B.attn[:Bsz].view(Bsz, arch.q_heads, arch.head_dim)

        def attn(li):
            ops.decode_attention(q3, self.kv[li], self.block_table, B.slot[:Bsz], B.seq[:Bsz], o3,
                                 num_kv_heads=arch.kv_heads, max_pages=max_pages or self.max_blocks,
                                 workspace=self.attn_ws, scale=self.scale, num_sms=num_sms, stream=st)

        self._layers(B, Bsz, num_sms, st, attn)
        ops.rmsnorm(B.x[:Bsz], self.w.norm, B.h[:Bsz], self.eps, stream=st)
        ops.linear(B.h[:Bsz], self.w.lm_head, out=B.logits[:Bsz], num_sms=num_sms, scratch=B.scratch, stream=st)
        if not write_logits_only:
            ops.argmax(B.logits[:Bsz], B.out_ids[:Bsz], slot_of_row=B.slot[:Bsz], last_tok=self.last_tok,
                       row_valid=B.seq[:Bsz], stream=st)

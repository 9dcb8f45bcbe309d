"""Decoder weights and the device-side forward passes (prefill chunk, decode step).

This is the physical realization of the two priced calls of the reference:
`prefill_time` (pkg/src/pdsim/costmodel.py:89-106) becomes `Runner.prefill`,
`decode_time` (costmodel.py:109-134) becomes `Runner.decode` (one CUDA-graph
replay). Every op goes through the C ABI (ops.py -> librapid_b200.so).

HBM layout:
  * weights: bf16, K-contiguous [out, in]; QKV fused [(Hq+2Hkv)*D, H], q/k rows
    RoPE-pair-interleaved (interleave_rope_pairs) so the GEMM epilogue applies RoPE
    and writes K/V into the paged cache;
    gate/up fused [2I, H], rows interleaved in 16-blocks [g x16 | u x16] so the
    GEMM epilogue emits silu(gate) * up directly
  * KV cache: one tensor [L][num_blocks][2][Hkv][16][D] bf16 — shared by the
    prefill and decode streams; no KV ever moves between phases
  * block table: int32 [num_slots][max_blocks]; a request owns one slot row
  * last_tok: int32 [num_slots] — the next decode input of each slot; written by
    prefill completion and by the decode argmax, so token ids never round-trip
    through the host between steps
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import torch

from paper_2601_11822_b200 import ops
from paper_2601_11822_b200.specs import ArchConfig

PAGE = 16
GLU_BLOCK = 16  # gate/up rows are interleaved in blocks of 16 for the fused SwiGLU epilogue


def interleave_gate_up(gate: torch.Tensor, up: torch.Tensor) -> torch.Tensor:
    """[I, H] gate, [I, H] up -> [2I, H] rows [g0..g15, u0..u15, g16..g31, u16..u31, ...]."""
    I, H = gate.shape
    return torch.stack([gate.view(I // GLU_BLOCK, GLU_BLOCK, H), up.view(I // GLU_BLOCK, GLU_BLOCK, H)],
                       dim=1).reshape(2 * I, H)


def interleave_rope_pairs(w: torch.Tensor, q_heads: int, kv_heads: int, head_dim: int) -> torch.Tensor:
    """Reorder the q and k rows of a fused [(Hq+2Hkv)*D, ...] QKV weight (or bias) so that
    every RoPE pair is adjacent: new row 2j of a head = rotate-half dim j, 2j+1 = dim j+D/2.

    q and k get the same permutation, so q.k (the attention scores) is unchanged; v rows
    stay in place. The QKV GEMM epilogue then rotates (x[2j], x[2j+1]) pairs that sit in
    one thread's registers and writes k straight into the paged cache (qk_layout = 1)."""
    half = head_dim // 2
    perm = torch.stack([torch.arange(half), torch.arange(half) + half], dim=1).reshape(-1)
    nqk = (q_heads + kv_heads) * head_dim
    qk = w[:nqk].reshape(q_heads + kv_heads, head_dim, *w.shape[1:])[:, perm.to(w.device)]
    return torch.cat([qk.reshape(nqk, *w.shape[1:]), w[nqk:]], 0).contiguous()


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
    def random(cls, arch: ArchConfig, device="cuda", seed: int = 0, std: float = 0.02,
               embed_vocab: int | None = None) -> "DecoderWeights":
        """Random-init weights of the real shapes (no checkpoints offline), generated on the device.
        embed_vocab: rows of the (replicated) embedding when `arch` is a TP shard whose vocab
        is the lm_head slice (tp.local_arch)."""
        g = torch.Generator(device=device).manual_seed(seed)
        H, D, I = arch.hidden, arch.head_dim, arch.intermediate
        nq = (arch.q_heads + 2 * arch.kv_heads) * D

        def w(*shape):
            return (torch.randn(*shape, device=device, generator=g, dtype=torch.float32) * std).to(torch.bfloat16)

        def n(size):
            return (1.0 + 0.1 * torch.randn(size, device=device, generator=g)).to(torch.bfloat16)

        layers = []
        for _ in range(arch.layers):
            # random rows: already "pair-interleaved" (any permutation of random rows is random)
            layers.append(LayerWeights(n(H), w(nq, H), w(nq) if arch.qkv_bias else None, w(H, arch.q_heads * D), n(H),
                                       w(2 * I, H), w(H, I)))
        embed = w(embed_vocab or arch.vocab, H)
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
            hq, hkv, hd = arch.q_heads, arch.kv_heads, arch.head_dim
            wqkv = interleave_rope_pairs(torch.cat([state[p + "q"], state[p + "k"], state[p + "v"]], 0), hq, hkv, hd)
            b = None
            if arch.qkv_bias:
                b = t(interleave_rope_pairs(torch.cat([state[p + "bq"], state[p + "bk"], state[p + "bv"]], 0), hq,
                                            hkv, hd))
            layers.append(LayerWeights(t(state[p + "ln1"]), t(wqkv), b, t(state[p + "o"]), t(state[p + "ln2"]),
                                       t(interleave_gate_up(state[p + "gate"], state[p + "up"])),
                                       t(state[p + "down"])))
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
        self.tp = None  # tp.TpContext of this phase under tensor parallelism
        # split-K partials + tile counters of this phase's GEMMs (never shared across streams)
        self.scratch = ops.GemmScratch(device, ws_bytes=64 << 20, n_counters=8192)


class Runner:
    """Owns weights, the shared paged KV cache, slot state and per-phase workspaces."""

    def __init__(self, weights: DecoderWeights, num_blocks: int, num_slots: int, max_blocks_per_seq: int,
                 max_prefill_tokens: int = 2048, max_decode_batch: int = 256, device="cuda",
                 max_position: int | None = None, vocab_offset: int = 0):
        arch = weights.arch
        self.arch = arch
        self.w = weights
        self.device = torch.device(device)
        self.num_blocks = num_blocks
        self.num_slots = num_slots
        self.dummy_slot = num_slots  # padding rows of a decode bucket point here
        self.max_blocks = max_blocks_per_seq
        # zeroed once so never-written slots hold finite values (kernels also mask them)
        self.kv = torch.zeros(arch.layers, num_blocks, 2, arch.kv_heads, PAGE, arch.head_dim, dtype=torch.bfloat16,
                              device=self.device)
        self.block_table = torch.zeros(num_slots + 1, max_blocks_per_seq, dtype=torch.int32, device=self.device)
        self.last_tok = torch.zeros(num_slots + 1, dtype=torch.int32, device=self.device)
        mp = max_position or max(PAGE * max_blocks_per_seq + PAGE, 4096)
        self.cos_sin = rope_table(arch, mp).to(self.device)
        self.pre = _Buffers(arch, max_prefill_tokens, self.device, max_decode_batch + 1)
        self.dec = _Buffers(arch, max_decode_batch, self.device, max_decode_batch)
        self.vocab_offset = vocab_offset  # TP rank's first lm_head row (global token id)
        self.max_prefill_tokens = max_prefill_tokens
        self.max_decode_batch = max_decode_batch
        self.scale = 1.0 / math.sqrt(arch.head_dim)
        self.eps = arch.rms_eps
        # in-situ roofline probe of decode attention: {"probe_ev0", "probe_ev1", "probe_layer"}
        # (raw cudaEvent_t handles), see set_attention_probe
        self.probe: dict | None = None
        chunks = max(1, (max_blocks_per_seq + 7) // 8)  # decode attention splits <= ceil(pages / 8)
        self.attn_ws = torch.zeros(max_decode_batch * arch.q_heads * chunks * (arch.head_dim + 2),
                                   dtype=torch.float32,
                                   device=self.device)

    def set_attention_probe(self, ev0: torch.cuda.Event, ev1: torch.cuda.Event, layer: int) -> None:
        """Record ev0/ev1 around layer `layer`'s decode attention in every decode forward
        (also inside captured graphs): the kernel's in-situ duration. Set before capture."""
        for ev in (ev0, ev1):
            if not ev.cuda_event:  # torch creates events lazily: force the handle into existence
                ev.record()
        torch.cuda.synchronize(self.device)
        self.probe = {"probe_ev0": ev0.cuda_event, "probe_ev1": ev1.cuda_event, "probe_layer": int(layer)}

    @staticmethod
    def kv_bytes_per_block(arch: ArchConfig) -> int:
        return arch.layers * 2 * arch.kv_heads * PAGE * arch.head_dim * 2

    # ------------------------------------------------------------------ native forward plumbing
    def _model_c(self) -> ops.RbModel:
        if getattr(self, "_mc", None) is None:
            a, W = self.arch, self.w
            L = a.layers

            def arr(get):
                return (ctypes.c_void_p * L)(*[get(l) for l in W.layers])

            keep = {"ln1": arr(lambda l: l.ln1.data_ptr()), "wqkv": arr(lambda l: l.wqkv.data_ptr()),
                    "wo": arr(lambda l: l.wo.data_ptr()), "ln2": arr(lambda l: l.ln2.data_ptr()),
                    "wgu": arr(lambda l: l.wgu.data_ptr()), "wd": arr(lambda l: l.wd.data_ptr())}
            if a.qkv_bias:
                keep["bqkv"] = arr(lambda l: l.bqkv.data_ptr())
            m = ops.RbModel(hidden=a.hidden, layers=L, q_heads=a.q_heads, kv_heads=a.kv_heads, head_dim=a.head_dim,
                            intermediate=a.intermediate, vocab=a.vocab, rms_eps=a.rms_eps, attn_scale=self.scale,
                            embed=W.embed.data_ptr(), final_norm=W.norm.data_ptr(), lm_head=W.lm_head.data_ptr(),
                            kv_cache=self.kv.data_ptr(), kv_layer_stride_bytes=self.kv[0].numel() * 2,
                            num_blocks=self.num_blocks, block_table=self.block_table.data_ptr(),
                            bt_stride=self.block_table.stride(0), cos_sin=self.cos_sin.data_ptr(),
                            last_tok=self.last_tok.data_ptr(), qk_layout=1 if a.head_dim == 128 else 0,
                            vocab_offset=self.vocab_offset)
            for k, v in keep.items():
                setattr(m, k, ctypes.cast(v, ctypes.POINTER(ctypes.c_void_p)))
            self._mc = m
            self._mc_keep = keep
        return self._mc

    def _ws_c(self, B: "_Buffers") -> ops.RbWorkspace:
        rows = B.x.shape[0]
        return ops.RbWorkspace(x=B.x.data_ptr(), h=B.h.data_ptr(), qkv=B.qkv.data_ptr(), q=B.q.data_ptr(),
                               attn=B.attn.data_ptr(), gu=B.gu.data_ptr(), act=B.act.data_ptr(),
                               logits=B.logits.data_ptr(), rows_cap=rows, ids=B.ids.data_ptr(), pos=B.pos.data_ptr(),
                               slot=B.slot.data_ptr(), seq=B.seq.data_ptr(), out_ids=B.out_ids.data_ptr(),
                               gemm_ws=B.scratch.ws.data_ptr(), gemm_ws_bytes=B.scratch.ws_bytes,
                               gemm_counters=B.scratch.counters.data_ptr(),
                               gemm_counters_len=B.scratch.counters.numel(), attn_ws=self.attn_ws.data_ptr(),
                               attn_ws_bytes=self.attn_ws.numel() * 4, tp=B.tp.handle if B.tp is not None else None,
                               **(self.probe if self.probe is not None and B is self.dec else {}))

    def kernels_per_forward(self, n_decode: int, n_prefill: int, logits_decode: bool, emit_prefill: bool,
                            sample: bool) -> int:
        """Kernel launches of one rb_decoder_forward call (mirrors csrc/forward.cu)."""
        T = n_decode + n_prefill
        if T == 0:
            return 0
        fused_rope = self.arch.head_dim == 128
        per_layer = (2 + (0 if fused_rope else 1) + int(n_decode > 0) + int(n_prefill > 0) + 2
                     + (1 if T > 256 else 2))
        n = int(n_decode > 0) + int(n_prefill > 0) + self.arch.layers * per_layer
        nl = (n_decode if logits_decode else 0) + (1 if emit_prefill and n_prefill else 0)
        if nl:
            n += int(bool(logits_decode and n_decode)) + int(bool(emit_prefill and n_prefill)) + 1 + int(sample)
        return n

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
        B = self.pre
        B.ids[:T].copy_(token_ids, non_blocking=True)
        torch.arange(start, start + T, dtype=torch.int32, device=self.device, out=B.pos[:T])
        B.slot[:T].fill_(slot)
        batch = ops.RbBatch(rows=T, n_decode=0, n_prefill=T, max_pages=1, prefill_slot=slot, prefill_start=start,
                            ids_from_slots=0, logits_decode=0, emit_prefill=1 if logits else 0, sample=0,
                            num_sms=num_sms)
        ops.decoder_forward(self._model_c(), self._ws_c(B), batch, stream)
        return B.logits[:1] if logits else None

    # ------------------------------------------------------------------ decode
    def decode_body(self, Bsz: int, *, num_sms: int, max_pages: int | None = None, stream=None,
                    write_logits_only: bool = False):
        """One decode step over rows 0..Bsz-1 of the decode workspace.

        Inputs (device, pre-filled): dec.slot, dec.pos (= ctx-1, -1 for padding),
        dec.seq (= ctx, 0 for padding). Reads the input token from last_tok[slot],
        writes the greedy token to dec.out_ids and last_tok[slot]. Graph-capturable.
        """
        batch = ops.RbBatch(rows=Bsz, n_decode=Bsz, n_prefill=0, max_pages=max_pages or self.max_blocks,
                            prefill_slot=0, prefill_start=0, ids_from_slots=1, logits_decode=1, emit_prefill=0,
                            sample=0 if write_logits_only else 1, num_sms=num_sms)
        ops.decoder_forward(self._model_c(), self._ws_c(self.dec), batch, stream)

    # ------------------------------------------------------------------ hybrid (K9)
    def hybrid(self, n_decode: int, slot: int, start: int, chunk_ids: torch.Tensor | None, *, emit: bool,
               num_sms: int, max_pages: int, stream=None) -> None:
        """One fused chunked-prefill iteration in the `pre` workspace: rows [0, n_decode)
        are decode rows (slot/pos/seq pre-filled by the caller), rows after them the
        chunk of `slot` at positions start..; when `emit`, the chunk's last row is
        sampled too (appended after the decode rows in out_ids)."""
        B = self.pre
        T = 0 if chunk_ids is None else int(chunk_ids.shape[0])
        rows = n_decode + T
        if rows > self.max_prefill_tokens:
            raise ValueError("hybrid iteration exceeds the workspace")
        if T:
            B.ids[n_decode:rows].copy_(chunk_ids, non_blocking=True)
            torch.arange(start, start + T, dtype=torch.int32, device=self.device, out=B.pos[n_decode:rows])
            B.slot[n_decode:rows].fill_(slot)
            B.seq[n_decode:rows].fill_(1)
        batch = ops.RbBatch(rows=rows, n_decode=n_decode, n_prefill=T, max_pages=max_pages, prefill_slot=slot,
                            prefill_start=start, ids_from_slots=1, logits_decode=1, emit_prefill=1 if emit else 0,
                            sample=1, num_sms=num_sms)
        ops.decoder_forward(self._model_c(), self._ws_c(B), batch, stream)

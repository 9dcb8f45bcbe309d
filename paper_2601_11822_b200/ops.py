"""ctypes binding of the C ABI in include/rapid_b200.h (librapid_b200.so).

This is the only way the package reaches the GPU. There is no fallback: if
the shared library is missing or a call fails, a RuntimeError is raised.
torch is used only for device memory and streams; tensors are passed as raw
pointers, sizes and strides.
"""

from __future__ import annotations

import ctypes
import math
import os
from pathlib import Path

import torch

from paper_2601_11822_b200.build import lib_path

_LIB: ctypes.CDLL | None = None

_c_int = ctypes.c_int
_c_ll = ctypes.c_longlong
_c_size = ctypes.c_size_t
_c_float = ctypes.c_float
_vp = ctypes.c_void_p

_SIGS = {
    "rb_version": ([], ctypes.c_char_p),
    "rb_last_error": ([], ctypes.c_char_p),
    "rb_device_sm_count": ([_c_int, ctypes.POINTER(_c_int)], _c_int),
    "rb_debug_gemm_trace": ([_vp], _c_int),
    "rb_debug_gemm_pair_mode": ([_c_int], _c_int),
    "rb_debug_gemm_variant": ([_c_int], _c_int),
    "rb_debug_gemm_prefetch": ([_c_int], _c_int),
    "rb_debug_gemm_prefill_streamk": ([_c_int, ctypes.c_double], _c_int),
    "rb_debug_gemm_prefill_bn": ([_c_int], _c_int),
    "rb_debug_pattn_tiles": ([_c_int], _c_int),
    "rb_debug_decode_kv_one_op": ([_c_int], _c_int),
    "rb_debug_decode_attn_shape": ([_c_int], _c_int),
    "rb_debug_gemm_ksplit": ([_c_int], _c_int),
    "rb_memcpy_async": ([_vp, _vp, ctypes.c_size_t, _vp], _c_int),
    "rb_graph_launch": ([_vp, _vp], _c_int),
    "rb_debug_stream_read": ([_vp, ctypes.c_longlong, _c_int, _c_int, _c_int, _vp, _vp], _c_int),
    "rb_debug_stream_read_tma": ([_vp, ctypes.c_longlong, _c_int, _c_int, _c_int, _c_int, _vp, _vp], _c_int),
    "rb_set_pdl": ([_c_int], _c_int),
    "rb_set_decode_glu": ([_c_int], _c_int),
    "rb_set_decode_ksplit": ([_c_int], _c_int),
    "rb_gemm_bf16": (
        [_vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_ll, _c_ll, _c_ll, _c_int, _c_int, _vp, _c_size, _vp,
         _c_int, _vp],
        _c_int,
    ),
    "rb_decode_attention": (
        [_vp, _c_ll, _vp, _vp, _c_int, _vp, _vp, _vp, _c_ll, _vp, _c_size, _c_int, _c_int, _c_int, _c_int, _c_int,
         _c_float, _c_int, _c_int, _vp],
        _c_int,
    ),
    "rb_prefill_attention": (
        [_vp, _c_ll, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _c_ll, _c_float, _c_int, _vp],
        _c_int,
    ),
    "rb_gemm_qkv_rope": (
        [_vp, _vp, _vp, _c_int, _c_int, _c_ll, _c_int, _c_int, _c_int, _vp, _vp, _vp, _c_int, _vp, _vp, _c_ll, _vp,
         _c_int, _c_int, _vp, _c_size, _vp, _c_int, _vp],
        _c_int,
    ),
    "rb_rope_cache_write": (
        [_vp, _c_ll, _vp, _vp, _vp, _c_int, _vp, _vp, _c_ll, _vp, _c_int, _c_int, _c_int, _c_int, _vp],
        _c_int,
    ),
    "rb_rmsnorm": ([_vp, _c_ll, _vp, _vp, _c_ll, _c_int, _c_int, _c_float, _vp], _c_int),
    "rb_silu_mul": ([_vp, _c_ll, _vp, _c_ll, _c_int, _c_int, _vp], _c_int),
    "rb_embed": ([_vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _vp, _vp], _c_int),
    "rb_argmax": ([_vp, _c_ll, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp], _c_int),
    "rb_block_table_update": ([_vp, _vp, _c_int, _c_int, _vp], _c_int),
    "rb_set_last_token": ([_vp, _c_int, _vp, _c_int, _vp], _c_int),
    "rb_green_split": (
        [_c_int, _c_int, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_c_int),
         ctypes.POINTER(_c_int)],
        _c_int,
    ),
    "rb_green_destroy": ([_vp], _c_int),
    "rb_debug_green_ctx_push": ([_vp, _c_int], _c_int),
    "rb_debug_ctx_pop": ([], _c_int),
    "rb_tp_nccl_available": ([], _c_int),
    "rb_tp_nccl_unique_id": ([_vp], _c_int),
    "rb_tp_nccl_comm_init": ([_vp, _c_int, _c_int, ctypes.POINTER(_vp)], _c_int),
    "rb_tp_nccl_comm_destroy": ([_vp], _c_int),
    "rb_tp_create": ([_c_int, _c_int, _c_int, _vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                      ctypes.POINTER(_vp), _vp, _c_size, ctypes.POINTER(_vp)], _c_int),
    "rb_tp_destroy": ([_vp], _c_int),
    "rb_tp_flag_words": ([], _c_size),
    "rb_tp_debug_nowait": ([_vp, _c_int], _c_int),
    "rb_tp_allreduce": ([_vp, _vp, _c_ll, _vp], _c_int),
}

class RbModel(ctypes.Structure):
    """Mirror of rb_model_t (include/rapid_b200.h)."""

    _fields_ = [(n, _c_int) for n in ("hidden", "layers", "q_heads", "kv_heads", "head_dim", "intermediate",
                                      "vocab")] + [
        ("rms_eps", _c_float), ("attn_scale", _c_float), ("embed", _vp), ("final_norm", _vp), ("lm_head", _vp),
        ("ln1", ctypes.POINTER(_vp)), ("wqkv", ctypes.POINTER(_vp)), ("bqkv", ctypes.POINTER(_vp)),
        ("wo", ctypes.POINTER(_vp)), ("ln2", ctypes.POINTER(_vp)), ("wgu", ctypes.POINTER(_vp)),
        ("wd", ctypes.POINTER(_vp)), ("kv_cache", _vp), ("kv_layer_stride_bytes", _c_size), ("num_blocks", _c_int),
        ("block_table", _vp), ("bt_stride", _c_int), ("cos_sin", _vp), ("last_tok", _vp),
        ("qk_layout", _c_int), ("vocab_offset", _c_int)]


class RbWorkspace(ctypes.Structure):
    _fields_ = [(n, _vp) for n in ("x", "h", "qkv", "q", "attn", "gu", "act", "logits")] + [("rows_cap", _c_int)] + [
        (n, _vp) for n in ("ids", "pos", "slot", "seq", "out_ids")] + [
        ("gemm_ws", _vp), ("gemm_ws_bytes", _c_size), ("gemm_counters", _vp), ("gemm_counters_len", _c_int),
        ("attn_ws", _vp), ("attn_ws_bytes", _c_size), ("tp", _vp), ("probe_ev0", _vp), ("probe_ev1", _vp),
        ("probe_layer", _c_int)]


class RbBatch(ctypes.Structure):
    _fields_ = [(n, _c_int) for n in ("rows", "n_decode", "n_prefill", "max_pages", "prefill_slot", "prefill_start",
                                      "ids_from_slots", "logits_decode", "emit_prefill", "sample", "num_sms")]


_SIGS["rb_decoder_forward"] = ([ctypes.POINTER(RbModel), ctypes.POINTER(RbWorkspace), ctypes.POINTER(RbBatch), _vp],
                               _c_int)

EXPORTED_SYMBOLS = tuple(_SIGS)


def decoder_forward(model: RbModel, ws: RbWorkspace, batch: RbBatch, stream=None) -> None:
    """One whole forward iteration launched natively (rb_decoder_forward)."""
    _check(load().rb_decoder_forward(ctypes.byref(model), ctypes.byref(ws), ctypes.byref(batch), _stream(stream)),
           "rb_decoder_forward")


def load(path: str | Path | None = None) -> ctypes.CDLL:
    """Load (once) and type the C-ABI library; raises if it is absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    p = Path(path) if path is not None else lib_path()
    if not p.exists():
        raise RuntimeError(
            f"librapid_b200.so not found at {p}; run `python -m paper_2601_11822_b200.build` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(str(p))
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if os.environ.get("RB_PDL", "1") == "0":  # programmatic dependent launch off (profiling A/B)
        lib.rb_set_pdl(0)
    _LIB = lib
    return lib


def _check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().rb_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed (rc={rc}): {msg}")


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _need_cuda(*ts: torch.Tensor | None) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise RuntimeError("rapid_b200 ops take CUDA tensors only (no CPU fallback)")


_SM_COUNT: dict[int, int] = {}


def device_sm_count(device: int = 0) -> int:
    if device not in _SM_COUNT:
        out = _c_int()
        _check(load().rb_device_sm_count(device, ctypes.byref(out)), "rb_device_sm_count")
        _SM_COUNT[device] = out.value
    return _SM_COUNT[device]


class GemmScratch:
    """Split-K scratch for rb_gemm_bf16 (fp32 partials + self-resetting tile counters)."""

    def __init__(self, device, ws_bytes: int = 64 << 20, n_counters: int = 8192):
        self.ws = torch.empty(ws_bytes // 4, dtype=torch.float32, device=device)
        self.counters = torch.zeros(n_counters, dtype=torch.int32, device=device)

    @property
    def ws_bytes(self) -> int:
        return self.ws.numel() * 4


def linear(x: torch.Tensor, w: torch.Tensor, out: torch.Tensor | None = None, bias: torch.Tensor | None = None,
           residual: torch.Tensor | None = None, *, mode: int = 0, num_sms: int | None = None,
           scratch: GemmScratch | None = None, stream=None) -> torch.Tensor:
    """out[t, o] = x[t, :] . w[o, :] (+ bias[o]) (+ residual[t, o]) on tcgen05 (bf16 in/out, fp32 accumulate)."""
    _need_cuda(x, w, out, bias, residual)
    T, K = x.shape
    O, K2 = w.shape
    if K != K2:
        raise ValueError(f"linear: K mismatch {K} vs {K2}")
    if x.dtype != torch.bfloat16 or w.dtype != torch.bfloat16:
        raise TypeError("linear: bf16 operands required")
    if x.stride(1) != 1 or w.stride(1) != 1:
        raise ValueError("linear: operands must be K-contiguous")
    if out is None:
        out = torch.empty((T, O), dtype=torch.bfloat16, device=x.device)
    if residual is not None and residual.stride() != out.stride():
        raise ValueError("linear: residual must share out's strides")
    sms = num_sms if num_sms is not None else device_sm_count(x.device.index or 0)
    ws = scratch.ws if scratch is not None else None
    _check(
        load().rb_gemm_bf16(
            _ptr(x), _ptr(w), _ptr(out), _ptr(bias), _ptr(residual), T, O, K, x.stride(0), w.stride(0),
            out.stride(0), mode, sms, _ptr(ws), scratch.ws_bytes if scratch else 0,
            _ptr(scratch.counters) if scratch else None, scratch.counters.numel() if scratch else 0, _stream(stream),
        ),
        "rb_gemm_bf16",
    )
    return out


def decode_attention(q: torch.Tensor, cache_layer: torch.Tensor, block_table: torch.Tensor, row_slot: torch.Tensor,
                     seq_lens: torch.Tensor, out: torch.Tensor, *, num_kv_heads: int, max_pages: int | None = None,
                     workspace: torch.Tensor | None = None, scale: float | None = None, num_sms: int | None = None,
                     stream=None) -> torch.Tensor:
    """q, out: [B, Hq, D] (token stride may be padded); cache_layer: [nb, 2, Hkv, 16, D].

    max_pages bounds ceil(seq_len/16) over the rows (default: the block table width)."""
    _need_cuda(q, cache_layer, block_table, row_slot, seq_lens, out, workspace)
    B, Hq, D = q.shape
    sc = scale if scale is not None else 1.0 / math.sqrt(D)
    mp = max_pages if max_pages is not None else block_table.shape[1]
    sms = num_sms if num_sms is not None else device_sm_count(q.device.index or 0)
    _check(
        load().rb_decode_attention(
            _ptr(q), q.stride(0), _ptr(cache_layer), _ptr(block_table), block_table.stride(0), _ptr(row_slot),
            _ptr(seq_lens), _ptr(out), out.stride(0), _ptr(workspace),
            workspace.numel() * workspace.element_size() if workspace is not None else 0, B, Hq, num_kv_heads, D,
            mp, sc, cache_layer.shape[0], sms, _stream(stream),
        ),
        "rb_decode_attention",
    )
    return out


def prefill_attention(q: torch.Tensor, cache_layer: torch.Tensor, block_table_row: torch.Tensor, start: int,
                      out: torch.Tensor, *, num_kv_heads: int, scale: float | None = None,
                      stream=None) -> torch.Tensor:
    """q, out: [T, Hq, D] for chunk positions start..start+T-1 of one request (tcgen05/TMEM/TMA kernel)."""
    _need_cuda(q, cache_layer, block_table_row, out)
    T, Hq, D = q.shape
    sc = scale if scale is not None else 1.0 / math.sqrt(D)
    _check(
        load().rb_prefill_attention(
            _ptr(q), q.stride(0), _ptr(cache_layer), _ptr(block_table_row), T, start, Hq, num_kv_heads, D,
            _ptr(out), out.stride(0), sc, cache_layer.shape[0], _stream(stream),
        ),
        "rb_prefill_attention",
    )
    return out


def rope_cache_write(qkv: torch.Tensor, pos: torch.Tensor, tok_slot: torch.Tensor, block_table: torch.Tensor,
                     cos_sin: torch.Tensor, q_out: torch.Tensor, cache_layer: torch.Tensor, *, num_q_heads: int,
                     num_kv_heads: int, head_dim: int, stream=None) -> None:
    _need_cuda(qkv, pos, tok_slot, block_table, cos_sin, q_out, cache_layer)
    T = qkv.shape[0]
    _check(
        load().rb_rope_cache_write(
            _ptr(qkv), qkv.stride(0), _ptr(pos), _ptr(tok_slot), _ptr(block_table), block_table.stride(0),
            _ptr(cos_sin), _ptr(q_out), q_out.stride(0), _ptr(cache_layer), T, num_q_heads, num_kv_heads, head_dim,
            _stream(stream),
        ),
        "rb_rope_cache_write",
    )


def qkv_rope(x: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None, pos: torch.Tensor, tok_slot: torch.Tensor,
             block_table: torch.Tensor, cos_sin: torch.Tensor, q_out: torch.Tensor, cache_layer: torch.Tensor, *,
             num_q_heads: int, num_kv_heads: int, mode: int = 0, num_sms: int | None = None,
             scratch: GemmScratch | None = None, stream=None) -> None:
    """Fused QKV projection + RoPE + paged K/V write (rb_gemm_qkv_rope); w in the
    pair-interleaved q/k row order of model.interleave_rope_pairs."""
    _need_cuda(x, w, bias, pos, tok_slot, block_table, cos_sin, q_out, cache_layer)
    T, K = x.shape
    D = cache_layer.shape[-1]
    if w.shape != ((num_q_heads + 2 * num_kv_heads) * D, K) or w.stride(1) != 1 or x.stride(1) != 1:
        raise ValueError("qkv_rope: w must be [(Hq + 2 Hkv) * D, K], K-contiguous")
    sms = num_sms if num_sms is not None else device_sm_count(x.device.index or 0)
    _check(
        load().rb_gemm_qkv_rope(
            _ptr(x), _ptr(w), _ptr(bias), T, K, x.stride(0), num_q_heads, num_kv_heads, D, _ptr(pos), _ptr(tok_slot),
            _ptr(block_table), block_table.stride(0), _ptr(cos_sin), _ptr(q_out), q_out.stride(0), _ptr(cache_layer),
            mode, sms, _ptr(scratch.ws) if scratch else None, scratch.ws_bytes if scratch else 0,
            _ptr(scratch.counters) if scratch else None, scratch.counters.numel() if scratch else 0, _stream(stream),
        ),
        "rb_gemm_qkv_rope",
    )


def rmsnorm(x: torch.Tensor, w: torch.Tensor, out: torch.Tensor, eps: float, stream=None) -> torch.Tensor:
    _need_cuda(x, w, out)
    T, H = x.shape
    _check(load().rb_rmsnorm(_ptr(x), x.stride(0), _ptr(w), _ptr(out), out.stride(0), T, H, eps, _stream(stream)),
           "rb_rmsnorm")
    return out


def silu_mul(gate_up: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
    _need_cuda(gate_up, out)
    T, I = out.shape
    _check(load().rb_silu_mul(_ptr(gate_up), gate_up.stride(0), _ptr(out), out.stride(0), T, I, _stream(stream)),
           "rb_silu_mul")
    return out


def embed(table: torch.Tensor, out: torch.Tensor, ids: torch.Tensor | None = None,
          slot_of_row: torch.Tensor | None = None, last_tok: torch.Tensor | None = None,
          ids_out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    _need_cuda(table, out, ids, slot_of_row, last_tok, ids_out)
    T, H = out.shape
    _check(load().rb_embed(_ptr(ids), _ptr(slot_of_row), _ptr(last_tok), _ptr(table), _ptr(out), T, H, _ptr(ids_out),
                           _stream(stream)), "rb_embed")
    return out


def argmax(logits: torch.Tensor, out: torch.Tensor, slot_of_row: torch.Tensor | None = None,
           last_tok: torch.Tensor | None = None, row_valid: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    _need_cuda(logits, out, slot_of_row, last_tok, row_valid)
    T, V = logits.shape
    _check(load().rb_argmax(_ptr(logits), logits.stride(0), T, V, _ptr(out), _ptr(slot_of_row), _ptr(last_tok),
                            _ptr(row_valid), _stream(stream)), "rb_argmax")
    return out


def block_table_update(upd: torch.Tensor, block_table: torch.Tensor, max_updates: int, stream=None) -> None:
    _need_cuda(upd, block_table)
    _check(load().rb_block_table_update(_ptr(upd), _ptr(block_table), block_table.stride(0), max_updates,
                                        _stream(stream)), "rb_block_table_update")


def set_last_token(last_tok: torch.Tensor, slot: int, value: int = 0, value_ptr: torch.Tensor | None = None,
                   stream=None) -> None:
    _need_cuda(last_tok, value_ptr)
    _check(load().rb_set_last_token(_ptr(last_tok), slot, _ptr(value_ptr), value, _stream(stream)),
           "rb_set_last_token")


class GreenSplit:
    """Two disjoint SM partitions (CUDA green contexts), one stream each."""

    def __init__(self, first_sms: int, device: int = 0):
        h, s0, s1 = _vp(), _vp(), _vp()
        n0, n1 = _c_int(), _c_int()
        _check(load().rb_green_split(device, first_sms, ctypes.byref(h), ctypes.byref(s0), ctypes.byref(s1),
                                     ctypes.byref(n0), ctypes.byref(n1)), "rb_green_split")
        self.handle = h.value
        self.stream_handles = (s0.value, s1.value)
        self.sms = (n0.value, n1.value)
        dev = torch.device("cuda", device)
        self.streams = tuple(torch.cuda.ExternalStream(s, device=dev) for s in self.stream_handles)

    def close(self) -> None:
        if self.handle:
            load().rb_green_destroy(self.handle)
            self.handle = None

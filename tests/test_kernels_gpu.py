"""Per-kernel parity of the sm_100a library against plain PyTorch fp32 references.

Every call goes through the C ABI (librapid_b200.so via ctypes). Tolerances are
bf16-output tolerances: relative L2 error <= 1e-2 for GEMMs / attention.
"""

import math

import pytest
import torch

from paper_2601_11822_b200 import ops

pytestmark = pytest.mark.gpu

DEV = "cuda"


def rel_l2(a: torch.Tensor, b: torch.Tensor) -> float:
    a = a.float()
    b = b.float()
    return (torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b).clamp_min(1e-12)).item()


@pytest.fixture(scope="module")
def scratch():
    return ops.GemmScratch(DEV)


@pytest.mark.parametrize("T,O,K", [(1024, 4096, 4096), (1000, 1536, 1024), (300, 6144, 512), (2048, 256, 128)])
def test_linear_normal(T, O, K, scratch):
    g = torch.Generator(device=DEV).manual_seed(T + O + K)
    x = torch.randn(T, K, device=DEV, generator=g).bfloat16()
    w = (torch.randn(O, K, device=DEV, generator=g) * 0.05).bfloat16()
    y = ops.linear(x, w, mode=1, scratch=scratch)
    torch.cuda.synchronize()
    ref = x.float() @ w.float().T
    assert rel_l2(y, ref) < 1e-2


def test_linear_bias_residual(scratch):
    g = torch.Generator(device=DEV).manual_seed(7)
    T, O, K = 513, 1024, 640
    x = torch.randn(T, K, device=DEV, generator=g).bfloat16()
    w = (torch.randn(O, K, device=DEV, generator=g) * 0.05).bfloat16()
    b = torch.randn(O, device=DEV, generator=g).bfloat16()
    r = torch.randn(T, O, device=DEV, generator=g).bfloat16()
    ref = x.float() @ w.float().T + b.float() + r.float()
    y = r.clone()
    ops.linear(x, w, out=y, bias=b, residual=y, mode=1, scratch=scratch)  # in-place residual
    torch.cuda.synchronize()
    assert rel_l2(y, ref) < 1e-2


@pytest.mark.parametrize("T", [1, 7, 16, 33, 64, 128, 200, 256])
@pytest.mark.parametrize("O,K", [(4096, 4096), (6144, 4096), (1024, 14336), (8192, 4096)])
def test_linear_swap_ab(T, O, K, scratch):
    g = torch.Generator(device=DEV).manual_seed(T * 31 + O)
    x = torch.randn(T, K, device=DEV, generator=g).bfloat16()
    w = (torch.randn(O, K, device=DEV, generator=g) * 0.05).bfloat16()
    b = torch.randn(O, device=DEV, generator=g).bfloat16()
    r = torch.randn(T, O, device=DEV, generator=g).bfloat16()
    y = ops.linear(x, w, bias=b, residual=r, mode=2, scratch=scratch)
    y2 = ops.linear(x, w, bias=b, residual=r, mode=2, scratch=None)  # no split-K
    # a decode-partition grid: two A sub-tiles per stage at small batches (MT=2 kernels)
    y3 = ops.linear(x, w, bias=b, residual=r, mode=2, scratch=scratch, num_sms=64)
    torch.cuda.synchronize()
    ref = x.float() @ w.float().T + b.float() + r.float()
    assert rel_l2(y, ref) < 1e-2
    assert rel_l2(y2, ref) < 1e-2
    assert rel_l2(y3, ref) < 1e-2


@pytest.mark.parametrize("bn", [0, 128, 160, 192, 224, 256])
def test_linear_prefill_tile_widths(bn, scratch):
    """Token-major GEMM at every tile width the wave-aware chooser can pick (0 = its own choice
    on an 84-SM grid: 224 for a 1023-token O projection), plain + bias/residual and SwiGLU."""
    from paper_2601_11822_b200.model import interleave_gate_up

    lib = ops.load()
    assert lib.rb_debug_gemm_prefill_bn(bn) == 0
    try:
        g = torch.Generator(device=DEV).manual_seed(bn + 7)
        T, O, K = 1023, 4096, 1024
        x = torch.randn(T, K, device=DEV, generator=g).bfloat16()
        w = (torch.randn(O, K, device=DEV, generator=g) * 0.05).bfloat16()
        b = torch.randn(O, device=DEV, generator=g).bfloat16()
        r = torch.randn(T, O, device=DEV, generator=g).bfloat16()
        y = ops.linear(x, w, bias=b, residual=r, mode=1, num_sms=84, scratch=scratch)
        I = 1792
        gate = (torch.randn(I, K, device=DEV, generator=g) * 0.05).bfloat16()
        up = (torch.randn(I, K, device=DEV, generator=g) * 0.05).bfloat16()
        wgu = interleave_gate_up(gate, up).contiguous()
        a = torch.empty(T, I, device=DEV, dtype=torch.bfloat16)
        lib.rb_gemm_bf16(x.data_ptr(), wgu.data_ptr(), a.data_ptr(), None, None, T, 2 * I, K, K, K, I, 1 | 4, 84,
                         scratch.ws.data_ptr(), scratch.ws_bytes, scratch.counters.data_ptr(), scratch.counters.numel(),
                         torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
    finally:
        lib.rb_debug_gemm_prefill_bn(0)
    assert rel_l2(y, x.float() @ w.float().T + b.float() + r.float()) < 1e-2
    ref = torch.nn.functional.silu(x.float() @ gate.float().T) * (x.float() @ up.float().T)
    assert rel_l2(a, ref) < 1e-2


def test_prefill_tile_width_rejects_bad_values():
    lib = ops.load()
    assert lib.rb_debug_gemm_prefill_bn(100) != 0
    assert lib.rb_debug_gemm_prefill_bn(512) != 0
    assert lib.rb_debug_gemm_prefill_bn(0) == 0


@pytest.mark.parametrize("T,mode,sms", [(1, 2, 148), (1, 2, 64), (37, 2, 148), (37, 2, 64), (200, 2, 148),
                                        (300, 1, 148), (1023, 1, 148)])
@pytest.mark.parametrize("I", [1024, 3584])
def test_linear_fused_swiglu(T, mode, sms, I, scratch):
    """mode | 4: gate/up rows interleaved in 16-blocks, epilogue emits silu(gate) * up."""
    from paper_2601_11822_b200.model import interleave_gate_up

    g = torch.Generator(device=DEV).manual_seed(T + I)
    K = 1024
    x = torch.randn(T, K, device=DEV, generator=g).bfloat16()
    gate = (torch.randn(I, K, device=DEV, generator=g) * 0.05).bfloat16()
    up = (torch.randn(I, K, device=DEV, generator=g) * 0.05).bfloat16()
    w = interleave_gate_up(gate, up).contiguous()
    y = torch.empty(T, I, device=DEV, dtype=torch.bfloat16)
    ops.load().rb_gemm_bf16(x.data_ptr(), w.data_ptr(), y.data_ptr(), None, None, T, 2 * I, K, K, K, I, mode | 4, sms,
                            scratch.ws.data_ptr(), scratch.ws_bytes, scratch.counters.data_ptr(),
                            scratch.counters.numel(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = torch.nn.functional.silu(x.float() @ gate.float().T) * (x.float() @ up.float().T)
    assert rel_l2(y, ref) < 1e-2


def _make_cache(nb, Hkv, D, gen):
    return (torch.randn(nb, 2, Hkv, 16, D, device=DEV, generator=gen) * 0.5).bfloat16()


def _gather_kv(cache, bt_row, n):
    # -> K, V [n, Hkv, D]
    pages = bt_row[: (n + 15) // 16].long()
    kv = cache[pages]  # [np, 2, Hkv, 16, D]
    k = kv[:, 0].permute(0, 2, 1, 3).reshape(-1, cache.shape[2], cache.shape[4])[:n]
    v = kv[:, 1].permute(0, 2, 1, 3).reshape(-1, cache.shape[2], cache.shape[4])[:n]
    return k, v


def _ref_attn(q, k, v, causal_offset=None):
    # q [T, Hq, D], k/v [n, Hkv, D]
    T, Hq, D = q.shape
    Hkv = k.shape[1]
    G = Hq // Hkv
    kf = k.float().repeat_interleave(G, dim=1)
    vf = v.float().repeat_interleave(G, dim=1)
    s = torch.einsum("thd,nhd->htn", q.float(), kf) / math.sqrt(D)
    if causal_offset is not None:
        tpos = torch.arange(T, device=q.device)[:, None] + causal_offset
        npos = torch.arange(k.shape[0], device=q.device)[None, :]
        s = s.masked_fill((npos > tpos)[None], float("-inf"))
    p = torch.softmax(s, dim=-1)
    return torch.einsum("htn,nhd->thd", p, vf)


@pytest.mark.parametrize("Hq,Hkv", [(32, 8), (8, 2), (40, 8), (8, 1), (16, 8)])
@pytest.mark.parametrize("sms", [148, 72, 8])
def test_decode_attention(Hq, Hkv, sms):
    gen = torch.Generator(device=DEV).manual_seed(Hq * 10 + Hkv + sms)
    D, nb, B = 128, 512, 6
    cache = _make_cache(nb, Hkv, D, gen)
    seq = torch.tensor([1, 15, 16, 17, 300, 1000], dtype=torch.int32, device=DEV)
    maxb = 64
    perm = torch.randperm(nb, device=DEV, generator=gen).int()
    bt = perm[: B * maxb].view(B, maxb).contiguous()
    slots = torch.arange(B, dtype=torch.int32, device=DEV).flip(0).contiguous()
    q = torch.randn(B, Hq, D, device=DEV, generator=gen).bfloat16()
    out = torch.zeros(B, Hq, D, device=DEV, dtype=torch.bfloat16)
    ws = torch.zeros(B * Hq * 8 * (D + 2), device=DEV, dtype=torch.float32)
    ops.decode_attention(q, cache, bt, slots, seq, out, num_kv_heads=Hkv, max_pages=maxb, workspace=ws, num_sms=sms)
    torch.cuda.synchronize()
    for b in range(B):
        n = int(seq[b])
        k, v = _gather_kv(cache, bt[int(slots[b])], n)
        ref = _ref_attn(q[b : b + 1], k, v)
        assert rel_l2(out[b : b + 1], ref) < 1e-2, (b, n)


@pytest.mark.parametrize("one_op", [0, 1])
@pytest.mark.parametrize("shape", [1, 2, 3, 4])
def test_decode_attention_load_modes(one_op, shape):
    """Every ring shape (warps x stages) with both page-load forms: one 5D TMA op per page
    (default) and four 2D {64, 16} boxes."""
    lib = ops.load()
    gen = torch.Generator(device=DEV).manual_seed(7 * shape + one_op)
    D, nb, B, Hq, Hkv = 128, 512, 5, 32, 8
    cache = _make_cache(nb, Hkv, D, gen)
    seq = torch.tensor([3, 16, 33, 700, 1001], dtype=torch.int32, device=DEV)
    maxb = 64
    bt = torch.randperm(nb, device=DEV, generator=gen).int()[: B * maxb].view(B, maxb).contiguous()
    slots = torch.arange(B, dtype=torch.int32, device=DEV)
    q = torch.randn(B, Hq, D, device=DEV, generator=gen).bfloat16()
    out = torch.zeros(B, Hq, D, device=DEV, dtype=torch.bfloat16)
    ws = torch.zeros(B * Hq * 8 * (D + 2), device=DEV, dtype=torch.float32)
    assert lib.rb_debug_decode_kv_one_op(one_op) == 0 and lib.rb_debug_decode_attn_shape(shape) == 0
    try:
        ops.decode_attention(q, cache, bt, slots, seq, out, num_kv_heads=Hkv, max_pages=maxb, workspace=ws,
                             num_sms=40)
        torch.cuda.synchronize()
    finally:
        lib.rb_debug_decode_kv_one_op(1)
        lib.rb_debug_decode_attn_shape(0)
    for b in range(B):
        k, v = _gather_kv(cache, bt[b], int(seq[b]))
        assert rel_l2(out[b : b + 1], _ref_attn(q[b : b + 1], k, v)) < 1e-2, b


@pytest.mark.parametrize("sms", [148, 40])
def test_decode_attention_growing_max(sms):
    """Scores that grow along the context (and some that barely move) exercise the lazy
    running max: pages that raise it by more than 2^8 in some heads but not others."""
    gen = torch.Generator(device=DEV).manual_seed(5 + sms)
    D, nb, B, Hq, Hkv = 128, 512, 4, 32, 8
    cache = _make_cache(nb, Hkv, D, gen)
    seq = torch.tensor([40, 333, 700, 1001], dtype=torch.int32, device=DEV)
    maxb = 64
    bt = torch.randperm(nb, device=DEV, generator=gen).int()[: B * maxb].view(B, maxb).contiguous()
    ramp = torch.linspace(0.1, 8.0, 16 * maxb, device=DEV).view(maxb, 1, 16, 1)
    for b in range(B):
        pages = bt[b].long()
        cache[pages, 0] = (cache[pages, 0].float() * ramp).bfloat16()
    slots = torch.arange(B, dtype=torch.int32, device=DEV)
    q = torch.randn(B, Hq, D, device=DEV, generator=gen)
    q[:, ::3] *= 0.02  # some heads barely move their max
    q = q.bfloat16()
    out = torch.zeros(B, Hq, D, device=DEV, dtype=torch.bfloat16)
    ws = torch.zeros(B * Hq * 16 * (D + 2), device=DEV, dtype=torch.float32)
    ops.decode_attention(q, cache, bt, slots, seq, out, num_kv_heads=Hkv, max_pages=maxb, workspace=ws, num_sms=sms)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    for b in range(B):
        k, v = _gather_kv(cache, bt[b], int(seq[b]))
        assert rel_l2(out[b : b + 1], _ref_attn(q[b : b + 1], k, v)) < 1e-2, b


def test_decode_attention_stale_nan_tail():
    """Rows past the sequence end in the last page may hold non-finite stale data."""
    gen = torch.Generator(device=DEV).manual_seed(21)
    D, nb, Hq, Hkv = 128, 64, 32, 8
    cache = _make_cache(nb, Hkv, D, gen)
    seq = torch.tensor([5, 16, 37, 250], dtype=torch.int32, device=DEV)
    bt = torch.randperm(nb, device=DEV, generator=gen).int()[:4 * 16].view(4, 16).contiguous()
    for b in range(4):
        n = int(seq[b])
        if n % 16:
            cache[int(bt[b, n // 16]), :, :, n % 16:] = float("nan")
    slots = torch.arange(4, dtype=torch.int32, device=DEV)
    q = torch.randn(4, Hq, D, device=DEV, generator=gen).bfloat16()
    out = torch.empty(4, Hq, D, device=DEV, dtype=torch.bfloat16)
    ws = torch.zeros(4 * Hq * 2 * (D + 2), device=DEV, dtype=torch.float32)
    ops.decode_attention(q, cache, bt, slots, seq, out, num_kv_heads=Hkv, max_pages=16, workspace=ws)
    torch.cuda.synchronize()
    for b in range(4):
        k, v = _gather_kv(cache, bt[b], int(seq[b]))
        assert torch.isfinite(out[b]).all()
        assert rel_l2(out[b : b + 1], _ref_attn(q[b : b + 1], k, v)) < 1e-2


def test_decode_attention_padded_rows():
    gen = torch.Generator(device=DEV).manual_seed(3)
    D, nb, Hq, Hkv = 128, 64, 8, 2
    cache = _make_cache(nb, Hkv, D, gen)
    bt = torch.arange(nb, dtype=torch.int32, device=DEV).view(4, 16).contiguous()
    slots = torch.arange(4, dtype=torch.int32, device=DEV)
    seq = torch.tensor([40, 0, 0, 3], dtype=torch.int32, device=DEV)
    q = torch.randn(4, Hq, D, device=DEV, generator=gen).bfloat16()
    out = torch.full((4, Hq, D), 7.0, device=DEV, dtype=torch.bfloat16)
    ops.decode_attention(q, cache, bt, slots, seq, out, num_kv_heads=Hkv, max_pages=16)
    torch.cuda.synchronize()
    assert torch.all(out[1] == 7.0) and torch.all(out[2] == 7.0)  # padded rows untouched
    k, v = _gather_kv(cache, bt[3], 3)
    assert rel_l2(out[3:4], _ref_attn(q[3:4], k, v)) < 1e-2


@pytest.mark.parametrize("T,start,Hq,Hkv", [(100, 0, 8, 2), (64, 37, 8, 2), (200, 130, 32, 8), (1, 50, 40, 8),
                                            (257, 0, 8, 1), (300, 500, 32, 8), (1100, 0, 8, 2), (1300, 700, 8, 2)])
def test_prefill_attention(T, start, Hq, Hkv):
    # (1100, 0): 9 query tiles from position 0 -> one tile per CTA in the tcgen05 kernel; the
    # others run two tiles per CTA (paired warpgroups sharing K/V)
    gen = torch.Generator(device=DEV).manual_seed(T + start)
    D, nb = 128, 256
    cache = _make_cache(nb, Hkv, D, gen)
    bt_row = torch.randperm(nb, device=DEV, generator=gen).int()[:160].contiguous()
    assert (start + T + 15) // 16 <= 160
    q = torch.randn(T, Hq, D, device=DEV, generator=gen).bfloat16()
    out = torch.empty(T, Hq, D, device=DEV, dtype=torch.bfloat16)
    ops.prefill_attention(q, cache, bt_row, start, out, num_kv_heads=Hkv)
    torch.cuda.synchronize()
    k, v = _gather_kv(cache, bt_row, start + T)
    ref = _ref_attn(q, k, v, causal_offset=start)
    assert rel_l2(out, ref) < 1e-2


@pytest.mark.parametrize("tiles", [1, 2])
@pytest.mark.parametrize("T,start", [(1100, 0), (1023, 0), (640, 0), (129, 0), (700, 900)])
def test_prefill_attention_forced_tiles(T, start, tiles):
    """Both CTA shapes on every chunk shape: one query tile per CTA, or mirrored causal pairs
    (g, nqb-1-g) — odd tile counts leave the middle tile alone in its CTA."""
    lib = ops.load()
    gen = torch.Generator(device=DEV).manual_seed(3 * T + start + tiles)
    D, nb, Hq, Hkv = 128, 256, 8, 2
    cache = _make_cache(nb, Hkv, D, gen)
    bt_row = torch.randperm(nb, device=DEV, generator=gen).int()[:160].contiguous()
    q = torch.randn(T, Hq, D, device=DEV, generator=gen).bfloat16()
    out = torch.empty(T, Hq, D, device=DEV, dtype=torch.bfloat16)
    assert lib.rb_debug_pattn_tiles(tiles) == 0
    try:
        ops.prefill_attention(q, cache, bt_row, start, out, num_kv_heads=Hkv)
        torch.cuda.synchronize()
    finally:
        lib.rb_debug_pattn_tiles(0)
    k, v = _gather_kv(cache, bt_row, start + T)
    assert rel_l2(out, _ref_attn(q, k, v, causal_offset=start)) < 1e-2


@pytest.mark.parametrize("T,start", [(300, 0), (200, 333)])
def test_prefill_attention_growing_max(T, start):
    """Scores that grow along the keys force the tcgen05 kernel's lazy O rescale (row max
    rising by more than 2^8 after the first tile, in some rows of a warp but not others)."""
    gen = torch.Generator(device=DEV).manual_seed(T + 7 * start)
    D, nb, Hq, Hkv = 128, 128, 8, 2
    cache = _make_cache(nb, Hkv, D, gen)
    bt_row = torch.randperm(nb, device=DEV, generator=gen).int()[:48].contiguous()
    n = start + T
    q = torch.randn(T, Hq, D, device=DEV, generator=gen)
    q[::3] *= 0.05  # some rows barely move their max: a warp's rows disagree on rescaling
    q = q.bfloat16()
    pages = bt_row[: (n + 15) // 16].long()
    ramp = torch.linspace(0.2, 6.0, (n + 15) // 16 * 16, device=DEV).view(-1, 1, 16, 1)
    k = cache[pages, 0].float() * ramp  # [pages, Hkv, 16, D]: later keys score much higher
    cache[pages, 0] = k.bfloat16()
    out = torch.empty(T, Hq, D, device=DEV, dtype=torch.bfloat16)
    ops.prefill_attention(q, cache, bt_row, start, out, num_kv_heads=Hkv)
    torch.cuda.synchronize()
    kk, vv = _gather_kv(cache, bt_row, n)
    assert torch.isfinite(out).all()
    assert rel_l2(out, _ref_attn(q, kk, vv, causal_offset=start)) < 1e-2


def test_prefill_attention_stale_nan_tail():
    """Slots after the chunk end in its last page may never have been written."""
    gen = torch.Generator(device=DEV).manual_seed(99)
    D, nb, Hq, Hkv, T, start = 128, 64, 32, 8, 70, 25
    cache = _make_cache(nb, Hkv, D, gen)
    bt_row = torch.randperm(nb, device=DEV, generator=gen).int()[:16].contiguous()
    n = start + T
    cache[int(bt_row[n // 16]), :, :, n % 16:] = float("nan")
    q = torch.randn(T, Hq, D, device=DEV, generator=gen).bfloat16()
    out = torch.empty(T, Hq, D, device=DEV, dtype=torch.bfloat16)
    ops.prefill_attention(q, cache, bt_row, start, out, num_kv_heads=Hkv)
    torch.cuda.synchronize()
    k, v = _gather_kv(cache, bt_row, n)
    assert torch.isfinite(out).all()
    assert rel_l2(out, _ref_attn(q, k, v, causal_offset=start)) < 1e-2


def _cos_sin(max_pos, D, theta=10000.0):
    inv = 1.0 / (theta ** (torch.arange(0, D, 2, dtype=torch.float64) / D))
    ang = torch.arange(max_pos, dtype=torch.float64)[:, None] * inv[None]
    return torch.cat([ang.cos(), ang.sin()], dim=1).float()


def test_rope_cache_write():
    gen = torch.Generator(device=DEV).manual_seed(11)
    Hq, Hkv, D, T, nb = 8, 2, 128, 37, 32
    qkv = torch.randn(T, (Hq + 2 * Hkv) * D, device=DEV, generator=gen).bfloat16()
    pos = torch.arange(5, 5 + T, dtype=torch.int32, device=DEV)
    pos[3] = -1  # skipped row
    slots = torch.full((T,), 1, dtype=torch.int32, device=DEV)
    bt = torch.tensor([[0] * 8, [9, 4, 20, 3, 0, 0, 0, 0]], dtype=torch.int32, device=DEV)
    cs = _cos_sin(128, D).to(DEV)
    q_out = torch.zeros(T, Hq * D, device=DEV, dtype=torch.bfloat16)
    cache = torch.zeros(nb, 2, Hkv, 16, D, device=DEV, dtype=torch.bfloat16)
    ops.rope_cache_write(qkv, pos, slots, bt, cs, q_out, cache, num_q_heads=Hq, num_kv_heads=Hkv, head_dim=D)
    torch.cuda.synchronize()

    def rope(x, p):
        c = cs[p, : D // 2].to(DEV)
        s = cs[p, D // 2 :].to(DEV)
        x1, x2 = x[..., : D // 2].float(), x[..., D // 2 :].float()
        return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)

    for t in range(T):
        p = int(pos[t])
        if p < 0:
            assert torch.all(q_out[t] == 0)
            continue
        row = qkv[t]
        qr = rope(row[: Hq * D].view(Hq, D), p)
        kr = rope(row[Hq * D : (Hq + Hkv) * D].view(Hkv, D), p)
        v = row[(Hq + Hkv) * D :].view(Hkv, D)
        page = int(bt[1, p // 16])
        assert rel_l2(q_out[t].view(Hq, D), qr) < 1e-2
        assert rel_l2(cache[page, 0, :, p % 16], kr) < 1e-2
        assert torch.equal(cache[page, 1, :, p % 16], v)


@pytest.mark.parametrize("T,mode,bias,sms", [(7, 2, False, 148), (24, 2, True, 64), (128, 2, True, 72),
                                             (200, 0, False, 148),
                                             (777, 1, True, 76), (1023, 1, False, 148)])
def test_qkv_rope_fused(T, mode, bias, sms, scratch):
    """rb_gemm_qkv_rope (QKV GEMM with RoPE + paged K/V write in its epilogue) against
    fp32 torch: x @ W^T (+b) in the standard rotate-half layout, RoPE, scatter to pages."""
    from paper_2601_11822_b200.model import interleave_rope_pairs

    gen = torch.Generator(device=DEV).manual_seed(T + mode)
    Hq, Hkv, D, H = 32, 8, 128, 1024
    nq = (Hq + 2 * Hkv) * D
    x = torch.randn(T, H, device=DEV, generator=gen).bfloat16()
    w = (torch.randn(nq, H, device=DEV, generator=gen) * 0.03).bfloat16()
    b = (torch.randn(nq, device=DEV, generator=gen) * 0.5).bfloat16() if bias else None
    start = 37
    pos = torch.arange(start, start + T, dtype=torch.int32, device=DEV)
    pos[T // 2] = -1  # padding row: nothing written
    slots = torch.full((T,), 1, dtype=torch.int32, device=DEV)
    npg = (start + T + 15) // 16
    nb = npg + 8
    bt = torch.zeros(2, npg, dtype=torch.int32, device=DEV)
    bt[1] = torch.randperm(nb, generator=torch.Generator().manual_seed(T))[:npg].to(DEV, torch.int32)
    cs = _cos_sin(start + T + 16, D).to(DEV)
    q_out = torch.zeros(T, Hq * D, device=DEV, dtype=torch.bfloat16)
    cache = torch.zeros(nb, 2, Hkv, 16, D, device=DEV, dtype=torch.bfloat16)
    wi = interleave_rope_pairs(w, Hq, Hkv, D)
    bi = interleave_rope_pairs(b, Hq, Hkv, D) if bias else None
    ops.qkv_rope(x, wi, bi, pos, slots, bt, cs, q_out, cache, num_q_heads=Hq, num_kv_heads=Hkv, mode=mode,
                 num_sms=sms, scratch=scratch)
    torch.cuda.synchronize()

    ref = x.float() @ w.float().T
    if bias:
        ref = ref + b.float()
    p = pos.long().clamp_min(0)
    c, s = cs[p, : D // 2][:, None], cs[p, D // 2 :][:, None]

    def rope(z):  # [T, heads, D] rotate-half
        z1, z2 = z[..., : D // 2], z[..., D // 2 :]
        return torch.cat([z1 * c - z2 * s, z2 * c + z1 * s], dim=-1)

    qr = rope(ref[:, : Hq * D].view(T, Hq, D))
    kr = rope(ref[:, Hq * D:(Hq + Hkv) * D].view(T, Hkv, D))
    vr = ref[:, (Hq + Hkv) * D:].view(T, Hkv, D)
    half = D // 2
    perm = torch.stack([torch.arange(half), torch.arange(half) + half], dim=1).reshape(-1).to(DEV)
    valid = pos >= 0
    # q/k come out pair-interleaved: dim perm[i] of the standard layout sits at column i
    assert rel_l2(q_out.view(T, Hq, D)[valid], qr[valid][..., perm]) < 1e-2
    assert torch.all(q_out[~valid] == 0)
    page = bt[1][(p // 16)]
    k_got = cache[page, 0, :, p % 16]  # [T, Hkv, D]
    v_got = cache[page, 1, :, p % 16]
    assert rel_l2(k_got[valid], kr[valid][..., perm]) < 1e-2
    assert rel_l2(v_got[valid], vr[valid]) < 1e-2
    # the padding row's would-be slot stays untouched
    pp = start + T // 2
    assert torch.all(cache[bt[1][pp // 16], :, :, pp % 16] == 0)
    # scores are invariant: q.k with both permuted == q.k in the standard layout
    qk_std = (qr[valid][:, ::4] * kr[valid]).sum(-1)
    qk_int = (q_out.view(T, Hq, D)[valid][:, ::4].float() * k_got[valid].float()).sum(-1)
    assert rel_l2(qk_int, qk_std) < 2e-2


def test_rmsnorm_silu_embed_argmax():
    gen = torch.Generator(device=DEV).manual_seed(5)
    T, H, I, V = 9, 4096, 1024, 4096
    x = torch.randn(T, H, device=DEV, generator=gen).bfloat16()
    w = torch.randn(H, device=DEV, generator=gen).bfloat16()
    y = torch.empty_like(x)
    ops.rmsnorm(x, w, y, 1e-5)
    xf = x.float()
    ref = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-5) * w.float()
    assert rel_l2(y, ref) < 1e-2

    gu = torch.randn(T, 2 * I, device=DEV, generator=gen).bfloat16()
    a = torch.empty(T, I, device=DEV, dtype=torch.bfloat16)
    ops.silu_mul(gu, a)
    ref = torch.nn.functional.silu(gu[:, :I].float()) * gu[:, I:].float()
    assert rel_l2(a, ref) < 1e-2

    table = torch.randn(V, 512, device=DEV, generator=gen).bfloat16()
    ids = torch.randint(0, V, (T,), device=DEV, generator=gen, dtype=torch.int32)
    e = torch.empty(T, 512, device=DEV, dtype=torch.bfloat16)
    ops.embed(table, e, ids=ids)
    assert torch.equal(e, table[ids.long()])
    # decode-style: ids from device slot state
    last = torch.randint(0, V, (16,), device=DEV, generator=gen, dtype=torch.int32)
    slot_of_row = torch.tensor([3, 0, 15, 3, 1, 2, 9, 8, 7], dtype=torch.int32, device=DEV)
    ids_out = torch.empty(T, dtype=torch.int32, device=DEV)
    ops.embed(table, e, slot_of_row=slot_of_row, last_tok=last, ids_out=ids_out)
    assert torch.equal(ids_out, last[slot_of_row.long()])

    logits = torch.randn(T, V, device=DEV, generator=gen).bfloat16()
    logits[2, 100] = 50.0
    logits[2, 200] = 50.0  # tie -> lowest index
    out = torch.empty(T, dtype=torch.int32, device=DEV)
    last2 = torch.zeros(16, dtype=torch.int32, device=DEV)
    ops.argmax(logits, out, slot_of_row=slot_of_row, last_tok=last2)
    torch.cuda.synchronize()
    assert torch.equal(out.long(), logits.float().argmax(-1))
    assert int(out[2]) == 100
    assert int(last2[15]) == int(out[2])


def test_block_table_update_and_last_token():
    bt = torch.zeros(4, 8, dtype=torch.int32, device=DEV)
    upd = torch.tensor([2, 1, 3, 77, 3, 0, 5, 0, 0, 0], dtype=torch.int32, device=DEV)
    ops.block_table_update(upd, bt, max_updates=3)
    last = torch.zeros(4, dtype=torch.int32, device=DEV)
    ops.set_last_token(last, 2, value=99)
    torch.cuda.synchronize()
    assert int(bt[1, 3]) == 77 and int(bt[3, 0]) == 5 and int(bt.sum()) == 82
    assert int(last[2]) == 99


def test_green_split_streams(scratch):
    total = ops.device_sm_count(0)
    gs = ops.GreenSplit(72)
    try:
        assert gs.sms[0] >= 72 and gs.sms[0] + gs.sms[1] <= total
        x = torch.randn(256, 1024, device=DEV).bfloat16()
        w = torch.randn(512, 1024, device=DEV).bfloat16()
        ys = []
        for st, n in zip(gs.streams, gs.sms):
            with torch.cuda.stream(st):
                ys.append(ops.linear(x, w, mode=1, num_sms=n, stream=st))
        for st in gs.streams:
            st.synchronize()
        ref = x.float() @ w.float().T
        for y in ys:
            assert rel_l2(y, ref) < 1e-2
    finally:
        gs.close()

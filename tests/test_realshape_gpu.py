"""Parity at the BASELINE configs' real sizes (VERDICT r1 "configs untested at their real sizes").

  * K3 decode attention at the cfg-3 and cfg-5 contexts (2,304 = 2048 + 256 and 8,256 =
    8192 + 64 + 1 page) for every GQA group the configs use: G = 4 (Llama-3.1-8B, 32/8),
    G = 5 (Qwen2.5-14B, 40/8), G = 8 (Llama-3.1-70B, 64/8; TP=8 rank 8/1), on the full GPU and
    on a 32-SM decode partition (the width the measured ARM picks for cfg 5).
  * K2 prefill attention for a 2,048-token chunk after a 6,144-token paged prefix (the fourth
    chunk of a cfg-5 8,192-token prompt) with Qwen-14B and Llama-8B heads.
  * K1/K4 GEMMs at the Qwen2.5-14B shapes (QKV N = 7,168, O 5,120, gate|up 27,648 with the
    fused SwiGLU, down K = 13,824, lm_head N = 152,064) for a 2,048-token prefill chunk and
    decode batches 1 / 64 / 256 on full and partition grids.
  * A 2-layer Llama-3.1-8B and a 2-layer Qwen2.5-14B (QKV bias, theta 1e6, eps 1e-6, vocab
    152,064) through the native forward (chunked prefill, then batched CUDA-graph-shaped
    decode rows) against oracle/llama_fp32.py: per-step logits rel-L2 <= 2e-2 (north star), or
    <= 1.6x the error of an ideal bf16 pipeline where the bf16 format itself costs more (see TOL).

Tolerances: rel-L2 <= 1e-2 for bf16 kernel outputs vs fp32 torch, 2e-2 for model logits.
"""

import dataclasses
import math

import pytest
import torch

from paper_2601_11822_b200 import ops

pytestmark = pytest.mark.gpu
DEV = "cuda"
D = 128


def rel_l2(a, b) -> float:
    a, b = a.float(), b.float()
    return float(torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b).clamp_min(1e-12))


def _gather(cache, row, n):
    pages = row[: (n + 15) // 16].long()
    kv = cache[pages]
    k = kv[:, 0].permute(0, 2, 1, 3).reshape(-1, cache.shape[2], D)[:n]
    v = kv[:, 1].permute(0, 2, 1, 3).reshape(-1, cache.shape[2], D)[:n]
    return k, v


def _attn_ref(q, k, v, causal_offset=None):
    T, Hq, _ = q.shape
    G = Hq // k.shape[1]
    s = torch.einsum("thd,nhd->htn", q.float(), k.float().repeat_interleave(G, 1)) / math.sqrt(D)
    if causal_offset is not None:
        tpos = torch.arange(T, device=q.device)[:, None] + causal_offset
        s = s.masked_fill((torch.arange(k.shape[0], device=q.device)[None, :] > tpos)[None], float("-inf"))
    return torch.einsum("htn,nhd->thd", torch.softmax(s, -1), v.float().repeat_interleave(G, 1))


@pytest.mark.parametrize("Hq,Hkv", [(32, 8), (40, 8), (64, 8), (8, 1)])
@pytest.mark.parametrize("sms", [148, 32])
def test_decode_attention_long_context(Hq, Hkv, sms):
    gen = torch.Generator(device=DEV).manual_seed(Hq + 3 * Hkv + sms)
    seq = torch.tensor([2304, 8256, 1, 4097, 8255, 2303], dtype=torch.int32, device=DEV)
    B = seq.numel()
    maxp = (8256 + 15) // 16
    nb = B * maxp + 16
    cache = (torch.randn(nb, 2, Hkv, 16, D, device=DEV, generator=gen) * 0.5).bfloat16()
    bt = torch.randperm(nb, device=DEV, generator=gen).int()[: B * maxp].view(B, maxp).contiguous()
    slots = torch.tensor([4, 2, 0, 5, 1, 3], dtype=torch.int32, device=DEV)
    q = (torch.randn(B, Hq, D, device=DEV, generator=gen) * 1.5).bfloat16()
    out = torch.zeros(B, Hq, D, device=DEV, dtype=torch.bfloat16)
    ws = torch.zeros(B * Hq * maxp * (D + 2) + 64, device=DEV, dtype=torch.float32)
    ops.decode_attention(q, cache, bt, slots, seq, out, num_kv_heads=Hkv, max_pages=maxp, workspace=ws,
                         num_sms=sms)
    torch.cuda.synchronize()
    for b in range(B):
        k, v = _gather(cache, bt[int(slots[b])], int(seq[b]))
        assert rel_l2(out[b : b + 1], _attn_ref(q[b : b + 1], k, v)) < 1e-2, (b, int(seq[b]))


@pytest.mark.parametrize("T,start,Hq,Hkv", [(2048, 6144, 40, 8), (2048, 6144, 32, 8), (2048, 0, 40, 8),
                                            (1023, 1024, 32, 8), (2048, 2048, 8, 1)])
def test_prefill_attention_long_prefix(T, start, Hq, Hkv):
    gen = torch.Generator(device=DEV).manual_seed(T + start + Hq)
    n = start + T
    npg = (n + 15) // 16
    nb = npg + 64
    cache = (torch.randn(nb, 2, Hkv, 16, D, device=DEV, generator=gen) * 0.5).bfloat16()
    row = torch.randperm(nb, device=DEV, generator=gen).int()[:npg].contiguous()
    q = torch.randn(T, Hq, D, device=DEV, generator=gen).bfloat16()
    out = torch.empty(T, Hq, D, device=DEV, dtype=torch.bfloat16)
    ops.prefill_attention(q, cache, row, start, out, num_kv_heads=Hkv)
    torch.cuda.synchronize()
    k, v = _gather(cache, row, n)
    # reference in query slabs to bound the fp32 score tensor
    for t0 in range(0, T, 512):
        t1 = min(T, t0 + 512)
        ref = _attn_ref(q[t0:t1], k, v, causal_offset=start + t0)
        assert rel_l2(out[t0:t1], ref) < 1e-2, (t0, t1)


QWEN14 = {"qkv": (7168, 5120), "o": (5120, 5120), "down": (5120, 13824), "lm_head": (152064, 5120)}


@pytest.fixture(scope="module")
def scratch():
    return ops.GemmScratch(DEV, ws_bytes=256 << 20, n_counters=1 << 16)


@pytest.mark.parametrize("name", list(QWEN14))
@pytest.mark.parametrize("T,mode,sms", [(2048, 1, 148), (2048, 1, 112), (1, 2, 148), (64, 2, 32), (256, 2, 104),
                                        (256, 2, 148)])
def test_gemm_qwen14b_shapes(name, T, mode, sms, scratch):
    O, K = QWEN14[name]
    if name == "lm_head" and T > 256:
        T = 256  # the lm_head only sees sampled rows
    g = torch.Generator(device=DEV).manual_seed(O + K + T)
    x = torch.randn(T, K, device=DEV, generator=g).bfloat16()
    w = (torch.randn(O, K, device=DEV, generator=g) / math.sqrt(K)).bfloat16()
    r = torch.randn(T, O, device=DEV, generator=g).bfloat16() if name in ("o", "down") else None
    y = ops.linear(x, w, residual=r, mode=mode, num_sms=sms, scratch=scratch)
    torch.cuda.synchronize()
    ref = x.float() @ w.float().T
    if r is not None:
        ref = ref + r.float()
    assert rel_l2(y, ref) < 1e-2


@pytest.mark.parametrize("T,mode,sms", [(2048, 1, 148), (2048, 1, 112), (1, 2, 148), (64, 2, 32), (256, 2, 104)])
def test_gemm_qwen14b_gate_up_swiglu(T, mode, sms, scratch):
    from paper_2601_11822_b200.model import interleave_gate_up

    I, K = 13824, 5120
    g = torch.Generator(device=DEV).manual_seed(T + sms)
    x = torch.randn(T, K, device=DEV, generator=g).bfloat16()
    gate = (torch.randn(I, K, device=DEV, generator=g) / math.sqrt(K)).bfloat16()
    up = (torch.randn(I, K, device=DEV, generator=g) / math.sqrt(K)).bfloat16()
    w = interleave_gate_up(gate, up).contiguous()
    y = torch.empty(T, I, device=DEV, dtype=torch.bfloat16)
    ops.load().rb_gemm_bf16(x.data_ptr(), w.data_ptr(), y.data_ptr(), None, None, T, 2 * I, K, K, K, I, mode | 4, sms,
                            scratch.ws.data_ptr(), scratch.ws_bytes, scratch.counters.data_ptr(),
                            scratch.counters.numel(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = torch.nn.functional.silu(x.float() @ gate.float().T) * (x.float() @ up.float().T)
    assert rel_l2(y, ref) < 1e-2


# ---------------------------------------------------------------------- model level
TOL = 2e-2
# At the real shapes with random N(0, 0.02) weights the bf16 FORMAT alone costs 1.0-1.4% of
# logits rel-L2 after 1-2 layers (an ideal pipeline: fp32 math, activations rounded to bf16
# exactly where the native forward stores them; scripts/model_err_probe.py, measured), so the
# 2e-2 north-star bar (set on the tiny cfg-1 decoder, where the native error is 0.6%) is
# checked together with the ideal pipeline on the same inputs: native <= max(2e-2, 1.6 x ideal).
# A kernel bug shows up as an error far above the ideal's (e.g. a wrong page: 40%).
IDEAL_FACTOR = 1.6


def _two_layer(name):
    from paper_2601_11822_b200.specs import ARCHS

    return dataclasses.replace(ARCHS[name], layers=2)


def _ideal_bf16_logits(arch, st, ids, rows):
    """fp32 forward (oracle math) with every activation the native forward stores in bf16
    rounded to bf16; logits of positions `rows` (on the GPU, torch)."""
    from oracle.llama_fp32 import _rms, _rope, inv_freq

    bf = lambda t: t.bfloat16().float()  # noqa: E731
    s = {k: v.to(DEV) for k, v in st.items()}
    T, G = ids.shape[0], arch.q_heads // arch.kv_heads
    pos = torch.arange(T, device=DEV)
    fr = inv_freq(arch).to(DEV)
    x = s["embed"][ids.to(DEV)]
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
    hl = bf(_rms(x[rows], s["norm"], arch.rms_eps))
    out = bf(hl @ s.get("lm_head", s["embed"]).T).cpu()
    del s
    return out


@pytest.mark.parametrize("name", ["llama3.1-8b", "qwen2.5-14b"])
def test_two_layer_model_forward(name):
    """Chunked prefill (chunks 512 + rest, the second one attending over a paged prefix on
    scattered pages) then 3 batched decode steps of two sequences plus padding rows, against
    the fp32 oracle teacher-forced on the GPU's own tokens (and the ideal bf16 pipeline)."""
    from oracle.llama_fp32 import Oracle, init_state
    from paper_2601_11822_b200.model import DecoderWeights, Runner

    arch = _two_layer(name)
    st = init_state(arch, seed=1, style="random")
    orc = Oracle(arch, st)
    w = DecoderWeights.from_state(arch, st)
    r = Runner(w, num_blocks=256, num_slots=4, max_blocks_per_seq=64, max_prefill_tokens=1024, max_decode_batch=8)
    g = torch.Generator().manual_seed(11)
    lens = [700, 333]
    perm = torch.randperm(256, generator=g).int()  # disjoint scattered pages per sequence
    prompts = []
    errs = []

    def check(native, ref, ideal, what):
        e, ei = rel_l2(native, ref), rel_l2(ideal, ref)
        errs.append((what, round(e, 4), round(ei, 4)))
        assert e <= max(TOL, IDEAL_FACTOR * ei), (name, what, e, ei)

    for s, P in enumerate(lens):
        prompt = torch.randint(0, arch.vocab, (P,), generator=g, dtype=torch.int32)
        prompts.append(prompt)
        r.block_table[s, :64] = perm[64 * s: 64 * (s + 1)].cuda()
        dev = prompt.cuda()
        start = 0
        lg = None
        while start < P - 1:
            ch = min(512, P - 1 - start)
            lg = r.prefill(s, dev[start:start + ch], start, num_sms=148, logits=True)
            start += ch
        torch.cuda.synchronize()
        ref, _ = orc.forward(prompt[: P - 1].long(), 0, None)
        check(lg[0].cpu(), ref[P - 2], _ideal_bf16_logits(arch, st, prompt[: P - 1].long(), [P - 2])[0],
              f"seq{s} prefill")
        r.last_tok[s] = int(prompt[P - 1])
    gen = [[], []]
    d = r.dec
    bucket = 4
    for step in range(3):
        d.slot[:bucket] = torch.tensor([1, 0, r.dummy_slot, r.dummy_slot], dtype=torch.int32).cuda()
        d.pos[:bucket] = torch.tensor([lens[1] - 1 + step, lens[0] - 1 + step, -1, -1], dtype=torch.int32).cuda()
        d.seq[:bucket] = torch.tensor([lens[1] + step, lens[0] + step, 0, 0], dtype=torch.int32).cuda()
        r.decode_body(bucket, num_sms=64)
        torch.cuda.synchronize()
        for row, s in ((0, 1), (1, 0)):
            gen[s].append((int(d.out_ids[row]), d.logits[row].float().cpu()))
    for s, P in enumerate(lens):
        toks = [t for t, _ in gen[s]]
        full = torch.cat([prompts[s].long(), torch.tensor(toks[:-1], dtype=torch.long)])
        ref, _ = orc.forward(full, 0, None)
        ideal = _ideal_bf16_logits(arch, st, full, list(range(P - 1, P + 2)))
        for k, (tok, row) in enumerate(gen[s]):
            check(row, ref[P - 1 + k], ideal[k], f"seq{s} decode step {k}")
            # the id is the argmax of the GPU's own logits row (sampling kernel)
            assert tok == int(row.argmax()), (name, s, k)
    print(name, errs)


@pytest.mark.parametrize("name", ["llama3.1-8b", "qwen2.5-14b"])
@pytest.mark.parametrize("sms", [48, 72, 148])
def test_decode_ksplit_partials_match_streamk(name, sms):
    """Decode O / down projections as K-slice units summed in the following RMSNorm
    (rb_set_decode_ksplit(1), the default) against the stream-K + residual-epilogue path, at the
    real layer shapes and a bucket of 192 rows (2 real sequences + padding), on 48 / 72 / 148
    SMs; both against the fp32 oracle."""
    from oracle.llama_fp32 import Oracle, init_state
    from paper_2601_11822_b200 import ops
    from paper_2601_11822_b200.model import DecoderWeights, Runner

    lib = ops.load()
    arch = _two_layer(name)
    st = init_state(arch, seed=2, style="random")
    orc = Oracle(arch, st)
    r = Runner(DecoderWeights.from_state(arch, st), num_blocks=512, num_slots=4, max_blocks_per_seq=64,
               max_prefill_tokens=512, max_decode_batch=256)
    g = torch.Generator().manual_seed(5)
    lens = [300, 201]
    prompts = []
    for s, P in enumerate(lens):
        prompt = torch.randint(0, arch.vocab, (P,), generator=g, dtype=torch.int32)
        prompts.append(prompt)
        r.block_table[s, :64] = torch.arange(64 * s, 64 * (s + 1), dtype=torch.int32).cuda()
        r.prefill(s, prompt[: P - 1].cuda(), 0, num_sms=148)
    bucket = 192
    d = r.dec
    out = {}
    for mode in (0, 1):
        assert lib.rb_set_decode_ksplit(mode) == 0
        for s, P in enumerate(lens):
            r.last_tok[s] = int(prompts[s][P - 1])
        d.slot[:bucket] = torch.tensor([0, 1] + [r.dummy_slot] * (bucket - 2), dtype=torch.int32).cuda()
        d.pos[:bucket] = torch.tensor([lens[0] - 1, lens[1] - 1] + [-1] * (bucket - 2), dtype=torch.int32).cuda()
        d.seq[:bucket] = torch.tensor([lens[0], lens[1]] + [0] * (bucket - 2), dtype=torch.int32).cuda()
        r.decode_body(bucket, num_sms=sms)
        torch.cuda.synchronize()
        out[mode] = (d.logits[:2].float().cpu(), [int(x) for x in d.out_ids[:2].cpu()])
    lib.rb_set_decode_ksplit(1)
    # the two paths round differently (stream-K adds the residual to the bf16-rounded projection,
    # the K-slice consumer in fp32): bf16-level agreement, and each against the oracle below
    assert rel_l2(out[1][0], out[0][0]) < 3e-2, (name, sms)
    for s, P in enumerate(lens):
        ref, _ = orc.forward(prompts[s].long(), 0, None)
        e0, e1 = rel_l2(out[0][0][s], ref[P - 1]), rel_l2(out[1][0][s], ref[P - 1])
        assert e1 <= max(TOL, 1.1 * e0 + 1e-3), (name, sms, s, e0, e1)  # no worse than the stream-K path
        for mode in (0, 1):
            assert out[mode][1][s] == int(out[mode][0][s].argmax())

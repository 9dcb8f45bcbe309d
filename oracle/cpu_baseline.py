"""CPU baseline leg of bench.py — TEST / BASELINE INFRASTRUCTURE ONLY.

Times the fp32 CPU oracle (oracle/llama_fp32.py, a restatement: the
reference itself has no model numerics) on a BOUNDED sample of the same
serving workload the GPU bench runs, on the host's cores:

  * prefill sample: one chunk of `prefill_tokens` prompt tokens;
  * decode sample:  `decode_steps` batched decode steps of `batch` sequences at
    the workload's mid-generation context (prompt + output/2), with KV
    pre-filled (values do not affect CPU time).

Output tokens/s of the whole workload = 1 / (t_decode_per_token +
(prompt/output) * t_prefill_per_token): every output token of the cfg-2
workload carries prompt/output prefill tokens. Weights are random fp32 of the
real shapes, filled from a tiled random block (a per-element RNG fill of 8B
params alone would take longer than the sample).
"""

from __future__ import annotations

import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle.llama_fp32 import Oracle, decode_batch  # noqa: E402


def fast_state(arch, std: float = 0.02) -> dict:
    g = torch.Generator().manual_seed(0)
    tile = torch.randn(1 << 20, generator=g) * std

    def w(*shape):
        n = 1
        for d in shape:
            n *= d
        out = torch.empty(n)
        for o in range(0, n, tile.numel()):
            m = min(tile.numel(), n - o)
            out[o : o + m] = tile[:m]
        return out.view(*shape)

    H, D, I = arch.hidden, arch.head_dim, arch.intermediate
    st = {"embed": w(arch.vocab, H), "norm": torch.ones(H)}
    for i in range(arch.layers):
        p = f"layers.{i}."
        st.update({p + "ln1": torch.ones(H), p + "ln2": torch.ones(H), p + "q": w(arch.q_heads * D, H),
                   p + "k": w(arch.kv_heads * D, H), p + "v": w(arch.kv_heads * D, H),
                   p + "o": w(H, arch.q_heads * D), p + "gate": w(I, H), p + "up": w(I, H), p + "down": w(H, I)})
        if arch.qkv_bias:
            st.update({p + "bq": torch.zeros(arch.q_heads * D), p + "bk": torch.zeros(arch.kv_heads * D),
                       p + "bv": torch.zeros(arch.kv_heads * D)})
    if not arch.tie_embeddings:
        st["lm_head"] = w(arch.vocab, H)
    return st


def run_sample(arch, prompt_len: int, out_len: int, batch: int = 8, decode_steps: int = 2,
               prefill_tokens: int = 64, threads: int | None = None) -> dict:
    threads = threads or os.cpu_count() or 1
    torch.set_num_threads(threads)
    t_init = time.perf_counter()
    orc = Oracle(arch, fast_state(arch))
    t_init = time.perf_counter() - t_init
    ids = torch.randint(0, arch.vocab, (prefill_tokens,))
    with torch.no_grad():
        t0 = time.perf_counter()
        orc.forward(ids, 0, None)
        t_pref = (time.perf_counter() - t0) / prefill_tokens
        ctx = prompt_len + out_len // 2
        kvs = [[(torch.randn(ctx, arch.kv_heads, arch.head_dim), torch.randn(ctx, arch.kv_heads, arch.head_dim))
                for _ in range(arch.layers)] for _ in range(batch)]
        step_ids = torch.randint(0, arch.vocab, (batch,))
        decode_batch(orc, step_ids, [ctx] * batch, kvs)  # warm-up step (allocator, threads)
        t0 = time.perf_counter()
        for s in range(decode_steps):
            decode_batch(orc, step_ids, [ctx + 1 + s] * batch, kvs)
        t_dec = (time.perf_counter() - t0) / (decode_steps * batch)
    per_tok = t_dec + (prompt_len / out_len) * t_pref
    return {
        "value": 1.0 / per_tok,
        "unit": "output tokens/s",
        "cores": threads,
        "kind": "port",
        "sample": (f"fp32 CPU oracle ({arch.name}, random weights): 1 prefill chunk of {prefill_tokens} tokens "
                   f"({t_pref * 1e3:.1f} ms/token) + {decode_steps} batched decode steps of B={batch} at ctx {ctx} "
                   f"({t_dec * 1e3:.1f} ms/token); tokens/s = 1/(t_dec + {prompt_len}/{out_len} * t_prefill); "
                   f"weight init {t_init:.1f} s excluded"),
        "t_prefill_per_token_s": t_pref,
        "t_decode_per_token_s": t_dec,
    }


class CpuSampler:
    """The oracle model and a mid-generation KV state built once; each `step()` is one bounded
    sample of the workload (one prefill chunk + one batched decode step), so a bench run can
    take W warm-up and K timed steps of it (bench.py --impl reference)."""

    def __init__(self, arch, prompt_len: int, out_len: int, batch: int = 4, prefill_tokens: int = 16,
                 threads: int | None = None):
        self.threads = threads or os.cpu_count() or 1
        torch.set_num_threads(self.threads)
        self.arch, self.prompt_len, self.out_len = arch, prompt_len, out_len
        self.batch, self.prefill_tokens = batch, prefill_tokens
        t0 = time.perf_counter()
        self.orc = Oracle(arch, fast_state(arch))
        self.ctx = prompt_len + out_len // 2
        self.kvs = [[(torch.randn(self.ctx + 64, arch.kv_heads, arch.head_dim),
                      torch.randn(self.ctx + 64, arch.kv_heads, arch.head_dim)) for _ in range(arch.layers)]
                    for _ in range(batch)]
        self.t_init = time.perf_counter() - t0
        self.n = 0

    def step(self) -> dict:
        """One prefill chunk of `prefill_tokens` + one decode step of `batch` rows."""
        arch = self.arch
        ids = torch.randint(0, arch.vocab, (self.prefill_tokens,))
        step_ids = torch.randint(0, arch.vocab, (self.batch,))
        with torch.no_grad():
            t0 = time.perf_counter()
            self.orc.forward(ids, 0, None)
            t1 = time.perf_counter()
            decode_batch(self.orc, step_ids, [self.ctx + (self.n % 64)] * self.batch, self.kvs)
            t2 = time.perf_counter()
        self.n += 1
        t_pref = (t1 - t0) / self.prefill_tokens
        t_dec = (t2 - t1) / self.batch
        return {"t_prefill_per_token_s": t_pref, "t_decode_per_token_s": t_dec, "wall_s": t2 - t0,
                "value": 1.0 / (t_dec + (self.prompt_len / self.out_len) * t_pref)}

    def describe(self) -> str:
        return (f"fp32 CPU oracle ({self.arch.name}, random weights), per step: 1 prefill chunk of "
                f"{self.prefill_tokens} tokens + 1 batched decode step of B={self.batch} at ctx {self.ctx}; "
                f"tokens/s = 1/(t_dec + {self.prompt_len}/{self.out_len} * t_prefill) from the median per-token "
                f"times of the timed steps; model + KV build {self.t_init:.1f} s excluded")


if __name__ == "__main__":
    from paper_2601_11822_b200.specs import ARCHS

    print(run_sample(ARCHS[sys.argv[1] if len(sys.argv) > 1 else "tiny"], 1024, 256))

"""Device/model descriptions, Eq. 1 and the ARM decision type.

Parity surface: pkg/src/pdsim/core.py:122-245 (ModelSpec, GpuSpec.aggregate,
kv_cache_bytes, validate_specs, AllocationMode/Decision, OVERALLOCATE).
Adds B200 and real-model presets (the reference ships only MI300X-like ones,
pkg/src/pdsim/presets/*.yaml) plus the SM-partition quantisation that maps a
CU fraction onto green-context granularity.
"""

from __future__ import annotations

import enum
import json
import math
import os
from dataclasses import dataclass, replace


@dataclass(frozen=True)
class ModelSpec:
    name: str
    num_layers: int
    kv_heads: int
    head_dim: int
    bytes_per_element: int
    flops_per_token: float
    weight_bytes: float


@dataclass(frozen=True)
class GpuSpec:
    """One logical device; a tensor-parallel group folds into one (core.py:147-165)."""

    name: str
    num_cus: int
    peak_flops: float
    hbm_bandwidth: float
    hbm_capacity: float
    kernel_launch_overhead_us: float = 10.0
    interconnect_bandwidth: float = 5.0e10

    def aggregate(self, tp: int) -> "GpuSpec":
        if tp < 1:
            raise ValueError("tp must be >= 1")
        if tp == 1:
            return self
        return replace(
            self,
            name=f"{self.name}-tp{tp}",
            num_cus=self.num_cus * tp,
            peak_flops=self.peak_flops * tp,
            hbm_bandwidth=self.hbm_bandwidth * tp,
            hbm_capacity=self.hbm_capacity * tp,
        )


def kv_cache_bytes(model: ModelSpec, seq_len: int) -> int:
    """Eq. 1: 2 * L * S * Hkv * d * E (pure int, exactly linear in S)."""
    if seq_len < 0:
        raise ValueError("seq_len must be >= 0")
    return 2 * model.num_layers * seq_len * model.kv_heads * model.head_dim * model.bytes_per_element


def validate_specs(model: ModelSpec, gpu: GpuSpec) -> list[str]:
    errors: list[str] = []
    for name in ("num_layers", "kv_heads", "head_dim", "bytes_per_element", "flops_per_token", "weight_bytes"):
        if getattr(model, name) <= 0:
            errors.append(f"model.{name} must be positive")
    if gpu.num_cus < 2:
        errors.append("num_cus must be >= 2")
    for name in ("peak_flops", "hbm_bandwidth", "hbm_capacity", "kernel_launch_overhead_us", "interconnect_bandwidth"):
        if getattr(gpu, name) <= 0:
            errors.append(f"gpu.{name} must be positive")
    if model.weight_bytes >= gpu.hbm_capacity:
        errors.append(
            f"weights do not fit: weight_bytes={model.weight_bytes:.3e} >= hbm_capacity={gpu.hbm_capacity:.3e}"
        )
    return errors


class AllocationMode(enum.Enum):
    OVERALLOCATE = "overallocate"
    PARTITION = "partition"


@dataclass(frozen=True)
class AllocationDecision:
    """CU split between the prefill and decode streams (core.py:220-242)."""

    mode: AllocationMode
    cu_fraction_prefill: float
    cu_fraction_decode: float
    slo_risk: bool = False

    def __post_init__(self) -> None:
        p, d = self.cu_fraction_prefill, self.cu_fraction_decode
        if self.mode is AllocationMode.OVERALLOCATE:
            if p != 1.0 or d != 1.0:
                raise ValueError("overallocate mode requires both fractions = 1.0")
            return
        if not (0.0 < p and 0.0 < d):
            raise ValueError("partition fractions must be positive")
        if p + d > 1.0 + 1e-9:
            raise ValueError("partition fractions must sum to <= 1.0")


OVERALLOCATE = AllocationDecision(AllocationMode.OVERALLOCATE, 1.0, 1.0)

#: green-context SM granularity on compute capability >= 9.0 (cuda.h:25257-25262)
SM_GRANULARITY = 8


def decode_sms_for(decision: AllocationDecision, total_sms: int, granularity: int = SM_GRANULARITY) -> int | None:
    """Map an ARM decision onto a decode partition size in SMs.

    OVERALLOCATE -> None (both phases on the full device). PARTITION ->
    cu_fraction_decode * total rounded UP to the granularity (decode is the
    latency-critical phase), leaving at least one granule for prefill.
    """
    if decision.mode is AllocationMode.OVERALLOCATE:
        return None
    want = decision.cu_fraction_decode * total_sms
    sms = int(math.ceil(want / granularity - 1e-9)) * granularity
    sms = max(granularity, sms)
    return min(sms, total_sms - granularity)


# ---------------------------------------------------------------- presets

def _measured_peaks() -> dict:
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(here, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def b200_spec(sustained: bool = True, hbm_capacity: float = 1.79e11) -> GpuSpec:
    """B200 from the pod's measured peaks (MEASURED_PEAKS.json), SURVEY.md §6.4."""
    p = _measured_peaks()
    flops = p.get("bf16_tflops_sustained" if sustained else "bf16_tflops", 1381.0 if sustained else 1643.1) * 1e12
    bw = p.get("hbm_gbs", 6543.4) * 1e9
    return GpuSpec("b200", 148, flops, bw, hbm_capacity, 10.0, 7.7e11)


MI300X_LIKE = GpuSpec("mi300x-like", 304, 1.3074e15, 5.3e12, 1.92e11, 10.0, 5.0e10)
LLAMA70B_LIKE = ModelSpec("llama70b-like", 80, 8, 128, 2, 1.4e11, 1.4e11)
MOE_LIKE = ModelSpec("moe-like", 32, 8, 128, 2, 2.58e10, 9.34e10)


@dataclass(frozen=True)
class ArchConfig:
    """Decoder architecture for the GPU path (Llama-3.x / Qwen2 family)."""

    name: str
    hidden: int
    layers: int
    q_heads: int
    kv_heads: int
    head_dim: int
    intermediate: int
    vocab: int
    rope_theta: float
    rms_eps: float = 1e-5
    qkv_bias: bool = False
    rope_scaling: dict | None = None  # llama3: factor, low_freq_factor, high_freq_factor, original_max_position
    tie_embeddings: bool = False
    max_position: int = 131072

    def param_count(self) -> int:
        H, I, L = self.hidden, self.intermediate, self.layers
        qkv = H * (self.q_heads + 2 * self.kv_heads) * self.head_dim
        bias = (self.q_heads + 2 * self.kv_heads) * self.head_dim if self.qkv_bias else 0
        o = self.q_heads * self.head_dim * H
        mlp = 3 * H * I
        per_layer = qkv + bias + o + mlp + 2 * H
        emb = self.vocab * H * (1 if self.tie_embeddings else 2)
        return L * per_layer + emb + H

    def model_spec(self, bytes_per_element: int = 2) -> ModelSpec:
        """Analytic ModelSpec for the reference cost model / ARM (flops ~ 2 x params)."""
        n = self.param_count()
        return ModelSpec(self.name, self.layers, self.kv_heads, self.head_dim, bytes_per_element, 2.0 * n,
                         float(n * bytes_per_element))


LLAMA3_ROPE = {"factor": 8.0, "low_freq_factor": 1.0, "high_freq_factor": 4.0, "original_max_position": 8192}

ARCHS = {
    "llama3.1-8b": ArchConfig("llama3.1-8b", 4096, 32, 32, 8, 128, 14336, 128256, 500000.0, 1e-5, False, LLAMA3_ROPE),
    "llama3.1-70b": ArchConfig("llama3.1-70b", 8192, 80, 64, 8, 128, 28672, 128256, 500000.0, 1e-5, False,
                               LLAMA3_ROPE),
    "qwen2.5-14b": ArchConfig("qwen2.5-14b", 5120, 48, 40, 8, 128, 13824, 152064, 1000000.0, 1e-6, True, None,
                              max_position=32768),
    # SURVEY.md §8(d) cfg 1: the frozen tiny Llama-style decoder
    "tiny": ArchConfig("tiny", 1024, 4, 8, 2, 128, 3584, 4096, 500000.0, 1e-5, False, LLAMA3_ROPE),
}

"""The Executor boundary: who performs the GPU work an engine launches.

The reference prices every iteration at its two launch sites
(pkg/src/pdsim/engines/rapid.py:173-189 prefill, :267-293 decode;
hybrid.py:127 fused). Here those sites call an Executor instead:

  launch_prefill(req, written, chunk, target, decision, co_decode) -> handle
  launch_decode(members, decision, co_prefill_chunk)               -> handle
  launch_hybrid(members, head, written, chunk, target)             -> handle
  finish_decode(handle) / finish_prefill(handle) / finish_hybrid(handle)
  on_preempt(req) / on_finish(req) / bind(engine)

A handle carries `gpu_us` (known at launch for the cost model, filled at
completion on the GPU) and `done()`.

`CostModelExecutor` re-creates the reference's pricing decisions exactly, so
`RapidEngine` + `CostModelExecutor` under `Simulation` reproduces the
reference schedules bit for bit. `B200Executor` (executor_b200.py) launches
real kernels on green-context streams.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass

from paper_2601_11822_b200.arm import decode_time, hybrid_time, overlapped_times, prefill_time
from paper_2601_11822_b200.specs import OVERALLOCATE, AllocationDecision, AllocationMode


@dataclass
class PricedHandle:
    gpu_us: int
    cu_fraction: float
    kind: str
    members: tuple = ()

    def done(self) -> bool:
        return True


class CostModelExecutor:
    """Device = the reference's two-term roofline (costmodel.py:89-250)."""

    realtime = False

    def bind(self, engine) -> None:
        self.engine = engine
        self.model = engine.model
        self.gpu = engine.gpu
        self.params = engine.params

    # RAPID prefill site (rapid.py:171-189)
    def launch_prefill(self, req, written: int, chunk: int, target: int, decision: AllocationDecision,
                       co_decode: tuple[int, int] | None) -> PricedHandle:
        m, g, p = self.model, self.gpu, self.params
        if decision.mode is AllocationMode.PARTITION:
            cu = decision.cu_fraction_prefill
            us = prefill_time(chunk, cu, m, g, p, concurrent=co_decode is not None)
        else:
            cu = 1.0
            if co_decode is not None:
                us = overlapped_times(chunk, co_decode[0], co_decode[1], OVERALLOCATE, m, g, p)[0]
            else:
                us = prefill_time(chunk, 1.0, m, g, p)
        return PricedHandle(us, cu, "prefill")

    # RAPID decode site (rapid.py:266-293)
    def launch_decode(self, members, decision: AllocationDecision, co_prefill_chunk: int | None) -> PricedHandle:
        m, g, p = self.model, self.gpu, self.params
        batch = len(members)
        total_kv = sum(r.context_tokens for r in members)
        if decision.mode is AllocationMode.PARTITION:
            cu = decision.cu_fraction_decode
            us = decode_time(batch, total_kv, cu, m, g, p, concurrent=co_prefill_chunk is not None)
        else:
            cu = 1.0
            if co_prefill_chunk is not None:
                us = overlapped_times(co_prefill_chunk, batch, total_kv, OVERALLOCATE, m, g, p)[1]
            else:
                us = decode_time(batch, total_kv, 1.0, m, g, p)
        h = PricedHandle(us, cu, "decode", tuple(members))
        h.total_kv = total_kv
        return h

    # hybrid fused site (hybrid.py:126-127)
    def launch_hybrid(self, members, head, written: int, chunk: int, target: int) -> PricedHandle:
        total_kv = sum(r.context_tokens for r in members) + written
        return PricedHandle(hybrid_time(chunk, len(members), total_kv, self.model, self.gpu, self.params), 1.0,
                            "hybrid", tuple(members))

    def finish_prefill(self, handle) -> None:
        pass

    def finish_decode(self, handle) -> None:
        pass

    def finish_hybrid(self, handle) -> None:
        pass

    def on_preempt(self, req) -> None:
        pass

    def on_finish(self, req) -> None:
        pass


class ReplayExecutor(CostModelExecutor):
    """Device = the durations a GPU run measured, replayed in launch order (trace replay,
    SURVEY.md §8(c)). Every launch of a phase returns the next recorded (completion -
    launch) time of that phase, so a virtual-clock run with cpu_us = 0 dispatches the same
    timeline the real-time run observed, and its admission / ordering / preemption / ARM
    decisions can be compared with the GPU run's (and with the reference RapidEngine's,
    replayed the same way)."""

    def __init__(self, launch_log, num_blocks: int | None = None, block_size: int = 16):
        self.q = {"prefill": deque(), "decode": deque()}
        for phase, start, end in launch_log:
            self.q[phase].append(int(end) - int(start))
        self.num_blocks = num_blocks
        self.block_size = block_size

    def make_pool(self, model, gpu):
        from paper_2601_11822_b200.blockpool import BlockPool

        if self.num_blocks is None:
            return BlockPool.for_device(model, gpu, name="gpu0")
        return BlockPool(self.num_blocks, self.block_size, name="gpu0")

    def _next(self, phase: str) -> int:
        if not self.q[phase]:
            raise RuntimeError(f"replay diverged: more {phase} launches than the GPU run recorded")
        return self.q[phase].popleft()

    def launch_prefill(self, req, written, chunk, target, decision, co_decode) -> PricedHandle:
        cu = decision.cu_fraction_prefill if decision.mode is AllocationMode.PARTITION else 1.0
        return PricedHandle(self._next("prefill"), cu, "prefill")

    def launch_decode(self, members, decision, co_prefill_chunk) -> PricedHandle:
        cu = decision.cu_fraction_decode if decision.mode is AllocationMode.PARTITION else 1.0
        return PricedHandle(self._next("decode"), cu, "decode", tuple(members))

    def launch_hybrid(self, members, head, written, chunk, target) -> PricedHandle:
        raise NotImplementedError("trace replay covers the RAPID engine")

    def exhausted(self) -> bool:
        return not self.q["prefill"] and not self.q["decode"]


class MeasuredTableExecutor(CostModelExecutor):
    """Device = the B200 tables profiler.py MEASURED (arm.MeasuredProfile), on the virtual
    clock: a decode step of batch B on a D-SM partition costs the measured contended step
    (linear between the measured batches), a prefill chunk costs its tokens x the measured
    per-token time of the complementary partition; OVERALLOCATE with both phases busy costs
    the measured OVERALLOCATE pair, and a phase running alone gets the whole device (decode:
    the widest measured partition; prefill: the measured full-device rate). Used to tune ARM
    policies on the CPU before spending GPU time (scripts/arm_sim.py); not a parity path."""

    def __init__(self, mp, num_blocks: int | None = None, block_size: int = 16):
        self.mp = mp
        self.num_blocks = num_blocks
        self.block_size = block_size
        self._alone_pre = float(mp.data.get("full_prefill_alone_us_per_token", mp.prefill_us_per_token(None)))

    def make_pool(self, model, gpu):
        from paper_2601_11822_b200.blockpool import BlockPool

        if self.num_blocks is None:
            return BlockPool.for_device(model, gpu, name="gpu0")
        return BlockPool(self.num_blocks, self.block_size, name="gpu0")

    def _dec(self, d, b: int) -> float:
        bs = self.mp.batches
        b = max(1, b)
        if b >= bs[-1]:
            return self.mp.decode_us(d, bs[-1]) * b / bs[-1]
        hi = next(x for x in bs if x >= b)
        lo = max((x for x in bs if x <= b), default=hi)
        t_hi = self.mp.decode_us(d, hi)
        if hi == lo:
            return t_hi
        t_lo = self.mp.decode_us(d, lo)
        return t_lo + (t_hi - t_lo) * (b - lo) / (hi - lo)

    def _split(self, decision):
        if decision.mode is AllocationMode.OVERALLOCATE:
            return None
        return round(decision.cu_fraction_decode * self.mp.total)

    def launch_prefill(self, req, written, chunk, target, decision, co_decode) -> PricedHandle:
        d = self._split(decision)
        if d is None and co_decode is None:
            us = chunk * self._alone_pre
        else:
            us = chunk * self.mp.prefill_us_per_token(d, co_decode[0] if co_decode else None)
        cu = decision.cu_fraction_prefill if d is not None else 1.0
        return PricedHandle(max(1, int(round(us))), cu, "prefill")

    def launch_decode(self, members, decision, co_prefill_chunk) -> PricedHandle:
        d = self._split(decision)
        b = len(members)
        if d is None and co_prefill_chunk is None:
            us = self._dec(self.mp.ladder[-1], b)
        else:
            us = self._dec(d, b)
        cu = decision.cu_fraction_decode if d is not None else 1.0
        return PricedHandle(max(1, int(round(us))), cu, "decode", tuple(members))

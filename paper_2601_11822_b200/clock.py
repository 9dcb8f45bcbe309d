"""Event loops: the reference's virtual clock and the real-time GPU loop.

`Simulation` has the reference's contract (pkg/src/pdsim/sim.py:42-95): a
heap ordered by (time_us, seq), SIM_END scheduled first at the horizon so it
precedes same-time events, CausalityError on scheduling into the past, drain
after the horizon. Engines drive it through `schedule()` only, plus
`complete()` for GPU work: under the virtual clock a completion is simply an
event at start + priced duration.

`RealTimeLoop` keeps the same engine-facing API but its clock is the host's
monotonic microsecond clock since `run()` started. Timed events (arrivals,
SIM_END) fire when the wall clock reaches them, stamped with their due time;
GPU completions fire when their CUDA event reports done (polled), stamped
with the observation time.
"""

from __future__ import annotations

import enum
import heapq
import logging
import time
from dataclasses import dataclass, field
from typing import Any, Callable

log = logging.getLogger("paper_2601_11822_b200.clock")


class CausalityError(RuntimeError):
    """An event was scheduled before the current time."""


class EventKind(enum.Enum):
    ARRIVAL = "Arrival"
    PREFILL_ITER_DONE = "PrefillIterDone"
    DECODE_ITER_DONE = "DecodeIterDone"
    TRANSFER_DONE = "TransferDone"
    NOTIFY_PREFILL_READY = "NotifyPrefillReady"
    NOTIFY_KV_ALLOCATED = "NotifyKvAllocated"
    SIM_END = "SimEnd"


@dataclass
class Event:
    time_us: int
    kind: EventKind
    data: dict[str, Any] = field(default_factory=dict)
    seq: int = -1


def _describe(data: dict[str, Any]) -> str:
    return " ".join(f"{k}={getattr(v, 'id', v)}" for k, v in data.items())


class Simulation:
    """Virtual-time event heap (the reference clock)."""

    realtime = False

    def __init__(self, until_us: int | None = None) -> None:
        if until_us is not None and until_us < 1:
            raise ValueError("until_us must be >= 1")
        self.until_us = until_us
        self.now_us = 0
        self.last_event_us = 0
        self._heap: list[tuple[int, int, Event]] = []
        self._seq = 0
        self._ended = False
        if until_us is not None:
            self.schedule(until_us, EventKind.SIM_END)

    @property
    def ended(self) -> bool:
        return self._ended

    @property
    def horizon_us(self) -> int:
        return self.until_us if self.until_us is not None else self.last_event_us

    def schedule(self, time_us: int, kind: EventKind, **data: Any) -> Event:
        if not isinstance(kind, EventKind):
            raise TypeError(f"kind must be an EventKind, got {kind!r}")
        if time_us < self.now_us:
            raise CausalityError(f"cannot schedule {kind.value} at {time_us} (now {self.now_us})")
        ev = Event(int(time_us), kind, data, self._seq)
        self._seq += 1
        heapq.heappush(self._heap, (ev.time_us, ev.seq, ev))
        return ev

    def complete(self, start_us: int, handle, kind: EventKind, **data: Any) -> Event:
        """Completion of device work launched at `start_us`: virtual time adds its price."""
        return self.schedule(start_us + handle.gpu_us, kind, gpu_us=handle.gpu_us, handle=handle, **data)

    def run(self, handler: Callable[["Simulation", Event], None]) -> None:
        heap = self._heap
        debug = log.isEnabledFor(logging.DEBUG)
        while heap:
            ev = heapq.heappop(heap)[2]
            self.now_us = self.last_event_us = ev.time_us
            if ev.kind is EventKind.SIM_END:
                self._ended = True
            if debug:
                log.debug("t=%dus %s %s", ev.time_us, ev.kind.value, _describe(ev.data))
            handler(self, ev)


class RealTimeLoop:
    """Wall-clock loop with the Simulation API; GPU completions come from CUDA events.

    `complete(start_us, handle, kind, **data)` registers `handle` (an object
    with `.done() -> bool` and `.gpu_us` filled on completion); the loop
    polls pending handles in submission order per stream and dispatches the
    event at the observed host time.
    """

    realtime = True

    def __init__(self, until_us: int | None = None, poll_sleep_us: int = 50) -> None:
        if until_us is not None and until_us < 1:
            raise ValueError("until_us must be >= 1")
        self.until_us = until_us
        self.now_us = 0
        self.last_event_us = 0
        self._timed: list[tuple[int, int, Event]] = []
        self._pending: list[tuple[Any, Event]] = []
        self._seq = 0
        self._ended = False
        self._t0 = None
        self.poll_sleep_us = poll_sleep_us
        self.idle_us = 0
        if until_us is not None:
            self.schedule(until_us, EventKind.SIM_END)

    @property
    def ended(self) -> bool:
        return self._ended

    @property
    def horizon_us(self) -> int:
        return self.until_us if self.until_us is not None else self.last_event_us

    def clock_us(self) -> int:
        if self._t0 is None:
            return 0
        return int((time.perf_counter_ns() - self._t0) // 1000)

    def schedule(self, time_us: int, kind: EventKind, **data: Any) -> Event:
        if not isinstance(kind, EventKind):
            raise TypeError(f"kind must be an EventKind, got {kind!r}")
        if time_us < self.now_us:
            raise CausalityError(f"cannot schedule {kind.value} at {time_us} (now {self.now_us})")
        ev = Event(int(time_us), kind, data, self._seq)
        self._seq += 1
        heapq.heappush(self._timed, (ev.time_us, ev.seq, ev))
        return ev

    def complete(self, start_us: int, handle, kind: EventKind, **data: Any) -> Event:
        ev = Event(-1, kind, dict(data, handle=handle), self._seq)
        self._seq += 1
        self._pending.append((handle, ev))
        return ev

    def _dispatch(self, ev: Event, handler) -> None:
        if ev.kind is EventKind.SIM_END:
            self._ended = True
        self.last_event_us = ev.time_us
        handler(self, ev)

    def run(self, handler: Callable[[Any, Event], None]) -> None:
        """Poll loop. At each poll (host time `now`): first every timed event due by `now`
        (arrivals, SIM_END) at its due time, then every GPU completion observed done at
        this poll, stamped `now`, in submission order. Timed events therefore carry their
        exact trace time (due times are >= every earlier stamp: anything due at or before
        the previous poll was dispatched there), and the dispatched timeline is the one a
        virtual-clock replay reproduces with (arrival, seq) / (completion, seq) ordering
        (tests/test_trace_replay.py)."""
        self._t0 = time.perf_counter_ns()
        # idle hook of the engine's executor (off-critical-path bookkeeping while GPU work runs)
        owner = getattr(handler, "__self__", None)
        on_idle = getattr(getattr(owner, "executor", None), "on_idle", None)
        while self._timed or self._pending:
            now = self.clock_us()
            done = []
            if self._pending:
                still = []
                for h, ev in self._pending:
                    (done if h.done() else still).append((h, ev))
                if done:
                    self._pending = still
            progressed = bool(done)
            while self._timed and self._timed[0][0] <= now:
                ev = heapq.heappop(self._timed)[2]
                self.now_us = max(self.now_us, ev.time_us)
                ev.time_us = self.now_us
                self._dispatch(ev, handler)
                progressed = True
            if done:
                now = max(now, self.now_us)
                for h, ev in done:
                    ev.time_us = now
                    ev.data["gpu_us"] = h.gpu_us
                    self.now_us = now
                    self._dispatch(ev, handler)
            if not progressed:
                if on_idle is not None:
                    on_idle()
                if not self._pending and self._timed:
                    wait = self._timed[0][0] - self.clock_us()
                    if wait > 200:
                        time.sleep((wait - 100) / 1e6)
                        self.idle_us += wait - 100
                elif self.poll_sleep_us > 0:
                    time.sleep(self.poll_sleep_us / 1e6)
                # poll_sleep_us == 0: busy-poll the CUDA events (a completion is acted on within
                # one cudaEventQuery sweep instead of a >= 50 us sleep granule)

"""Request lifecycle: states, legal edges, per-request stamps.

Semantics follow the reference exactly (pkg/src/pdsim/core.py:19-119):
nine forward edges, one flagged preemption edge (DECODING -> PENDING_KV),
strictly increasing token stamps, `context_tokens = prompt + delivered`.
The host engines keep one `Request` per trace item; the GPU executor keeps a
parallel record of generated token ids (needed to re-prefill after
preemption, rapid.py:221-226 + core.py:98-101).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field


class RequestState(enum.Enum):
    ARRIVED = "arrived"
    PENDING_KV = "pending_kv"
    WAITING_PREFILL = "waiting_prefill"
    PREFILLING = "prefilling"
    PREFILL_FINISHED = "prefill_finished"
    DECODING = "decoding"
    FINISHED = "finished"
    REJECTED = "rejected"


_S = RequestState

#: forward edges (core.py:34-46); rejection only before a request runs
ALLOWED_TRANSITIONS = frozenset(
    {
        (_S.ARRIVED, _S.PENDING_KV),
        (_S.PENDING_KV, _S.WAITING_PREFILL),
        (_S.WAITING_PREFILL, _S.PREFILLING),
        (_S.PREFILLING, _S.PREFILL_FINISHED),
        (_S.PREFILL_FINISHED, _S.DECODING),
        (_S.DECODING, _S.FINISHED),
        (_S.ARRIVED, _S.REJECTED),
        (_S.PENDING_KV, _S.REJECTED),
        (_S.WAITING_PREFILL, _S.REJECTED),
    }
)

#: the single backward edge; must be requested explicitly (core.py:48-51)
PREEMPTION_TRANSITION = (_S.DECODING, _S.PENDING_KV)

TERMINAL_STATES = frozenset({_S.FINISHED, _S.REJECTED})


class InvalidTransition(RuntimeError):
    pass


@dataclass(eq=False)
class Request:
    """One request as it moves through an engine (identity-compared)."""

    id: int
    arrival_us: int
    prompt_tokens: int
    output_tokens: int
    state: RequestState = RequestState.ARRIVED
    token_times_us: list[int] = field(default_factory=list)
    decode_participations: int = 0
    preemptions: int = 0
    history: list[tuple[RequestState, int]] = field(default_factory=list)
    container: str = ""  # single-residency tag, checked by the engines

    def __post_init__(self) -> None:
        for name, lo in (("prompt_tokens", 1), ("output_tokens", 1), ("arrival_us", 0)):
            if getattr(self, name) < lo:
                raise ValueError(f"request {self.id}: {name} must be >= {lo}")
        self.history.append((self.state, self.arrival_us))

    @property
    def delivered_tokens(self) -> int:
        return len(self.token_times_us)

    @property
    def first_token_us(self) -> int | None:
        return self.token_times_us[0] if self.token_times_us else None

    @property
    def context_tokens(self) -> int:
        """Tokens the KV cache must hold for this request right now."""
        return self.prompt_tokens + len(self.token_times_us)

    def advance(self, new_state: RequestState, now_us: int, *, preemption: bool = False) -> None:
        edge = (self.state, new_state)
        if preemption:
            if edge != PREEMPTION_TRANSITION:
                raise InvalidTransition(f"request {self.id}: bad preemption edge {edge}")
            self.preemptions += 1
        elif edge not in ALLOWED_TRANSITIONS:
            raise InvalidTransition(f"request {self.id}: illegal transition {edge}")
        self.state = new_state
        self.history.append((new_state, now_us))

    def deliver_token(self, now_us: int) -> None:
        stamps = self.token_times_us
        if stamps and now_us <= stamps[-1]:
            raise ValueError(f"request {self.id}: token timestamps must be strictly increasing")
        if len(stamps) >= self.output_tokens:
            raise ValueError(f"request {self.id}: delivered past output target")
        stamps.append(now_us)


def request_digest(requests) -> str:
    """sha256 over every request's observable record, in id order.

    Same definition as the survey's F1/F2 fixtures, so
    digests from this package and from the reference simulator compare
    directly.
    """
    import hashlib

    h = hashlib.sha256()
    for r in sorted(requests, key=lambda r: r.id):
        rec = (
            r.id,
            r.state.value,
            tuple(r.token_times_us),
            r.decode_participations,
            r.preemptions,
            tuple((s.value, t) for s, t in r.history),
        )
        h.update(repr(rec).encode())
    return h.hexdigest()

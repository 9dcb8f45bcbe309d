"""Tensor-parallel serving layer (cfg 4): one engine, N ranks.

The reference runs one engine over an aggregate GPU (GpuSpec.aggregate, core.py:147-165).
Here rank 0 runs the real RapidEngine + B200Executor on its shard; every launch the engine
makes becomes a device command (B200Executor.run_command: block-table deltas, slot rows,
token ids, the partition key) that rank 0 also broadcasts, and every worker rank replays the
same command on its own shard, in the same order, on the same green-context partition. The
row-parallel GEMMs' all-reduces (tp.py / csrc/tp.cu, one communicator per phase) then line up
across ranks by construction; sampled ids are identical on every rank (the vocab-parallel
argmax is a max-reduce), so only rank 0 reads them back.

    rank 0:  ex = B200Executor(local_arch, ...); attach_leader(ex, CommandChannel(group))
             ... drive RapidEngine as usual ...; stop_workers(channel)
    rank r:  ex = B200Executor(local_arch, ..., num_blocks=<rank 0's>); serve_worker(ex, channel)

Wire format: a command is flattened into int32 words (encode_command / decode_command) and
sent as ONE fixed-size int32 broadcast (CAPACITY words, word 0 = the command's length); a
command longer than the frame (a large prefill's page grants) continues in further frames.
A decode step at bucket 256 with no page grants is 4 + 3 + 768 words, so the steady state is
one 64 KB broadcast per launch, no pickling and no length round trip.
"""

from __future__ import annotations

import os
import sys

import numpy as np

_DEBUG = bool(os.environ.get("RB_DEBUG_TP"))

STOP = ("stop",)
CAPACITY = 16384  # int32 words per frame

_KIND = {"stop": 0, "prefill": 1, "decode": 2}


def encode_command(cmd) -> np.ndarray:
    """Flatten a device command into int32 words: [len, kind, key|-1, n_upd, upd*3, body...].

    prefill body: slot, lo, last|-1, n_ids, ids...
    decode body:  B, bucket, slots[bucket], pos[bucket], seq[bucket]
    """
    kind = cmd[0]
    if kind == "stop":
        return np.array([2, 0], dtype=np.int32)
    key = -1 if cmd[1] is None else int(cmd[1])
    upd = cmd[2]
    head = [0, _KIND[kind], key, len(upd)]
    flat_upd = np.asarray(upd, dtype=np.int32).reshape(-1) if upd else np.zeros(0, np.int32)
    if kind == "prefill":
        _, _, _, slot, ids, lo, last = cmd
        body = np.concatenate([np.array([slot, lo, -1 if last is None else last, len(ids)], dtype=np.int32),
                               np.asarray(ids, dtype=np.int32).reshape(-1)])
    elif kind == "decode":
        _, _, _, B, bucket, slots, pos, seq = cmd
        if not (len(slots) == len(pos) == len(seq) == bucket):
            raise ValueError("decode command rows must have bucket entries")
        body = np.concatenate([np.array([B, bucket], dtype=np.int32), np.asarray(slots, dtype=np.int32),
                               np.asarray(pos, dtype=np.int32), np.asarray(seq, dtype=np.int32)])
    else:
        raise ValueError(f"unknown device command {kind!r}")
    words = np.concatenate([np.array(head, dtype=np.int32), flat_upd, body])
    words[0] = words.shape[0]
    return words


def decode_command(words: np.ndarray):
    """Inverse of encode_command (same tuple/list structure run_command takes)."""
    w = [int(x) for x in words[: int(words[0])]]
    kind = w[1]
    if kind == 0:
        return STOP
    key = None if w[2] == -1 else w[2]
    n_upd = w[3]
    upd = [tuple(w[4 + 3 * i : 7 + 3 * i]) for i in range(n_upd)]
    o = 4 + 3 * n_upd
    if kind == 1:
        slot, lo, last, n = w[o : o + 4]
        ids = w[o + 4 : o + 4 + n]
        return ("prefill", key, upd, slot, ids, lo, None if last == -1 else last)
    if kind == 2:
        B, bucket = w[o], w[o + 1]
        o += 2
        return ("decode", key, upd, B, bucket, w[o : o + bucket], w[o + bucket : o + 2 * bucket],
                w[o + 2 * bucket : o + 3 * bucket])
    raise ValueError(f"bad command kind {kind}")


class CommandChannel:
    """Rank 0 -> every rank, in order: fixed-size int32 frames (torch.distributed.broadcast)."""

    def __init__(self, group=None, capacity: int = CAPACITY):
        import torch
        import torch.distributed as dist

        self._dist = dist
        self.group = group
        self.capacity = capacity
        self._frame = torch.zeros(capacity, dtype=torch.int32)
        self.sent = 0
        self.frames = 0

    def _bcast(self) -> None:
        self._dist.broadcast(self._frame, src=0, group=self.group)
        self.frames += 1

    def send(self, cmd) -> None:
        if _DEBUG:
            print(f"[tp leader] send #{self.sent} {cmd[0]}", file=sys.stderr, flush=True)
        words = encode_command(cmd)
        f = self._frame.numpy()
        for off in range(0, words.shape[0], self.capacity):
            part = words[off : off + self.capacity]
            f[: part.shape[0]] = part
            self._bcast()
        self.sent += 1

    def recv(self):
        self._bcast()
        f = self._frame.numpy()
        n = int(f[0])
        if n <= self.capacity:
            return decode_command(f[:n].copy())
        words = np.empty(n, dtype=np.int32)
        words[: self.capacity] = f
        for off in range(self.capacity, n, self.capacity):
            self._bcast()
            k = min(self.capacity, n - off)
            words[off : off + k] = f[:k]
        return decode_command(words)


def attach_leader(executor, channel: CommandChannel) -> None:
    """Rank 0: every device command the executor runs is broadcast first."""
    executor.command_sink = channel.send


def stop_workers(channel: CommandChannel) -> None:
    channel.send(STOP)


def serve_worker(executor, channel: CommandChannel) -> int:
    """Worker ranks: replay rank 0's device commands until STOP; returns how many ran."""
    n = 0
    while True:
        cmd = channel.recv()
        if cmd == STOP:
            return n
        if _DEBUG:
            print(f"[tp worker] run #{n} {cmd[0]}", file=sys.stderr, flush=True)
        executor.run_command(cmd)
        n += 1

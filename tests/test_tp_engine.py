"""TP serving layer (tp_engine.py) over gloo, world 2: every device command the leader's
executor runs reaches the worker's executor in the same order with the same payload."""

import os

import pytest

from paper_2601_11822_b200.tp_engine import (CommandChannel, attach_leader, decode_command, encode_command,
                                             serve_worker, stop_workers)
from paper_2601_11822_b200.tp_serve import agreed_num_blocks


class _RecordingExecutor:
    """Stands in for B200Executor: run_command records; _issue mirrors its sink-then-run order."""

    command_sink = None

    def __init__(self):
        self.ran = []

    def run_command(self, cmd):
        self.ran.append(cmd)

    def _issue(self, cmd):
        if self.command_sink is not None:
            self.command_sink(cmd)
        return self.run_command(cmd)


def _commands():
    out = []
    for i in range(25):
        if i % 5 == 0:
            out.append(("prefill", 64 if i % 2 else None, [(i, 0, 3 * i), (i, 1, 3 * i + 1)], i, list(range(i, i + 7)),
                        0, i + 11 if i % 3 == 0 else None))
        else:
            B = 1 + i % 7
            out.append(("decode", 56, [(i, 4, 100 + i)] if i % 4 == 0 else [], B, 8, list(range(8)),
                        [i] * B + [-1] * (8 - B), [i + 1] * B + [0] * (8 - B)))
    return out


def _rank(rank, world, port, q, capacity):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ch = CommandChannel(capacity=capacity)
    agreed = agreed_num_blocks(1000 - 7 * rank, None)  # every rank's cache must hold rank 0's page ids
    ex = _RecordingExecutor()
    if rank == 0:
        attach_leader(ex, ch)
        for cmd in _commands():
            ex._issue(cmd)
        stop_workers(ch)
        q.put((rank, ex.ran, ch.sent, ch.frames, agreed))
    else:
        n = serve_worker(ex, ch)
        q.put((rank, ex.ran, n, ch.frames, agreed))
    dist.destroy_process_group()


def test_command_wire_format_round_trip():
    for cmd in _commands() + [("prefill", 0, [], 3, [], 5, 7), ("stop",)]:
        w = encode_command(cmd)
        assert w.dtype.name == "int32" and int(w[0]) == w.shape[0]
        assert decode_command(w) == cmd


@pytest.mark.parametrize("capacity", [16384, 16])
def test_leader_commands_replay_on_worker(capacity):
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q, capacity)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, leader_ran, sent, f0, a0), (_, worker_ran, n, f1, a1) = out
    assert a0 == a1 == 993
    want = _commands()
    assert leader_ran == want
    assert worker_ran == want
    assert n == len(want) and sent == len(want) + 1  # + STOP
    assert f0 == f1  # every frame the leader broadcast was received
    if capacity >= 16384:
        assert f0 == sent  # one fixed-size frame per command
    else:
        assert f0 > sent  # long commands continued in further frames

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

The channel is a torch.distributed object broadcast (gloo on the host). Multi-GPU TP was not
run in this round (one GPU per call); the command path is exercised by the gloo test and by
rank 0's own executor, which executes exactly the commands it broadcasts.
"""

from __future__ import annotations

STOP = ("stop",)


class CommandChannel:
    """Rank 0 -> every rank, in order (torch.distributed.broadcast_object_list)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self._dist = dist
        self.group = group
        self.sent = 0

    def send(self, cmd) -> None:
        self._dist.broadcast_object_list([cmd], src=0, group=self.group)
        self.sent += 1

    def recv(self):
        buf = [None]
        self._dist.broadcast_object_list(buf, src=0, group=self.group)
        return buf[0]


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
        if cmd == STOP or cmd[0] == "stop":
            return n
        executor.run_command(cmd)
        n += 1

"""B200Executor: the engines' launch sites realized as sm_100a kernels.

RAPID (engines/rapid.py) calls launch_prefill / launch_decode exactly where the
reference prices an iteration (pkg/src/pdsim/engines/rapid.py:171-189,
:266-293); completions come back through CUDA events polled by RealTimeLoop.

Phases and SM partitions (K7): the ARM decision selects the streams —
  * OVERALLOCATE: both phases on full-device streams (148 SMs, contending);
  * PARTITION:    decode on a green context of cu_fraction_decode*148 SMs
                  rounded up to 8, prefill on the complementary green context.
A static split (cfg 2) fixes one partition for the whole run.

Token-position contract: a prefill of `target`
context tokens computes KV for positions 0..target-2 only; decode
participation k consumes the token at position target-2+k (its input id
lives in last_tok[slot] on the device) and writes its KV there.

Block-table mirroring: the BlockPool reports every new page; admission pages
are applied on the prefill stream before that request's first chunk, decode
extensions on the decode stream before the step that needs them.
"""

from __future__ import annotations

import math
import os
import sys
import time

import numpy as np
import torch

from paper_2601_11822_b200 import ops
from paper_2601_11822_b200.arm import DEFAULT_BATCH_GRID
from paper_2601_11822_b200.blockpool import BlockPool
from paper_2601_11822_b200.model import PAGE, DecoderWeights, Runner
from paper_2601_11822_b200.specs import AllocationDecision, AllocationMode, ArchConfig, decode_sms_for
from paper_2601_11822_b200.traffic import prompt_token_ids

MAX_UPDATES = 1 << 16


class GpuHandle:
    def __init__(self, kind, stream, cu_fraction, events=None):
        self.kind = kind
        # (executor-pooled) start / end events: creating two CUDA events per launch cost ~10-20 us of host time
        self.ev0, self.ev1 = events if events is not None else (torch.cuda.Event(enable_timing=True),
                                                                torch.cuda.Event(enable_timing=True))
        self.ev0.record(stream)
        self.gpu_us = 0
        self.cu_fraction = cu_fraction
        self.members = ()
        self.start_us = 0
        self.launch_ns = time.perf_counter_ns()

    def finish_record(self, stream):
        self.ev1.record(stream)

    def done(self) -> bool:
        if self.ev1.query():
            self.gpu_us = max(1, int(round(self.ev0.elapsed_time(self.ev1) * 1000.0)))
            return True
        return False


class _Partition:
    """A pair of streams (decode, prefill) with their SM counts."""

    def __init__(self, decode_stream, prefill_stream, decode_sms, prefill_sms, green=None):
        self.ds = decode_stream
        self.ps = prefill_stream
        self.d_sms = decode_sms
        self.p_sms = prefill_sms
        self.green = green
        self.graphs: dict[int, torch.cuda.CUDAGraph] = {}
        self.graph_exec: dict[int, int] = {}  # bucket -> cudaGraphExec_t of graphs[bucket]
        self.key = None  # decode SM count this partition is registered under (None = full device)


class B200Executor:
    realtime = True

    def __init__(self, arch: ArchConfig, weights: DecoderWeights | None = None, *, seed: int = 0,
                 static_decode_sms: int | None = None, max_batch: int = 256, chunk_tokens: int = 2048,
                 num_blocks: int | None = None, kv_memory_fraction: float = 0.90, max_context: int | None = None,
                 num_slots: int = 1024, device: str = "cuda", token_source=None, use_graphs: bool = True,
                 batch_grid: tuple[int, ...] = DEFAULT_BATCH_GRID, serialize_phases: bool = False,
                 record_logits: bool = False, probe_attention: bool = False, vocab_offset: int = 0):
        self.arch = arch
        dev = torch.device(device)
        self.device = dev if dev.index is not None else torch.device("cuda", torch.cuda.current_device())
        torch.cuda.set_device(self.device)
        ops.load()
        self.weights = weights if weights is not None else DecoderWeights.random(arch, device=self.device, seed=seed)
        self.max_batch = max_batch
        self.chunk_tokens = chunk_tokens
        self.num_slots = num_slots
        self.use_graphs = use_graphs
        self.grid = tuple(b for b in batch_grid if b <= max_batch) or (max_batch,)
        # batches past the grid's last entry (max_batch > 256) get 32-row buckets, not one pad to max_batch
        self.grid = self.grid + tuple(range(self.grid[-1] + 32, max_batch, 32))
        if self.grid[-1] < max_batch:
            self.grid = self.grid + (max_batch,)
        self.total_sms = ops.device_sm_count(self.device.index or 0)
        self.token_source = token_source or (lambda req: prompt_token_ids(req.id, req.prompt_tokens, arch.vocab))
        max_ctx = max_context or 16384
        self.max_blocks_per_seq = (max_ctx + PAGE) // PAGE + 1
        bpb = Runner.kv_bytes_per_block(arch)
        if num_blocks is None:
            torch.cuda.synchronize()
            free, _ = torch.cuda.mem_get_info(self.device)
            # activations / graphs / workspaces: reserve generously, then the reference's 10% rule
            act = self._activation_bytes(max(chunk_tokens, 1), max_batch) + (2 << 30)
            num_blocks = int(max(0, free - act) * kv_memory_fraction // bpb)
        if num_blocks < 1:
            raise RuntimeError("no HBM left for the KV cache")
        self.num_blocks = num_blocks
        self.runner = Runner(self.weights, num_blocks, num_slots, self.max_blocks_per_seq,
                             max_prefill_tokens=max(chunk_tokens, 16), max_decode_batch=max_batch, device=self.device,
                             vocab_offset=vocab_offset)
        # host mirrors / staging (pinned)
        self._slot_of: dict[int, int] = {}
        self._free_slots = list(range(num_slots - 1, -1, -1))
        self._upd = {"prefill": [], "decode": []}
        self._upd_host = {k: torch.zeros(1 + 3 * MAX_UPDATES, dtype=torch.int32, pin_memory=True)
                          for k in self._upd}
        self._upd_dev = {k: torch.zeros(1 + 3 * MAX_UPDATES, dtype=torch.int32, device=self.device)
                         for k in self._upd}
        self._dec_in_host = torch.zeros(3, max_batch, dtype=torch.int32, pin_memory=True)
        self._dec_in_host_np = self._dec_in_host.numpy()
        self._dec_in_bytes = self._dec_in_host.numel() * 4
        self._lib = ops.load()
        self._ev_pool: list = []
        self._upd_host_np = {k: v.numpy() for k, v in self._upd_host.items()}
        self._bt_ptr = self.runner.block_table.data_ptr()
        self._bt_stride = self.runner.block_table.stride(0)
        self._dec_in_dev = torch.zeros(3, max_batch, dtype=torch.int32, device=self.device)
        d = self.runner.dec
        d.slot = self._dec_in_dev[0]
        d.pos = self._dec_in_dev[1]
        d.seq = self._dec_in_dev[2]
        self._dec_out_host = torch.zeros(max_batch, dtype=torch.int32, pin_memory=True)
        self._dec_out_host_np = self._dec_out_host.numpy()
        self._pre_ids_host = torch.zeros(max(chunk_tokens, 16), dtype=torch.int32, pin_memory=True)
        self._pre_ids_dev = torch.zeros(max(chunk_tokens, 16), dtype=torch.int32, device=self.device)
        self._generated: dict[int, list[int]] = {}
        self._pending_gen: list = []  # (members, lame, ids) of finished steps not yet in _generated
        # parity tests: fp32 host copy of the logits row behind every generated token
        self.record_logits = record_logits
        self.logits: dict[int, list[torch.Tensor]] = {}
        self._tokens_cache: dict[int, torch.Tensor] = {}
        # partitions
        self._partitions: dict[int | None, _Partition] = {}
        full_d = torch.cuda.Stream(device=self.device)
        full_p = full_d if serialize_phases else torch.cuda.Stream(device=self.device)
        self._partitions[None] = _Partition(full_d, full_p, self.total_sms, self.total_sms)
        self.static_decode_sms = static_decode_sms
        if static_decode_sms is not None:
            self._partition(static_decode_sms)
        # stats
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self.decode_steps = 0
        self.prefill_chunks = 0
        self.gpu_launches = 0
        self.lazy_captures = 0
        self.step_log: list[tuple[int, int, int]] = []  # (B, gpu_us, host launch ns)
        self.host_gap_log: list[int] = []  # us from a decode completion's handling to the next launch
        self._t_fin_ns = None
        # RB_HOST_PROFILE=1: ns spent per decode step in finish_decode / launch composition / command issue
        self.host_prof = {"finish": 0, "compose": 0, "issue": 0, "steps": 0} if os.environ.get("RB_HOST_PROFILE") \
            else None
        self.prefill_log: list[tuple[int, int]] = []  # (gpu_us, host launch ns)
        # in-situ decode-attention roofline: (algorithmic K+V bytes, kernel ms, decode SMs, host
        # launch ns) of the probed layer in every decode step (CUDA events inside the graphs)
        self.attn_probe_log: list[tuple[int, float, int, int]] = []
        self._probe_events = None
        if probe_attention:
            self._probe_events = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            self.runner.set_attention_probe(*self._probe_events, layer=arch.layers // 2)

    # ------------------------------------------------------------------ sizing
    def _activation_bytes(self, T: int, B: int) -> int:
        a = self.arch
        nq = (a.q_heads + 2 * a.kv_heads) * a.head_dim
        per_row = 2 * (2 * a.hidden + nq + 2 * a.q_heads * a.head_dim + 3 * a.intermediate)
        return per_row * (T + B) + B * a.vocab * 2 + B * a.q_heads * 16 * (a.head_dim + 2) * 4

    def make_pool(self, model, gpu) -> BlockPool:
        pool = BlockPool(self.num_blocks, PAGE, name="gpu0")
        pool.listener = self
        return pool

    def bind(self, engine) -> None:
        self.engine = engine
        if getattr(engine, "max_batch", self.max_batch) > self.max_batch:
            raise ValueError("engine max_batch exceeds the executor's decode workspace")

    # ------------------------------------------------------------------ partitions
    def _partition(self, decode_sms: int | None) -> _Partition:
        if decode_sms not in self._partitions:
            gs = ops.GreenSplit(decode_sms, device=self.device.index or 0)
            p = _Partition(gs.streams[0], gs.streams[1], gs.sms[0], gs.sms[1], gs)
            p.key = decode_sms
            self._partitions[decode_sms] = p
        return self._partitions[decode_sms]

    def _pick(self, decision: AllocationDecision) -> _Partition:
        if self.static_decode_sms is not None:
            return self._partitions[self.static_decode_sms]
        return self._partition(decode_sms_for(decision, self.total_sms))

    # ------------------------------------------------------------------ pool listener
    def _slot(self, req_id: int) -> int:
        s = self._slot_of.get(req_id)
        if s is None:
            if not self._free_slots:
                raise RuntimeError(f"out of request slots ({self.num_slots}): raise num_slots to cover the "
                                   f"requests the KV pool can hold at once")
            s = self._free_slots.pop()
            self._slot_of[req_id] = s
        return s

    def on_pages(self, req_id: int, first_index: int, ids: list[int]) -> None:
        s = self._slot(req_id)
        if first_index + len(ids) > self.max_blocks_per_seq:
            raise RuntimeError("request context exceeds max_blocks_per_seq")
        q = self._upd["prefill" if first_index == 0 else "decode"]
        for j, b in enumerate(ids):
            q.append((s, first_index + j, b))

    def on_release(self, req_id: int) -> None:
        s = self._slot_of.pop(req_id, None)
        if s is not None:
            # page grants still queued for this slot belong to the released request (e.g. a
            # decode extension of a member preempted in the same reservation pass): drop
            # them, or they would land after the slot's next owner writes its rows on the
            # other stream
            for q in self._upd.values():
                if any(u[0] == s for u in q):
                    q[:] = [u for u in q if u[0] != s]
            self._free_slots.append(s)

    def _flush_updates(self, phase: str, stream) -> None:
        q = self._upd[phase]
        if not q:
            return
        n = len(q)
        if n > MAX_UPDATES:
            raise RuntimeError("too many pending block-table updates")
        h = self._upd_host_np[phase]
        h[0] = n
        h[1 : 1 + 3 * n] = np.asarray(q, dtype=np.int32).reshape(-1)
        d = self._upd_dev[phase]
        lib = self._lib
        ops._check(lib.rb_memcpy_async(d.data_ptr(), self._upd_host[phase].data_ptr(), 4 * (1 + 3 * n),
                                       stream.cuda_stream), "rb_memcpy_async")
        ops._check(lib.rb_block_table_update(d.data_ptr(), self._bt_ptr, self._bt_stride, n, stream.cuda_stream),
                   "rb_block_table_update")
        self.h2d_bytes += 4 * (1 + 3 * n)
        self.gpu_launches += 1
        q.clear()  # one launch per phase is in flight, so the pinned buffer is free again at the next flush

    # ------------------------------------------------------------------ tokens
    def _token_seq(self, req) -> torch.Tensor:
        t = self._tokens_cache.get(req.id)
        if t is None:
            t = self.token_source(req)
            self._tokens_cache[req.id] = t
        return t

    def _context_ids(self, req, lo: int, hi: int) -> torch.Tensor:
        """Token ids at context positions [lo, hi): prompt then generated tokens."""
        prompt = self._token_seq(req)
        P = prompt.shape[0]
        if hi <= P:
            return prompt[lo:hi]
        gen = self.generated.get(req.id, [])
        tail = torch.tensor(gen[max(0, lo - P) : hi - P], dtype=torch.int32)
        if lo >= P:
            return tail
        return torch.cat([prompt[lo:P], tail])

    # ------------------------------------------------------------------ prefill
    # Device work of a launch as a plain command (tuple of ints / int lists): the single-GPU
    # executor runs it directly; under tensor parallelism (tp_engine.py) the leader rank also
    # broadcasts it and every worker rank runs the same command on its shard.
    command_sink = None  # callable(cmd) or None

    def _partition_key(self, part: _Partition) -> int | None:
        return part.key

    def _events(self):
        return self._ev_pool.pop() if self._ev_pool else None

    def _recycle(self, handle) -> None:
        # a handle someone still holds for timing (bench's window marks, h._win) keeps its events
        if handle is not None and not getattr(handle, "_win", False) and len(self._ev_pool) < 64:
            self._ev_pool.append((handle.ev0, handle.ev1))

    def run_command(self, cmd) -> _Partition:
        """Execute one device command (the same on every TP rank); returns its partition."""
        kind, key = cmd[0], cmd[1]
        part = self._partitions[key] if key in self._partitions else self._partition(key)
        if kind == "prefill":
            _, _, upd, slot, ids, lo, last = cmd
            st = part.ps
            self._upd["prefill"].extend(upd)
            self._flush_updates("prefill", st)
            if ids:
                n = len(ids)
                self._pre_ids_host[:n].copy_(torch.tensor(ids, dtype=torch.int32))
                with torch.cuda.stream(st):
                    self._pre_ids_dev[:n].copy_(self._pre_ids_host[:n], non_blocking=True)
                    self.runner.prefill(slot, self._pre_ids_dev[:n], lo, num_sms=part.p_sms, stream=st.cuda_stream)
                self.h2d_bytes += 4 * n
                self.gpu_launches += self.runner.kernels_per_forward(0, n, False, False, False)
            if last is not None:
                ops.set_last_token(self.runner.last_tok, slot, value=last, stream=st.cuda_stream)
                self.gpu_launches += 1
        elif kind == "decode":
            _, _, upd, B, bucket, slots, pos, seq = cmd
            st = part.ds
            self._upd["decode"].extend(upd)
            self._flush_updates("decode", st)
            h = self._dec_in_host_np  # numpy view of the pinned staging rows (list -> int32 without torch)
            h[0, :bucket] = slots
            h[1, :bucket] = pos
            h[2, :bucket] = seq
            lib, sh = self._lib, st.cuda_stream
            # the whole [3, max_batch] staging block (3 KB at 256 rows): one contiguous copy; rows past
            # the bucket are never read by the bucket's graph
            ops._check(lib.rb_memcpy_async(self._dec_in_dev.data_ptr(), self._dec_in_host.data_ptr(),
                                           self._dec_in_bytes, sh), "rb_memcpy_async")
            if self.use_graphs:
                g = self._capture(part, bucket)
                ex_h = part.graph_exec.get(bucket)
                if ex_h is None:
                    raw = g.raw_cuda_graph_exec()
                    ex_h = part.graph_exec[bucket] = raw if isinstance(raw, int) else 0
                if ex_h:
                    ops._check(lib.rb_graph_launch(ex_h, sh), "rb_graph_launch")
                else:  # no raw handle from this torch build: the framework's replay
                    with torch.cuda.stream(st):
                        g.replay()
            else:
                with torch.cuda.stream(st):
                    self.runner.decode_body(bucket, num_sms=part.d_sms, max_pages=(max(seq) + PAGE - 1) // PAGE,
                                            stream=sh)
            ops._check(lib.rb_memcpy_async(self._dec_out_host.data_ptr(), self.runner.dec.out_ids.data_ptr(), 4 * B,
                                           sh), "rb_memcpy_async")
            self.h2d_bytes += 12 * bucket
            self.d2h_bytes += 4 * B
            self.gpu_launches += self.runner.kernels_per_forward(bucket, 0, True, False, True)
        else:
            raise ValueError(f"unknown device command {kind!r}")
        return part

    def _issue(self, cmd) -> _Partition:
        if self.command_sink is not None:
            self.command_sink(cmd)
        return self.run_command(cmd)

    def _take_updates(self, phase: str) -> list:
        upd = list(self._upd[phase])
        self._upd[phase].clear()
        return upd

    def launch_prefill(self, req, written: int, chunk: int, target: int, decision, co_decode) -> GpuHandle:
        part = self._pick(decision)
        h = GpuHandle("prefill", part.ps, part.p_sms / self.total_sms, self._events())
        slot = self._slot_of[req.id]
        lo, hi = written, min(written + chunk, target - 1)
        ids = self._context_ids(req, lo, hi).tolist() if hi > lo else []
        last = int(self._context_ids(req, target - 1, target)[0]) if written + chunk == target else None
        self._issue(("prefill", self._partition_key(part), self._take_updates("prefill"), slot, ids, lo, last))
        h.finish_record(part.ps)
        h.req = req
        self.prefill_chunks += 1
        return h

    def finish_prefill(self, handle) -> None:
        if handle is not None:
            self.prefill_log.append((handle.gpu_us, handle.launch_ns))
            self._recycle(handle)

    # ------------------------------------------------------------------ decode
    def _bucket(self, B: int) -> int:
        for g in self.grid:
            if g >= B:
                return g
        return self.grid[-1]

    def _capture(self, part: _Partition, bucket: int) -> torch.cuda.CUDAGraph:
        g = part.graphs.get(bucket)
        if g is not None:
            return g
        r = self.runner
        st = part.ds
        # A decode step is not idempotent (argmax overwrites last_tok[slot], the QKV epilogue
        # writes KV at pos), so the eager warm-up must not run on live inputs: a lazy capture
        # during serving parks the step's inputs, warms up on padding rows only, and restores
        # them before the replay (stream-ordered on the decode stream).
        with torch.cuda.stream(st):
            live = self._dec_in_dev.clone()
            self._inert_decode_inputs()
            # warm up outside capture (tensor-map cache, function attributes)
            r.decode_body(bucket, num_sms=part.d_sms, stream=st.cuda_stream)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            r.decode_body(bucket, num_sms=part.d_sms, stream=st.cuda_stream)
        with torch.cuda.stream(st):
            self._dec_in_dev.copy_(live)
        st.synchronize()
        part.graphs[bucket] = g
        self.lazy_captures += 1
        return g

    def _inert_decode_inputs(self) -> None:
        """Padding rows only: dummy slot, no KV write (pos -1), empty context."""
        self._dec_in_dev[0].fill_(self.runner.dummy_slot)
        self._dec_in_dev[1].fill_(-1)
        self._dec_in_dev[2].fill_(0)

    def warmup(self, decode_sms_list=None) -> None:
        """Pre-capture decode graphs for every bucket on the partitions in use."""
        if not self.use_graphs:
            return
        keys = decode_sms_list if decode_sms_list is not None else (
            [self.static_decode_sms] if self.static_decode_sms is not None else [None])
        dbg = os.environ.get("RB_DEBUG_WARMUP")
        for k in keys:
            part = self._partition(k) if k is not None else self._partitions[None]
            for b in self.grid:
                if dbg:
                    print(f"[warmup pid {os.getpid()}] partition {k} bucket {b}", file=sys.stderr, flush=True)
                self._capture(part, b)
        torch.cuda.synchronize()
        self.lazy_captures = 0  # captures counted from here on happened while serving

    def launch_decode(self, members, decision, co_prefill_chunk) -> GpuHandle:
        t_prof = time.perf_counter_ns() if self.host_prof is not None else 0
        part = self._pick(decision)
        B = len(members)
        bucket = self._bucket(B)
        h = GpuHandle("decode", part.ds, part.d_sms / self.total_sms, self._events())
        slot_of = self._slot_of
        seq = [r.prompt_tokens + len(r.token_times_us) for r in members]  # context_tokens (core.py:98-101)
        slots = [slot_of[r.id] for r in members]
        pos = [c - 1 for c in seq]
        lame = [len(r.token_times_us) >= r.output_tokens for r in members]
        pad = bucket - B
        if pad:
            slots += [self.runner.dummy_slot] * pad
            pos += [-1] * pad
            seq += [0] * pad
        if t_prof:
            t_mid = time.perf_counter_ns()
        self._issue(("decode", self._partition_key(part), self._take_updates("decode"), B, bucket, slots, pos, seq))
        h.finish_record(part.ds)
        if t_prof:
            t_end = time.perf_counter_ns()
            self.host_prof["compose"] += t_mid - t_prof
            self.host_prof["issue"] += t_end - t_mid
            self.host_prof["steps"] += 1
        if self._t_fin_ns is not None:  # host time from the previous step's completion to this launch
            self.host_gap_log.append((time.perf_counter_ns() - self._t_fin_ns) // 1000)
            self._t_fin_ns = None
        h.members = tuple(members)
        h.lame = lame
        h.d_sms = part.d_sms
        # K+V bytes the probed layer's attention reads: every row's context (bf16)
        h.attn_bytes = sum(seq) * self.arch.kv_heads * self.arch.head_dim * 4
        self.decode_steps += 1
        return h

    @property
    def generated(self) -> dict[int, list[int]]:
        """Sampled ids per request (prompt excluded), in order."""
        self._drain_generated()
        return self._generated

    def _drain_generated(self) -> None:
        pend, self._pending_gen = self._pending_gen, []
        gen = self._generated
        for members, lame, ids in pend:
            for r, is_lame, tok in zip(members, lame, ids.tolist()):
                if not is_lame:
                    gen.setdefault(r.id, []).append(tok)

    def on_idle(self) -> None:
        """The real-time loop's idle hook (no event ready): bookkeeping that is off the critical path."""
        if self._pending_gen:
            self._drain_generated()

    def finish_decode(self, handle) -> None:
        if handle is None:
            return
        self._t_fin_ns = time.perf_counter_ns()
        B = len(handle.members)
        if self.record_logits:
            out = self._dec_out_host[:B].tolist()
            rows = self.runner.dec.logits[:B].float().cpu()
            for i, (r, is_lame, tok) in enumerate(zip(handle.members, handle.lame, out)):
                if not is_lame:
                    self.generated.setdefault(r.id, []).append(tok)
                    self.logits.setdefault(r.id, []).append(rows[i])
        else:
            # the ids are snapshotted (the next step's D2H reuses the pinned buffer) and filed into
            # `generated` when the loop idles or someone reads them (a re-prefill after preemption)
            self._pending_gen.append((handle.members, handle.lame, self._dec_out_host_np[:B].copy()))
        self.step_log.append((len(handle.members), handle.gpu_us, handle.launch_ns))
        if self._probe_events is not None:
            # the step's end event has completed, so this step's probe records are final
            self.attn_probe_log.append((handle.attn_bytes, self._probe_events[0].elapsed_time(self._probe_events[1]),
                                        handle.d_sms, handle.launch_ns))
        self._recycle(handle)
        if self.host_prof is not None:
            self.host_prof["finish"] += time.perf_counter_ns() - self._t_fin_ns

    # ------------------------------------------------------------------ hybrid (K9 fused iteration)
    def launch_hybrid(self, members, head, written, chunk, target):
        raise NotImplementedError("fused hybrid iterations run on HybridB200Executor")

    def finish_hybrid(self, handle) -> None:
        pass

    # ------------------------------------------------------------------ lifecycle hooks
    def on_preempt(self, req) -> None:
        pass  # generated ids are kept: the re-prefill rebuilds prompt + y1..y_{d-1}

    def on_finish(self, req) -> None:
        self._tokens_cache.pop(req.id, None)

    def close(self) -> None:
        # Graphs are dropped; green contexts live until process exit (torch
        # still holds ExternalStream / event objects bound to them).
        torch.cuda.synchronize()
        for p in self._partitions.values():
            p.graphs.clear()


class HybridB200Executor(B200Executor):
    """Same-engine hybrid batching (chunked prefill) on the B200 — the comparator.

    One fused iteration per launch on the whole device (K9): decode rows of all
    running sequences plus one prefill chunk share every GEMM; attention splits
    into the paged decode kernel (rows 0..B-1) and the chunk's causal kernel.
    Token-position contract of hybrid mode: the prefill
    computes every context position and its last chunk samples y1 from the
    final position (reference hybrid.py:144-155); a decode row at context c
    consumes the token at position c-1 and writes its KV there.
    """

    def __init__(self, arch: ArchConfig, weights: DecoderWeights | None = None, **kw):
        kw.pop("static_decode_sms", None)
        kw.setdefault("chunk_tokens", 512)
        super().__init__(arch, weights, static_decode_sms=None, **kw)
        cap = self.runner.max_prefill_tokens
        self._hyb_host = torch.zeros(3 * cap, dtype=torch.int32, pin_memory=True)
        self._hyb_dev = torch.zeros(3 * cap, dtype=torch.int32, device=self.device)
        pre = self.runner.pre
        pre.slot = self._hyb_dev[0:cap]
        pre.pos = self._hyb_dev[cap:2 * cap]
        pre.seq = self._hyb_dev[2 * cap:3 * cap]
        self._hyb_out_host = torch.zeros(cap, dtype=torch.int32, pin_memory=True)

    def warmup(self, decode_sms_list=None) -> None:
        pass  # fused iterations are not graph-captured (shape changes every iteration)

    def _flush_all(self, stream) -> None:
        self._upd["decode"].extend(self._upd["prefill"])
        self._upd["prefill"].clear()
        self._flush_updates("decode", stream)

    def launch_hybrid(self, members, head, written: int, chunk: int, target: int) -> GpuHandle:
        part = self._partitions[None]
        st = part.ds
        h = GpuHandle("hybrid", st, 1.0)
        self._flush_all(st)
        B = len(members)
        cap = self.runner.max_prefill_tokens
        hb = self._hyb_host
        slots = [self._slot_of[r.id] for r in members]
        ctxs = [r.context_tokens for r in members]
        if B:
            hb[0:B].copy_(torch.tensor(slots, dtype=torch.int32))
            hb[cap:cap + B].copy_(torch.tensor([c - 1 for c in ctxs], dtype=torch.int32))
            hb[2 * cap:2 * cap + B].copy_(torch.tensor(ctxs, dtype=torch.int32))
        emit = False
        chunk_dev = None
        hslot = 0
        if head is not None and chunk > 0:
            hslot = self._slot_of[head.id]
            ids = self._context_ids(head, written, written + chunk)
            self._pre_ids_host[:chunk].copy_(ids)
            emit = written + chunk == target
        with torch.cuda.stream(st):
            if B:
                for k in range(3):
                    self._hyb_dev[k * cap:k * cap + B].copy_(hb[k * cap:k * cap + B], non_blocking=True)
            if head is not None and chunk > 0:
                self._pre_ids_dev[:chunk].copy_(self._pre_ids_host[:chunk], non_blocking=True)
                chunk_dev = self._pre_ids_dev[:chunk]
            max_pages = max([(c + PAGE - 1) // PAGE for c in ctxs], default=1)
            self.runner.hybrid(B, hslot, written, chunk_dev, emit=emit, num_sms=part.d_sms, max_pages=max_pages,
                               stream=st.cuda_stream)
            n_out = B + (1 if emit else 0)
            if n_out:
                self._hyb_out_host[:n_out].copy_(self.runner.pre.out_ids[:n_out], non_blocking=True)
        h.finish_record(st)
        h.members = tuple(members)
        h.lame = [False] * B
        h.req = head if emit else None
        self.h2d_bytes += 12 * B + 4 * chunk
        self.d2h_bytes += 4 * (B + (1 if emit else 0))
        self.decode_steps += 1
        self.gpu_launches += self.runner.kernels_per_forward(B, chunk if chunk_dev is not None else 0, True, emit, True)
        return h

    def finish_hybrid(self, handle) -> None:
        if handle is None:
            return
        B = len(handle.members)
        n = B + (1 if handle.req is not None else 0)
        out = self._hyb_out_host[:n].tolist()
        rows = self.runner.pre.logits[:n].float().cpu() if self.record_logits else None
        for i, (r, tok) in enumerate(zip(handle.members, out)):
            self.generated.setdefault(r.id, []).append(tok)
            if rows is not None:
                self.logits.setdefault(r.id, []).append(rows[i])
        if handle.req is not None:
            self.generated.setdefault(handle.req.id, []).append(out[B])
            if rows is not None:
                self.logits.setdefault(handle.req.id, []).append(rows[B])
        self.step_log.append((B, handle.gpu_us, handle.launch_ns))

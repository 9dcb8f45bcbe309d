"""ARM policy study on the CPU: RapidEngine on the virtual clock with every launch priced
from the MEASURED B200 tables (executor.MeasuredTableExecutor), on the bench's cfg-3 trace.
Prints the reference summarize() run-level numbers per policy, plus per-second diagnostics.

    python scripts/arm_sim.py [--qps 56] [--duration 60] [--policies balanced,adaptive]
"""
import argparse
import collections
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2601_11822_b200.arm import CostParams, MeasuredArm, MeasuredProfile  # noqa: E402
from paper_2601_11822_b200.clock import Simulation  # noqa: E402
from paper_2601_11822_b200.engines.rapid import RapidEngine  # noqa: E402
from paper_2601_11822_b200.executor import MeasuredTableExecutor  # noqa: E402
from paper_2601_11822_b200.harness import check_invariants  # noqa: E402
from paper_2601_11822_b200.slo import SloSpec, summarize  # noqa: E402
from paper_2601_11822_b200.specs import ARCHS, b200_spec  # noqa: E402
from paper_2601_11822_b200.traffic import WorkloadSpec, synthesize  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--qps", type=float, default=56.0)
ap.add_argument("--duration", type=float, default=60.0)
ap.add_argument("--profile", default="profiles/arm/llama3.1-8b_ctx1152_chunk1023.json")
ap.add_argument("--model", default="llama3.1-8b")
ap.add_argument("--prompt", type=int, default=1024)
ap.add_argument("--output", type=int, default=256)
ap.add_argument("--policies", default="balanced,adaptive,slo-min")
ap.add_argument("--cpu-us", type=int, default=150, help="host gap per launch (the real-time loop's)")
ap.add_argument("--verbose", action="store_true")
a = ap.parse_args()

mp = MeasuredProfile.load(a.profile)
arch = ARCHS[a.model]
model = arch.model_spec()
slo = SloSpec(itl_slo_us=50_000)
horizon = int(a.duration * 1e6)
items = synthesize(WorkloadSpec(qps=a.qps, duration_s=a.duration, seed=42, mean_prompt_tokens=a.prompt,
                                mean_output_tokens=a.output, sigma=0.0))
for pol in a.policies.split(","):
    arm = MeasuredArm(mp, 50_000, 256, pol)
    ex = MeasuredTableExecutor(mp, num_blocks=69000)
    eng = RapidEngine(model, b200_spec(), CostParams(), slo, chunk_tokens=2048, max_batch=256, executor=ex,
                      arm_policy=arm, record_decisions=True, record_launches=True)
    eng.cpu_us = a.cpu_us
    sim = Simulation(until_us=horizon)
    eng.prime(sim, items)
    sim.run(eng.on_event)
    check_invariants(eng)
    s = summarize(pol, a.qps, eng.requests, slo, horizon, eng.busy_intervals, eng.pools)
    print(f"{pol:10s} tok/s {s.tokens_per_s:8.0f}  p99 ITL {s.itl_p99_us / 1e3:5.1f} ms  p50 TTFT "
          f"{s.ttft_p50_us / 1e3:7.0f} ms  goodput {s.goodput:5.2f}")
    if a.verbose:
        tok = collections.Counter(int(t // 1e6) for r in eng.requests for t in r.token_times_us)
        dec = collections.defaultdict(list)
        for (ph, st, en), (ph2, d) in zip([x for x in eng.launch_log if x[0] == "decode"],
                                         [x for x in eng.decision_log if x[0] == "decode"]):
            dec[int(st // 1e6)].append((en - st, round(d.cu_fraction_decode * 148)))
        for sec in range(int(a.duration) + 3):
            v = dec.get(sec, [])
            print(f"   {sec:3d}s tok {tok.get(sec, 0):6d}  steps {len(v):3d}  step ms "
                  f"{statistics.mean(x for x, _ in v) / 1e3 if v else 0:5.1f}  D {collections.Counter(d for _, d in v).most_common(2)}")

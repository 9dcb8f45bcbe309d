"""bench.py --impl reference: the CPU restatement timed as the reference arm (no GPU needed).

W warm-up and K timed steps, each one bounded sample (one prefill chunk + one batched decode
step of the fp32 oracle); the JSON line keeps the bench contract's keys."""

import json
import os
import subprocess
import sys

from oracle.cpu_baseline import CpuSampler
from paper_2601_11822_b200.specs import ARCHS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpu_sampler_steps_are_bounded_samples():
    s = CpuSampler(ARCHS["tiny"], 1024, 256, batch=2, prefill_tokens=8, threads=2)
    r = [s.step() for _ in range(3)]
    assert all(x["value"] > 0 and x["wall_s"] > 0 for x in r)
    assert "1 prefill chunk of 8 tokens" in s.describe()


def test_reference_arm_line_honours_steps_and_warmup():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--model", "tiny",
                          "--steps", "4", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["steps"] == 4 and line["warmup"] == 3
    assert line["value"] > 0 and line["unit"] == "output tokens/s" and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "output tokens/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}

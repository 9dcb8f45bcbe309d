import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle.llama_fp32 import Oracle, init_state
from paper_2601_11822_b200.model import DecoderWeights
from paper_2601_11822_b200.specs import ARCHS, b200_spec
from paper_2601_11822_b200.arm import CostParams
from paper_2601_11822_b200.engines.rapid import RapidEngine
from paper_2601_11822_b200.executor_b200 import B200Executor
from paper_2601_11822_b200.harness import run_items
from paper_2601_11822_b200.slo import SloSpec
from paper_2601_11822_b200.traffic import WorkloadSpec, prompt_token_ids, synthesize

arch = ARCHS["tiny"]
st = init_state(arch, seed=0)
orc = Oracle(arch, st)
w = DecoderWeights.from_state(arch, st)
items = synthesize(WorkloadSpec(qps=16.0, duration_s=4.0, seed=0, mean_prompt_tokens=64, mean_output_tokens=16))[:24]
refs = {}
for i, it in enumerate(items[:10]):
    refs[i] = orc.greedy(prompt_token_ids(i, it.prompt_tokens, arch.vocab).long(), it.output_tokens)[0]
for graphs, split, ser in ((False, None, True), (False, None, False), (True, 72, False)):
    ex = B200Executor(arch, weights=w, max_batch=32, chunk_tokens=32, num_blocks=600, max_context=1024, num_slots=64,
                      static_decode_sms=split, use_graphs=graphs, serialize_phases=ser)
    ex.warmup()
    model = arch.model_spec()
    eng = lambda: RapidEngine(model, b200_spec(), CostParams(), SloSpec(itl_slo_us=50_000), chunk_tokens=32,
                              max_batch=32, executor=ex)
    res = run_items("rapid", items, model, b200_spec(), CostParams(), SloSpec(itl_slo_us=50_000), engine_factory=eng)
    bad = [i for i in refs if ex.generated.get(i) != refs[i]]
    print(f"graphs={graphs} split={split} ser={ser} bad={bad}", flush=True)
    for i in bad[:3]:
        print("  req", i, "P", items[i].prompt_tokens, "O", items[i].output_tokens, "gpu", ex.generated.get(i)[:8], "ref", refs[i][:8])
    ex.close()

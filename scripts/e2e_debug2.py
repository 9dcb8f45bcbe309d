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
print("P/O:", [(i.prompt_tokens, i.output_tokens) for i in items[:12]])
refs = {i: orc.greedy(prompt_token_ids(i, it.prompt_tokens, arch.vocab).long(), it.output_tokens)[0]
        for i, it in enumerate(items[:12])}
ex = B200Executor(arch, weights=w, max_batch=32, chunk_tokens=32, num_blocks=600, max_context=1024, num_slots=64,
                  use_graphs=False, serialize_phases=True)
orig_fd = ex.finish_decode
orig_lp = ex.launch_prefill
state = {"step": 0, "done": False}
def lp(req, written, chunk, target, decision, co):
    if req.id < 12 and not state["done"]:
        print(f"prefill req {req.id} slot {ex._slot_of[req.id]} written {written} chunk {chunk} target {target} pages {ex.engine.pool.block_ids(req.id)[:6]}")
    return orig_lp(req, written, chunk, target, decision, co)
def fd(h):
    orig_fd(h)
    state["step"] += 1
    if state["done"]:
        return
    torch.cuda.synchronize()
    for r, lame in zip(h.members, h.lame):
        if r.id in refs and not lame:
            g = ex.generated[r.id]
            k = len(g)
            if g[-1] != refs[r.id][k - 1]:
                state["done"] = True
                slot = ex._slot_of[r.id]
                print(f"MISMATCH step {state['step']} req {r.id} k {k} P {r.prompt_tokens} slot {slot} got {g[-1]} want {refs[r.id][k-1]}")
                print("  members:", [(m.id, ex._slot_of.get(m.id), m.context_tokens, l) for m, l in zip(h.members, h.lame)])
                print("  pool pages:", {m.id: ex.engine.pool.block_ids(m.id)[:6] for m in h.members})
                print("  bt rows:", {m.id: ex.runner.block_table[ex._slot_of[m.id], :6].tolist() for m in h.members})
                print("  dec in:", ex._dec_in_dev[:, :len(h.members)].tolist())
                pool = ex.engine.pool
                live = {rid: (s_, pool.block_ids(rid)) for rid, s_ in ex._slot_of.items() if pool.holds(rid)}
                for rid, (s_, ids) in live.items():
                    row = ex.runner.block_table[s_, :8].tolist()
                    print(f"  live req {rid} slot {s_} pages {ids[:8]} bt {row}")
                # KV of req r vs oracle
                prompt = prompt_token_ids(r.id, r.prompt_tokens, arch.vocab).long()
                seq = torch.cat([prompt, torch.tensor(refs[r.id][:k])])
                _, kv = orc.forward(seq[: r.prompt_tokens + k - 1], 0, None)
                K0 = kv[0][0]  # layer 0 keys [n, Hkv, D]
                ids = pool.block_ids(r.id)
                cache = ex.runner.kv[0]
                for p_ in range(K0.shape[0]):
                    page = ids[p_ // 16]
                    got = cache[page, 0, :, p_ % 16].float().cpu()
                    err = float((got - K0[p_]).norm() / K0[p_].norm())
                    if err > 2e-2:
                        print(f"   K pos {p_} page {page} off {p_%16} err {err:.3f}")
                return
ex.finish_decode = fd
ex.launch_prefill = lp
model = arch.model_spec()
eng = lambda: RapidEngine(model, b200_spec(), CostParams(), SloSpec(itl_slo_us=50_000), chunk_tokens=32,
                          max_batch=32, executor=ex)
res = run_items("rapid", items, model, b200_spec(), CostParams(), SloSpec(itl_slo_us=50_000), engine_factory=eng)
print("done", state)
os._exit(0)

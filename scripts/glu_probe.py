import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa
from scripts.kbench import timeit  # noqa
dev = "cuda"
sc = ops.GemmScratch(dev)
lib = ops.load()
flush = torch.empty(256 << 20, dtype=torch.int8, device=dev)
for (T, sms) in [(128, 72), (256, 72), (64, 72), (1023, 76)]:
    K, I = 4096, 14336
    x = torch.randn(T, K, device=dev).bfloat16()
    w = (torch.randn(2 * I, K, device=dev) * 0.02).bfloat16()
    y2 = torch.empty(T, 2 * I, device=dev, dtype=torch.bfloat16)
    y1 = torch.empty(T, I, device=dev, dtype=torch.bfloat16)
    a = torch.empty(T, I, device=dev, dtype=torch.bfloat16)
    st = lambda: torch.cuda.current_stream().cuda_stream
    def plain():
        ops.linear(x, w, out=y2, num_sms=sms, scratch=sc)
        ops.silu_mul(y2, a)
    def glu():
        lib.rb_gemm_bf16(x.data_ptr(), w.data_ptr(), y1.data_ptr(), None, None, T, 2 * I, K, K, K, I, 4, sms,
                         sc.ws.data_ptr(), sc.ws_bytes, sc.counters.data_ptr(), sc.counters.numel(), st())
    def gemm_only():
        ops.linear(x, w, out=y2, num_sms=sms, scratch=sc)
    f = flush if T <= 256 else None
    print(json.dumps(dict(T=T, sms=sms, plain_us=round(timeit(plain, flush=f) * 1e3, 1),
                          gemm_only_us=round(timeit(gemm_only, flush=f) * 1e3, 1),
                          glu_us=round(timeit(glu, flush=f) * 1e3, 1))), flush=True)

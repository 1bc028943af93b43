import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
from paper_2406_17145_b200.runtime import lib
from tools.bench_gemm import timeit
dev = torch.device("cuda", 0)
T = 8192
for (N, K) in [(1024, 64), (1024, 128), (1024, 1024), (4096, 64), (4096, 1024)]:
    x = torch.randn(T, K, device=dev).bfloat16(); w = (torch.randn(N, K, device=dev) / 32).bfloat16()
    y = torch.empty(T, N, device=dev, dtype=torch.bfloat16); res = torch.randn(T, N, device=dev).bfloat16()
    b = torch.zeros(N, device=dev); pre = torch.empty_like(y)
    r = {"shape": [T, N, K]}
    r["plain"] = round(timeit(lambda: lib.linear_fwd(y, x, w, bias=None, act="none"), 20), 1)
    r["residual"] = round(timeit(lambda: lib.linear_fwd(y, x, w, bias=b, act="none", residual=res), 20), 1)
    r["gelu_pre"] = round(timeit(lambda: lib.linear_fwd(y, x, w, bias=b, act="gelu", pre=pre), 20), 1)
    r["cublas"] = round(timeit(lambda: torch.matmul(x, w.t()), 20), 1)
    print(json.dumps(r))

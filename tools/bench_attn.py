"""MMT attention kernels alone at the MMT step's shape (B = 16 samples x 16 heads, S = 512,
head dim 64), CUDA-graph replay (true per-launch time): the recompute kernels
(csrc/attn_flash_sm100.cu) vs the P-storing kernels (csrc/attn_sm100.cu) + the dV / dK
batched GEMMs, with algorithmic TFLOP/s (fw 4 S^2 dh per head; bw 10 S^2 dh with the
recompute, 8 S^2 dh without).

    python tools/bench_attn.py [--m 16]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2406_17145_b200.runtime import lib
from paper_2406_17145_b200.runtime.mmt import _spec
from paper_2406_17145_b200.runtime.profiler import _time_us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--S", type=int, default=512)
    ap.add_argument("--H", type=int, default=16)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    m, S, H = a.m, a.S, a.H
    d, dh, T, Z = 64 * H, 64, m * S, m * H
    qkv = torch.randn(T, 3 * d, device=dev).bfloat16()
    dout = torch.randn(T, d, device=dev).bfloat16()
    o = torch.empty(T, d, device=dev, dtype=torch.bfloat16)
    dqkv = torch.empty(T, 3 * d, device=dev, dtype=torch.bfloat16)
    lse = torch.empty(Z * S, device=dev)
    dvec = torch.empty(Z * S, device=dev)
    P = torch.empty(Z * S, S, device=dev, dtype=torch.bfloat16)
    dS = torch.empty(Z * S, S, device=dev, dtype=torch.bfloat16)
    sc = 0.125
    f_fw, f_bw = 4.0 * S * S * dh * Z, 10.0 * S * S * dh * Z
    r = {}
    r["flash_fwd_us"] = _time_us(lambda: lib.flash_attn_fwd(qkv, lse, o, m, S, d, H, sc), 10)
    r["flash_bwd_us"] = _time_us(lambda: lib.flash_attn_bwd(qkv, lse, o, dout, dvec, dqkv, m, S, d, H, sc), 10)
    r["stored_p_fwd_us"] = _time_us(lambda: lib.attn_fwd(qkv, P, o, m, S, d, H, sc), 10)

    def old_bw():
        lib.gemm_batched(dqkv, 3 * d, P, S, Z * S, True, dout, d, T, True, S, dh, S,
                         _spec(Z, H, a_k_hi=H * S, a_k_lo=S, b_n_lo=dh, b_k_hi=S, c0=2 * d, c_hi=S * 3 * d, c_lo=dh))
        lib.attn_bwd(qkv, P, o, dout, dS, dqkv, m, S, d, H, sc)
        lib.gemm_batched(dqkv, 3 * d, dS, S, Z * S, True, qkv, 3 * d, T, True, S, dh, S,
                         _spec(Z, H, a_k_hi=H * S, a_k_lo=S, b_n_lo=dh, b_k_hi=S, c0=d, c_hi=S * 3 * d, c_lo=dh))

    r["stored_p_bwd_us"] = _time_us(old_bw, 10)
    r["flash_fwd_tflops"] = round(f_fw / r["flash_fwd_us"] / 1e6, 1)
    r["flash_bwd_tflops"] = round(f_bw / r["flash_bwd_us"] / 1e6, 1)
    r["shape"] = {"m": m, "S": S, "H": H, "Z": Z}
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()}))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Context for the FP8 roofline (run on the GPU box): cuBLAS FP8 (torch._scaled_mm, E4M3, fp32
accumulate, bf16 out) on a dense GEMM of the same flops as the MoE configs and on 8192^3, clean L2
before every launch, CUDA events, median of 20."""
import json
import statistics

import torch


def timed(fn, reps=20):
    w = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    r = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
    for _ in range(3):
        fn()
    out = []
    for _ in range(reps):
        w.zero_()
        r.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)
        a.record()
        fn()
        b.record()
        b.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


def main():
    one = torch.tensor(1.0, device="cuda")
    for name, M, N, K in (("mix-equivalent", 8192, 14336, 4096), ("ds-equivalent", 49152, 1408, 2048),
                          ("8192^3", 8192, 8192, 8192)):
        A = (torch.randn(M, K, device="cuda") * 0.5).to(torch.float8_e4m3fn)
        B = (torch.randn(N, K, device="cuda") * 0.5).to(torch.float8_e4m3fn).t()     # column-major K x N
        ms = timed(lambda: torch._scaled_mm(A, B, scale_a=one, scale_b=one, out_dtype=torch.bfloat16))
        Ab, Bb = A.to(torch.bfloat16), B.to(torch.bfloat16)
        ms_bf16 = timed(lambda: Ab @ Bb)
        print(json.dumps({"shape": name, "M": M, "N": N, "K": K, "fp8_ms": ms, "fp8_tflops": 2 * M * N * K / ms / 1e9,
                          "bf16_ms": ms_bf16, "bf16_tflops": 2 * M * N * K / ms_bf16 / 1e9}), flush=True)


if __name__ == "__main__":
    main()

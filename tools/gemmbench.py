#!/usr/bin/env python3
"""Prefill GEMM throughput (hs_gemm3_tc) at the Llama2-7B layer shapes:
CUDA-event device time per call, useful TFLOP/s (2*R*N*K) and tensor TFLOP/s
(x3 activation planes).

    python tools/gemmbench.py [--rows 2048]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=2048)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    from paper_2404_11912_b200._abi import check, lib
    from paper_2404_11912_b200.runtime import ptr, stream_ptr
    R = a.rows
    out = {}
    for name, N, K in (("wqkv", 12288, 4096), ("wo", 4096, 4096), ("wgu", 22016, 4096), ("wdown", 4096, 11008),
                       ("head", 32000, 4096)):
        ld = (K + 63) // 64 * 64
        planes = [torch.randn((R, ld), device="cuda").to(torch.bfloat16) for _ in range(3)]
        W = (torch.randn((N, ld), device="cuda") * 0.02).to(torch.bfloat16)
        y = torch.zeros((R, N), device="cuda")
        args = (ptr(planes[0]), ptr(planes[1]), ptr(planes[2]), ld, R, ptr(W), ld, N, ptr(y), N, 0, stream_ptr())
        check(lib.hs_gemm3_tc(*args))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.reps):
            check(lib.hs_gemm3_tc(*args))
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / a.reps
        fl = 2.0 * R * N * K
        out[name] = {"us": us, "useful_TFLOPs": fl / us / 1e6, "tensor_TFLOPs": 3 * fl / us / 1e6}
        print(json.dumps({name: out[name]}), flush=True)


if __name__ == "__main__":
    main()

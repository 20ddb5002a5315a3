#!/usr/bin/env python3
"""Is a GEMV launch bound by HBM or by its own pipeline latency?  Times one
weight matrix of the Llama2-7B shape (t = 3) with the weights cold (an
L2-sized buffer written in between) and L2-resident (the same launch twice
back to back; every matrix but gate|up fits the 126 MB L2).  CUDA events on
the launching stream.

    python tools/l2probe.py
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    import paper_2404_11912_b200  # noqa: F401
    from paper_2404_11912_b200._abi import check, lib
    from paper_2404_11912_b200.runtime import ptr, stream_ptr
    s = stream_ptr()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    out = {}
    for name, N, K, epi in (("wqkv", 12288, 4096, 0), ("wo", 4096, 4096, 1), ("wdown", 4096, 11008, 1),
                            ("wgu", 22016, 4096, 2), ("small_wo_draft", 768, 768, 1)):
        W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        xs = torch.zeros((24, K), dtype=torch.bfloat16, device="cuda")
        xo = torch.zeros((24, max(K, N)), dtype=torch.bfloat16, device="cuda")
        y = torch.zeros((8, N), device="cuda")
        wsb = lib.hs_gemv_tc_workspace_bytes(N, K)
        ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")

        def run():
            check(lib.hs_gemv_tc(ptr(xs), 3, ptr(W), K, N, epi, ptr(y) if epi != 2 else None, N,
                                 ptr(xo) if epi == 2 else None, max(K, N) // 2 if epi == 2 else 0, ptr(ws), wsb, s))
        res = {}
        for mode in ("cold", "warm"):
            ts = []
            for _ in range(10):
                flush.fill_(1)
                if mode == "warm":
                    run()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            ts.sort()
            res[mode + "_us"] = ts[len(ts) // 2]
        res["MB"] = N * K * 2 / 1e6
        res["cold_TBps"] = res["MB"] / res["cold_us"] / 1e6 * 1e6 / 1e6
        out[name] = res
        print(name, json.dumps(res), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

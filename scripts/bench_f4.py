"""f4 measurement: GEMM + reduce-scatter at prefill scale on the megakernel (one GPU,
TP ranks as k-splits).  Per variant: ms per step, TFLOP/s (2 T N K) against the
measured bf16 peak, and the fused (Event Tensor per output tile) vs stage-barrier
("unfused": reduce only after every GEMM tile) comparison.

    python scripts/bench_f4.py [tokens] [n] [k]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2604_13327_b200.f4 import GemmReduceScatter  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
T = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
N = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
K = int(sys.argv[3]) if len(sys.argv) > 3 else 14336
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("bf16_tflops", 1625.0)
g = torch.Generator(device="cuda:0")
g.manual_seed(0)
x = torch.randn(T, K, device="cuda:0", generator=g).to(torch.bfloat16)
w = (torch.randn(N, K, device="cuda:0", generator=g) / K ** 0.5).to(torch.bfloat16)
ref = None
for ranks in (2, 8):
    for barrier in (False, True):
        m = GemmReduceScatter(tokens=T, n=N, k=K, ranks=ranks, x=x, w=w, stage_barriers=barrier)
        for _ in range(2):
            m.step()
        if ref is None:
            ref = m.reference()
        err = ((m.out.float() - ref).abs().max() / ref.abs().max()).item()
        ts = [m.executor.run({})["kernel_ms"] for _ in range(6)]
        ms = statistics.median(ts)
        tf = m.flops() / (ms * 1e-3) / 1e12
        print(json.dumps({"workload": f"gemm+reduce-scatter T={T} N={N} K={K}", "ranks": ranks,
                          "variant": "stage-barrier" if barrier else "event-tensor", "ms": round(ms, 4),
                          "tflops": round(tf, 1), "frac_of_bf16_peak": round(tf / peak, 3),
                          "rel_err": round(err, 5), "tasks": m.last_stats["tasks_executed"]}), flush=True)
        del m
        torch.cuda.empty_cache()

# ---- all-gather + GEMM (MLP-2 up projection shape: X [T][4096] gathered over 8 chunks)
from paper_2604_13327_b200.f4 import AllGatherGemm  # noqa: E402

NA, KA = 14336, 4096
xa = torch.randn(T, KA, device="cuda:0", generator=g).to(torch.bfloat16)
wa = (torch.randn(NA, KA, device="cuda:0", generator=g) / KA ** 0.5).to(torch.bfloat16)
refa = None
for chunks in (8,):
    m = AllGatherGemm(tokens=T, n=NA, k=KA, chunks=chunks, x=xa, w=wa)
    for _ in range(2):
        m.step()
    if refa is None:
        refa = m.reference()
    err = ((m.out - refa).abs().max() / refa.abs().max()).item()
    ts = [m.executor.run({})["kernel_ms"] for _ in range(6)]
    ms = statistics.median(ts)
    tf = m.flops() / (ms * 1e-3) / 1e12
    print(json.dumps({"workload": f"all-gather+gemm T={T} N={NA} K={KA}", "chunks": chunks,
                      "variant": "pull (L2 prefetch copies)", "ms": round(ms, 4), "tflops": round(tf, 1),
                      "frac_of_bf16_peak": round(tf / peak, 3), "rel_err": round(err, 6),
                      "tasks": m.last_stats["tasks_executed"]}), flush=True)
    del m
    torch.cuda.empty_cache()

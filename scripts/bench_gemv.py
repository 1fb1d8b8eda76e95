"""Single-call GEMV stage microbenchmark: one Event Tensor call of T tasks
streaming an [N][K] bf16 weight through the megakernel's ring."""
import json, sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_13327_b200 import etsim
from paper_2604_13327_b200.ops import OP_GEMV, EPI_F32, make_op, pack, ptr

def run(N, K, T=148, l2=0, reps=8):
    spec = {"symbols": [], "duration_models": {}, "device_functions": [{"name": "g", "grid": [str(T)], "resource": "sm"}],
            "event_tensors": [], "calls": [{"fn": "g"}]}
    g = etsim.Graph.from_json(json.dumps(spec))
    k = etsim.lower_static(g, [{}], num_sms=T)
    W = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    x = torch.randn(K, device="cuda", dtype=torch.bfloat16)
    y = torch.zeros(N, device="cuda", dtype=torch.float32)
    print("running", N, K, flush=True)
    ex = etsim.Executor(k, num_workers=T, record_trace=False, l2_prefetch=l2, watchdog_ns=500_000_000)
    ex.bind_ops(pack([make_op(OP_GEMV, i=[N, K, 1, 0, EPI_F32, -1, 0, 8], p=[ptr(W), 0, ptr(x), 0, ptr(y)])]))
    ts = [ex.run({})["kernel_ms"] for _ in range(reps)]
    ref = (W.float() @ x.float())
    err = (y - ref).abs().max().item() / ref.abs().max().item()
    t = statistics.median(ts[2:])
    print(f"N={N} K={K} T={T} l2={l2}: {t*1e3:8.1f} us  {N*K*2/t/1e6:7.0f} GB/s  relerr {err:.2e}", flush=True)

if __name__ == "__main__":
    for (N, K) in [(128256, 4096), (28672, 4096), (4096, 14336), (6144, 4096)]:
        run(N, K)

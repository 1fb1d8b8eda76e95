"""Stage timeline of one Qwen3-MoE-shaped layer at batch b (tensor-core variant above 8).
    python scripts/diag_moe_tc.py [b] [scheduler]"""
import collections
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_13327_b200.moe import QWEN3_30B_A3B, MoEDecodeModel  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 32
sched = sys.argv[2] if len(sys.argv) > 2 else "static"
m = MoEDecodeModel(QWEN3_30B_A3B, samples=(1024,), scheduler=sched, record_trace=True, max_batch=max(b, 16),
                   batch_samples=(b,))
m.fill_cache(1024)
m.set_token(list(range(1, max(b, 16) + 1)))
ts = [m.executor.run(m._binding(1024, b))["kernel_ms"] for _ in range(3)]
print("ms", [round(t, 2) for t in ts])
t = m.executor.trace()
calls = m.graph.call_functions
by = collections.defaultdict(list)
for r in t.records:
    by[r["call"]].append(r)
l1 = [c for c in range(len(calls)) if calls[c].startswith("L1.")]
base = min(r["exec"][0] for c in l1 for r in by[c] if not r["noop"])
for c in l1:
    rs = [r for r in by[c] if not r["noop"]]
    if not rs:
        print(f"{calls[c]:10s} all masked ({len(by[c])})")
        continue
    st = sorted(r["exec"][0] - base for r in rs)
    en = sorted(r["exec"][1] - base for r in rs)
    du = sorted(r["exec"][1] - r["exec"][0] for r in rs)
    print(f"{calls[c]:10s} n={len(rs):5d} masked={len(by[c]) - len(rs):5d} start min {st[0]/1e3:8.2f} end max "
          f"{en[-1]/1e3:8.2f}  dur med {du[len(du)//2]/1e3:7.2f} max {du[-1]/1e3:7.2f} us")

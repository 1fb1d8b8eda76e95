import sys, os, collections, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_13327_b200.decode import CONFIGS, DecodeModel
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"]
m = DecodeModel(cfg, samples=(1024,), record_trace=True, l2_prefetch=int(os.environ.get("L2PF", "0")))
m.fill_cache(1024); m.set_token(1)
for _ in range(3): st = m.executor.run({"s": 1024})
print("kernel_ms", st["kernel_ms"])
t = m.executor.trace()
fns = m.graph.call_functions
by = collections.defaultdict(list)
for r in t.records:
    by[r["call"]].append(r)
def show(calls):
    base = min(r["exec"][0] for c in calls for r in by[c])
    for c in calls:
        rs = by[c]
        st = [r["exec"][0] for r in rs]; en = [r["exec"][1] for r in rs]
        ex = [e - s for s, e in zip(st, en)]
        pro = [r["prologue"] for r in rs if r["prologue"] is not None]
        pm = statistics.median(pro) if pro else 0
        print(f"{fns[c]:12s} n={len(rs):4d} start[min {min(st)-base:8.0f} med {statistics.median(st)-base:8.0f}] "
              f"end[med {statistics.median(en)-base:8.0f} max {max(en)-base:8.0f}] exec med {statistics.median(ex):7.0f} max {max(ex):7.0f} prologue med {pm:6.0f}")
show(list(range(1, 14)))
print("layer spans:")
for l in [0, 1, 15, 31]:
    cs = list(range(1 + 6 * l, 7 + 6 * l))
    s0 = min(r["exec"][0] for c in cs for r in by[c]); e0 = max(r["exec"][1] for c in cs for r in by[c])
    print(l, (e0 - s0) / 1e3, "us")
show([len(fns) - 2, len(fns) - 1])

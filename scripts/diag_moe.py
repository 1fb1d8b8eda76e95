"""Stage timeline of one Qwen3-MoE decode layer (static scheduler, trace on; timing experiment)."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_13327_b200.moe import MOE_CONFIGS, MoEDecodeModel  # noqa: E402

cfg = MOE_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "qwen3-30b-a3b"]
sched = sys.argv[2] if len(sys.argv) > 2 else "static"
m = MoEDecodeModel(cfg, samples=(1024,), record_trace=True, scheduler=sched)
m.fill_cache(1024)
m.set_token(1)
for _ in range(3):
    st = m.executor.run({"s": 1024})
print("kernel_ms", st["kernel_ms"])
t = m.executor.trace()
calls = m.graph.call_functions
by = collections.defaultdict(list)
for r in t.records:
    by[r["call"]].append(r)
for L in (1, 20):
    cs = [c for c in range(len(calls)) if calls[c].startswith(f"L{L}.")]
    base = min(r["exec"][0] for c in cs for r in by[c] if not r["noop"])
    for c in cs:
        rs = [r for r in by[c] if not r["noop"]]
        if not rs:
            continue
        st_ = sorted(r["exec"][0] - base for r in rs)
        en = sorted(r["exec"][1] - base for r in rs)
        ex = sorted(r["exec"][1] - r["exec"][0] for r in rs)
        print(f"{calls[c]:12s} n={len(rs):4d} start min {st_[0]/1e3:7.2f} med {st_[len(st_)//2]/1e3:7.2f}  end med "
              f"{en[len(en)//2]/1e3:7.2f} max {en[-1]/1e3:7.2f}  exec med {ex[len(ex)//2]/1e3:6.2f} max {ex[-1]/1e3:6.2f}")

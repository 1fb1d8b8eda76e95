"""Dynamic scheduler hop anatomy (timing experiment): for each call of one layer,
relative to the previous call's last exec end: when its tasks were pushed, popped
(t_begin), finished waiting (t_wait_end) and notified.

    python scripts/diag_dyn_hops.py [layer]
"""
import collections
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_13327_b200.moe import MOE_CONFIGS, MoEDecodeModel  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 24
m = MoEDecodeModel(MOE_CONFIGS["qwen3-30b-a3b"], samples=(1024,), scheduler="dynamic", record_trace=True)
m.fill_cache(1024, seed=1)
m.set_token([1])
if len(sys.argv) > 2:
    m.executor.set_debug(int(sys.argv[2], 0))
for _ in range(4):
    st = m.executor.run(m._binding(1024, 1))
print("step ms", st["kernel_ms"])
recs = m.executor.raw_trace()
calls = m.graph.call_functions
t = m.executor.trace()
by = collections.defaultdict(list)
for rec, tr in zip(recs, t.records):
    by[tr["call"]].append(rec)
cs = [c for c in range(len(calls)) if calls[c].startswith(f"L{L}.")] + \
     [c for c in range(len(calls)) if calls[c].startswith(f"L{L + 1}.")][:1]
prev_end = prev_notify = None
for c in cs:
    rs = [r for r in by[c] if not (r[7] & 1)]
    if not rs:
        continue
    med = lambda xs: statistics.median(xs)
    push = [r[0] for r in rs if r[0] > 0]
    pop = [r[1] for r in rs]
    tw = [r[2] for r in rs]
    te = [r[4] for r in rs]
    tn = [r[5] for r in rs]
    if prev_end is not None:
        f = lambda xs: (min(xs) - prev_end) / 1e3
        print(f"{calls[c]:12s} n={len(rs):4d}  from prev last exec end: push first {f(push) if push else float('nan'):6.2f} "
              f"pop first {f(pop):6.2f} med {(med(pop) - prev_end) / 1e3:6.2f}  wait-end first {f(tw):6.2f}   "
              f"[prev last notify-end {(prev_notify - prev_end) / 1e3:5.2f}]  pop->waitend med {med([b - a for a, b in zip(pop, tw)]) / 1e3:5.2f}")
    if len(sys.argv) > 2:  # probe: push_time field holds the probe stamp of each task's finish
        last = max(rs, key=lambda r: r[4])
        print(f"   last task's finish probe {(last[0] - last[4]) / 1e3:6.2f} us after its exec end, notify-end "
              f"{(last[5] - last[4]) / 1e3:6.2f}")
    prev_end = max(te)
    prev_notify = max(tn)

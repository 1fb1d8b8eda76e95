"""Where does a decode step lose time?  (timing experiment, not a test)

  normal      : the step as benchmarked
  nowait      : ET_DEBUG=1, Event Tensor waits skipped -> pure streaming time of the same task layout
  stall       : ET_DEBUG=2 + trace: per call, median consumer ring-stall (warp 0) vs exec time
"""
import collections
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_13327_b200.decode import CONFIGS, DecodeModel  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"]
m = DecodeModel(cfg, samples=(1024,), record_trace=True)
m.fill_cache(1024)
m.set_token(1)


def timed(n=5):
    ts = [m.executor.run({"s": 1024})["kernel_ms"] for _ in range(n)]
    return statistics.median(ts[1:])


m.executor.set_debug(int("0"))
print("normal  ms", timed())
m.executor.set_debug(int("1"))
print("nowait  ms", timed())
m.executor.set_debug(int("4"))
print("nohbm   ms", timed())
m.executor.set_debug(int("5"))
print("nohbm+nowait ms", timed())
for f in ("16", "32", "48", "20", "36", "52"):
    m.executor.set_debug(int(f))
    print("flags", f, "ms", timed())
m.executor.set_debug(int("12"))
print("nohbm+busy ms", timed())
recs_nohbm = m.executor.raw_trace()
m.executor.set_debug(int("2"))
print("stall   ms", timed())
recs = m.executor.raw_trace()
calls = m.graph.call_functions
slot_call = m.kernel.sample_queues(0) if False else None
t = m.executor.trace()
by = collections.defaultdict(list)
for rec, tr in zip(recs, t.records):
    by[tr["call"]].append((rec, tr))
for c in list(range(1, 8)) + [len(calls) - 1]:
    rows = by[c]
    ex = [r[4] - r[2] for r, _ in rows if not (r[7] & 1)]
    st = [r[9] for r, _ in rows if not (r[7] & 1)]
    pro = [r[3] - r[2] for r, _ in rows if r[3] > 0]
    ex2 = [r[4] - r[2] for r in recs_nohbm if r[8] in {rr[8] for rr, _ in rows} and not (r[7] & 1)]
    bz = [r[9] for r in recs_nohbm if r[8] in {rr[8] for rr, _ in rows} and not (r[7] & 1)]
    print(f"   no-hbm exec med {statistics.median(ex2):8.0f}  busy(warp0) med {statistics.median(bz):8.0f}")
    print(f"{calls[c]:10s} n={len(rows):4d} exec med {statistics.median(ex):8.0f} max {max(ex):8.0f}  "
          f"ring-stall med {statistics.median(st):8.0f} max {max(st):8.0f}  prologue med "
          f"{statistics.median(pro) if pro else 0:6.0f}")

# stage timeline of layer 1 (normal run, trace on)
m.executor.set_debug(int("0"))
timed(3)
t = m.executor.trace()
by = collections.defaultdict(list)
for r in t.records:
    by[r["call"]].append(r)
names = {c: calls[c] for c in range(len(calls))}
l1 = [c for c in range(len(calls)) if calls[c].startswith("L1.")]
base = min(r["exec"][0] for c in l1 for r in by[c])
for c in l1 + [c for c in range(len(calls)) if calls[c].startswith("L2.")][:1]:
    rs = [r for r in by[c] if not r["noop"]]
    st = sorted(r["exec"][0] - base for r in rs)
    en = sorted(r["exec"][1] - base for r in rs)
    print(f"{calls[c]:10s} start min {st[0]/1e3:7.2f} med {st[len(st)//2]/1e3:7.2f}   end med {en[len(en)//2]/1e3:7.2f} "
          f"max {en[-1]/1e3:7.2f}  (us)")

"""Stage timeline of the batched (tensor-core GEMV) decode: per call of layer 1,
start/end of its tasks relative to the layer start, plus whole-step times with
Event Tensor waits skipped (ET_DEBUG=1) and with HBM traffic removed (ET_DEBUG=4).
    python scripts/diag_batch.py [b] [s]"""
import collections
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_13327_b200.batch import BatchDecodeModel  # noqa: E402
from paper_2604_13327_b200.decode import CONFIGS  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 1
s = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
cfg = CONFIGS["llama3-8b"]
m = BatchDecodeModel(cfg, samples=(s,), max_batch=64, record_trace=True)
m.fill_cache(s)
m.set_token(1)


def timed(n=4):
    ts = [m.executor.run({"s": s, "b": b})["kernel_ms"] for _ in range(n)]
    return statistics.median(ts[1:])


for dbg in ("0", "1", "4", "64", "68", "324"):
    m.executor.set_debug(int(dbg))
    print("ET_DEBUG", dbg, "ms", round(timed(), 3), flush=True)
m.executor.set_debug(int(os.environ.get("TL_DEBUG", "0")))  # timeline under this ET_DEBUG
timed(2)
t = m.executor.trace()
calls = m.graph.call_functions
by = collections.defaultdict(list)
for r in t.records:
    by[r["call"]].append(r)
l1 = [c for c in range(len(calls)) if calls[c].startswith("L1.")]
base = min(r["exec"][0] for c in l1 for r in by[c])
for c in l1:
    rs = [r for r in by[c] if not r["noop"]]
    st = sorted(r["exec"][0] - base for r in rs)
    en = sorted(r["exec"][1] - base for r in rs)
    du = sorted(r["exec"][1] - r["exec"][0] for r in rs)
    print(f"{calls[c]:10s} n={len(rs):4d} start min {st[0]/1e3:8.2f} med {st[len(st)//2]/1e3:8.2f}  end med "
          f"{en[len(en)//2]/1e3:8.2f} max {en[-1]/1e3:8.2f}  dur med {du[len(du)//2]/1e3:7.2f} max {du[-1]/1e3:7.2f} us")

recs_of = {}
for dbg in ("2", "8", "514", "6"):
    m.executor.set_debug(int(dbg))
    timed(2)
    recs_of[dbg] = m.executor.raw_trace()
t = m.executor.trace()
for c in l1:
    idx = [i for i, r in enumerate(t.records) if r["call"] == c and not r["noop"]]
    row = f"{calls[c]:10s}"
    for dbg, name in (("2", "ring-stall"), ("8", "busy"), ("514", "x-wait"), ("6", "ring-stall(nohbm)")):
        v = sorted(recs_of[dbg][i][9] for i in idx)
        row += f"  {name} med {v[len(v)//2]/1e3:7.2f}"
    print(row + " us")

# attention task phases (normal run): wait-end -> split work done (t_prologue stamp) -> exec end
m.executor.set_debug(0)
timed(2)
raw = m.executor.raw_trace()
t = m.executor.trace()
ca = [c for c in range(len(calls)) if calls[c] == "L1.attn"][0]
ph1, ph2 = [], []
for rec, tr in zip(raw, t.records):
    if tr["call"] == ca and not tr["noop"] and rec[3] > 0:
        ph1.append(rec[3] - rec[2])
        ph2.append(rec[4] - rec[3])
ph1.sort()
ph2.sort()
print(f"attn split phase med {ph1[len(ph1)//2]/1e3:.2f} us, merge+arrival phase med {ph2[len(ph2)//2]/1e3:.2f} us "
      f"max {ph2[-1]/1e3:.2f}")
for name in ("L1.attn", "L1.gateup", "L1.qkv"):
    ci = [c for c in range(len(calls)) if calls[c] == name][0]
    w, x = [], []
    for rec, tr in zip(raw, t.records):
        if tr["call"] == ci and not tr["noop"]:
            w.append(rec[2] - rec[1])
            x.append(rec[4] - rec[2])
    w.sort()
    x.sort()
    print(f"{name}: dependency wait med {w[len(w)//2]/1e3:.2f} max {w[-1]/1e3:.2f} us; work med {x[len(x)//2]/1e3:.2f} "
          f"max {x[-1]/1e3:.2f} us; exec field {t.records[0]['exec']}")

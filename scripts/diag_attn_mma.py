"""Per-phase time of the batched tensor-core attention tasks (ET_DEBUG 4096 + trace):
ring waits, barriers, compute, summed by thread 0 over a task's blocks.
    python scripts/diag_attn_mma.py [b] [s]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_13327_b200.batch import BatchDecodeModel  # noqa: E402
from paper_2604_13327_b200.decode import CONFIGS  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 64
s = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
m = BatchDecodeModel(CONFIGS["llama3-8b"], samples=(s,), max_batch=64, record_trace=True)
m.fill_cache(s)
m.set_token(1)
calls = m.graph.call_functions
ca = [c for c in range(len(calls)) if calls[c] == "L1.attn"][0]
for dbg, name in (("4098", "ring waits"), ("4104", "barriers"), ("4608", "compute"),
                  ("37376", "compute (no MMA)")):
    m.executor.set_debug(int(dbg))
    for _ in range(2):
        m.executor.run({"s": s, "b": b})
    raw = m.executor.raw_trace()
    t = m.executor.trace()
    v = sorted(rec[9] for rec, tr in zip(raw, t.records) if tr["call"] == ca and not tr["noop"])
    w = sorted(rec[4] - rec[2] for rec, tr in zip(raw, t.records) if tr["call"] == ca and not tr["noop"])
    print(f"{name:11s} med {v[len(v)//2]/1e3:7.2f} us of task work med {w[len(w)//2]/1e3:7.2f} us (n={len(v)})")

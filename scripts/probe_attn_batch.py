"""Phases of the batched (tensor-core instantiation) attention tasks of layer 1:
wait end -> q staged (debug bit 0x1000), wait end -> split work done (default
stamp), and the rest (arrival + merge).  Timing probe, not a test.
    python scripts/probe_attn_batch.py [b] [s]"""
import os
import statistics
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
for dbg, name in ((0x1000, "q staged"), (0, "split work done")):
    m.executor.set_debug(dbg)
    for _ in range(3):
        st = m.executor.run({"s": s, "b": b})
    raw = m.executor.raw_trace()
    t = m.executor.trace()
    ph1, ph2, tot = [], [], []
    for rec, tr in zip(raw, t.records):
        if tr["call"] == ca and not tr["noop"] and rec[3] > 0:
            ph1.append(rec[3] - rec[2])
            ph2.append(rec[4] - rec[3])
            tot.append(rec[4] - rec[2])
    print(f"b={b} s={s} kernel {st['kernel_ms']:.3f} ms  [{name}] wait-end -> stamp med {statistics.median(ph1)/1e3:.2f} us, "
          f"stamp -> end med {statistics.median(ph2)/1e3:.2f} us, task med {statistics.median(tot)/1e3:.2f} us (n={len(tot)})",
          flush=True)

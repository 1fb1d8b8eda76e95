"""Fused attention merge phases (ET_DEBUG=16; timing experiment): per merger, split
work done -> arrival observed -> merge done."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_13327_b200.decode import CONFIGS, DecodeModel  # noqa: E402

os.environ["ET_DEBUG"] = "16"
m = DecodeModel(CONFIGS["llama3-8b"], samples=(1024,), record_trace=True)
m.fill_cache(1024)
m.set_token(1)
for _ in range(3):
    m.executor.run({"s": 1024})
raw = m.executor.raw_trace()
t = m.executor.trace()
calls = m.graph.call_functions
c = calls.index("L1.attn")
rows = [(rec, tr) for rec, tr in zip(raw, t.records) if tr["call"] == c]
base = min(rec[2] for rec, _ in rows)
for rec, tr in sorted(rows, key=lambda x: x[0][4]):
    if rec[9] > 0:  # mergers: pad = arrival round trip
        t_wait, t_split, t_end = rec[2] - base, rec[3] - base, rec[4] - base
        print(f"group {tr['coord'][0]}: wait_end {t_wait/1e3:6.2f} split_done {t_split/1e3:6.2f} "
              f"arrival_rt {rec[9]/1e3:5.2f} merge {((t_end - t_split) - rec[9])/1e3:5.2f} end {t_end/1e3:6.2f}")

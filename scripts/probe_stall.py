"""Per-call ring stall (debug bit 2) and prologue stamps under debug probe bits (timing experiment).

    python scripts/probe_stall.py [bits ...]
"""
import os, sys, statistics, collections
sys.path.insert(0, "/root/repo")
from paper_2604_13327_b200.decode import LLAMA3_8B, DecodeModel
if os.environ.get("MODEL") == "moe":
    from paper_2604_13327_b200.moe import MOE_CONFIGS, MoEDecodeModel
    m = MoEDecodeModel(MOE_CONFIGS["qwen3-30b-a3b"], samples=(1024,), scheduler="static", record_trace=True)
    m.fill_cache(1024, seed=1); m.set_token([1])
    BIND = m._binding(1024, 1)
else:
    m = DecodeModel(LLAMA3_8B, samples=(1024,), record_trace=True)
    m.fill_cache(1024); m.set_token(1)
    BIND = {"s": 1024}
ex = m.executor
calls = m.graph.call_functions
for bits in [int(x, 0) for x in sys.argv[1:]] or (2, 2 | 0x2000, 4 | 0x2000, 2 | 4):
    ex.set_debug(bits)
    for _ in range(4): ms = ex.run(BIND)["kernel_ms"]
    recs = ex.raw_trace(); t = ex.trace()
    agg = collections.defaultdict(list); pro = collections.defaultdict(list)
    for rec, tr in zip(recs, t.records):
        if tr["noop"]: continue
        key = calls[tr["call"]].split(".")[-1]
        agg[key].append(rec[9] / 1e3)
        if tr["prologue"] is not None: pro[key].append(tr["prologue"] / 1e3)
    print("bits", hex(bits), "ms", round(ms, 3))
    for k in agg:
        v = sorted(agg[k]); p = sorted(pro[k]) or [0]
        print(f"   {k:8s} pad(stall us) med {v[len(v)//2]:6.2f} p90 {v[int(.9*len(v))]:6.2f}   pro med {p[len(p)//2]:6.2f}")

"""Phases of the Qwen3-30B-A3B bs=1 attention split tasks (layer 1, static
scheduler): wait end -> q staged (debug bit 0x1000: q/k-norm + RoPE + k/v append
done), -> first block's scores (0x2000), -> all blocks done (0x4000), -> split
work done (default stamp).  Timing probe, not a test.
    python scripts/probe_attn_moe.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_13327_b200.moe import MOE_CONFIGS, MoEDecodeModel  # noqa: E402

m = MoEDecodeModel(MOE_CONFIGS["qwen3-30b-a3b"], samples=(1024,), scheduler="static", record_trace=True)
m.fill_cache(1024, seed=1)
m.set_token([1])
calls = m.graph.call_functions
ca = [c for c in range(len(calls)) if calls[c] == "L1.attn"][0]
B = m._binding(1024, 1)
for dbg, name in ((0x1000, "q staged"), (0x2000, "block 0 scores"), (0x4000, "blocks done"), (0, "split work done")):
    m.executor.set_debug(dbg)
    for _ in range(3):
        st = m.executor.run(B)
    raw = m.executor.raw_trace()
    t = m.executor.trace()
    ph = [rec[3] - rec[2] for rec, tr in zip(raw, t.records) if tr["call"] == ca and not tr["noop"] and rec[3] > 0]
    tot = [rec[4] - rec[2] for rec, tr in zip(raw, t.records) if tr["call"] == ca and not tr["noop"]]
    print(f"[{name}] wait-end -> stamp med {statistics.median(ph)/1e3:.2f} us; task med "
          f"{statistics.median(tot)/1e3:.2f} us (n={len(tot)}), kernel {st['kernel_ms']:.3f} ms", flush=True)

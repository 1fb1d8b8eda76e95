"""Producer L2 run-ahead window sweep (timing experiment, not a test).

    python scripts/l2_sweep.py [llama|moe|both]

Per window (bytes per worker, 0 = off) the median kernel time of the headline
Llama-3-8B bs=1 s=1024 step and of the Qwen3-30B-A3B bs=1 static step, both on
one lowered artifact each (the window is a per-step knob: et_set_l2_prefetch).
'lsu' rows: the prefetch warp (prefetch.global.L2); 'tma' rows (debug bit 128):
the producer's own cp.async.bulk.prefetch.L2 while the ring is full.
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

WINDOWS = [0, 256 << 10, 512 << 10, 768 << 10, 1 << 20, 1536 << 10, 2 << 20]


def sweep(name, ex, binding, n=12):
    out = {}
    for mode, bits, wins in (("lsu", 0, WINDOWS), ("lsu-stoplazy", 32, WINDOWS[1:5])):
        for w in wins:
            ex.set_debug(bits)
            ex.set_l2_prefetch(w)
            ts = [ex.run(binding)["kernel_ms"] for _ in range(n)]
            key = f"{mode} {w >> 10}K"
            out[key] = round(statistics.median(ts[2:]), 4)
            print(name, key, out[key], flush=True)
    ex.set_debug(0)
    ex.set_l2_prefetch(-1)
    return out


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "both"
    res = {}
    if which in ("llama", "both"):
        from paper_2604_13327_b200.decode import LLAMA3_8B, DecodeModel
        m = DecodeModel(LLAMA3_8B, samples=(1024,))
        m.fill_cache(1024)
        m.set_token(1)
        res["llama3-8b"] = sweep("llama3-8b", m.executor, {"s": 1024})
        del m
        import torch
        torch.cuda.empty_cache()
    if which in ("moe", "both"):
        from paper_2604_13327_b200.moe import MOE_CONFIGS, MoEDecodeModel
        m = MoEDecodeModel(MOE_CONFIGS["qwen3-30b-a3b"], samples=(1024,), scheduler="static")
        m.fill_cache(1024, seed=1)
        m.set_token([1])
        res["qwen3-static"] = sweep("qwen3-static", m.executor, m._binding(1024, 1))
    print(json.dumps(res))


if __name__ == "__main__":
    main()

"""A/B of megakernel debug bits in ONE process (same box, same weights): median
kernel ms of the Llama-3-8B bs=1 step and the Qwen3-30B-A3B bs=1 static step per
bit set, interleaved rounds.  Timing experiment, not a test.

    python scripts/ab_debug.py [llama|moe|both] BITS [BITS ...]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def ab(name, ex, binding, variants, rounds=5, n=6):
    res = {v: [] for v in variants}
    for _ in range(rounds):
        for v in variants:
            ex.set_debug(v)
            ts = [ex.run(binding)["kernel_ms"] for _ in range(n)]
            res[v] += ts[1:]
    ex.set_debug(0)
    for v in variants:
        print(f"{name:14s} bits {v:#8x}  median {statistics.median(res[v]):.4f} ms  min {min(res[v]):.4f}", flush=True)


def main():
    which = sys.argv[1]
    variants = [int(x, 0) for x in sys.argv[2:]] or [0]
    if which in ("llama", "both"):
        from paper_2604_13327_b200.decode import LLAMA3_8B, DecodeModel
        m = DecodeModel(LLAMA3_8B, samples=(1024,))
        m.fill_cache(1024)
        m.set_token(1)
        ab("llama3-8b", m.executor, {"s": 1024}, variants)
        del m
        import torch
        torch.cuda.empty_cache()
    if which in ("moe", "both", "moe-dyn"):
        from paper_2604_13327_b200.moe import MOE_CONFIGS, MoEDecodeModel
        sched = "dynamic" if which == "moe-dyn" else "static"
        m = MoEDecodeModel(MOE_CONFIGS["qwen3-30b-a3b"], samples=(1024,), scheduler=sched)
        m.fill_cache(1024, seed=1)
        m.set_token([1])
        ab(f"qwen3-{sched}", m.executor, m._binding(1024, 1), variants)


if __name__ == "__main__":
    main()

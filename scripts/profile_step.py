"""A few decode steps of one bench workload, for ncu captures (not a benchmark).

    python scripts/profile_step.py [llama3-8b|qwen3-30b-a3b|qwen3-30b-a3b-dynamic] [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

which = sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
if which.startswith("qwen3"):
    from paper_2604_13327_b200.moe import MOE_CONFIGS, MoEDecodeModel
    m = MoEDecodeModel(MOE_CONFIGS["qwen3-30b-a3b"], samples=(1024,),
                       scheduler="dynamic" if which.endswith("dynamic") else "static")
    m.fill_cache(1024, seed=1)
    m.set_token([1])
    b = m._binding(1024, 1)
else:
    from paper_2604_13327_b200.decode import CONFIGS, DecodeModel
    m = DecodeModel(CONFIGS[which], samples=(1024,))
    m.fill_cache(1024)
    m.set_token(1)
    b = {"s": 1024}
for _ in range(steps):
    st = m.executor.run(b)
print("kernel_ms", st["kernel_ms"], flush=True)

"""A/B of the MoE expert row splits (timing experiment):
    python scripts/ab_moe_row_splits.py RS static|dynamic"""
import dataclasses
import statistics
import sys

sys.path.insert(0, '.')
from paper_2604_13327_b200.moe import MOE_CONFIGS, MoEDecodeModel  # noqa: E402

rs, sched = int(sys.argv[1]), sys.argv[2]
cfg = dataclasses.replace(MOE_CONFIGS["qwen3-30b-a3b"], row_splits=rs)
m = MoEDecodeModel(cfg, samples=(1024,), scheduler=sched)
m.fill_cache(1024, seed=1)
m.set_token([1])
B = m._binding(1024, 1)
ts = [m.executor.run(B)["kernel_ms"] for _ in range(30)]
print(f"row_splits={rs} {sched}: median {statistics.median(ts[3:]):.4f} ms min {min(ts[3:]):.4f}", flush=True)

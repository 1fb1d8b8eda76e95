"""A/B of MoE layout options (timing experiment):
    python scripts/ab_moe_head_split.py HS static|dynamic [ROUTE_TASKS]"""
import statistics, sys
sys.path.insert(0, '.')
from paper_2604_13327_b200.moe import MOE_CONFIGS, MoEDecodeModel
hs, sched = int(sys.argv[1]), sys.argv[2]
rt = int(sys.argv[3]) if len(sys.argv) > 3 else None
m = MoEDecodeModel(MOE_CONFIGS["qwen3-30b-a3b"], samples=(1024,), scheduler=sched, head_split=hs, route_tasks=rt)
m.fill_cache(1024, seed=1)
m.set_token([1])
B = m._binding(1024, 1)
ts = [m.executor.run(B)["kernel_ms"] for _ in range(30)]
print(f"head_split={hs} route_tasks={rt} {sched}: median {statistics.median(ts[3:]):.4f} ms min {min(ts[3:]):.4f}", flush=True)

"""Scheduler ablation on real hardware (measurement script), the paper's
static / dynamic / unfused comparison (ref simulate.cpp:682-794 is the
reference's barrier baseline; PAPER.md:818-836 the table):

  static          per-SM queues, fine-grained Event Tensors (the bench path)
  static-barrier  the same program with a barrier Event Tensor between consecutive
                  calls (graphs.add_stage_barriers): stage-by-stage, "unfused"
  dynamic         on-GPU ready queue (Algorithm 2), pushes on completion
  dynamic-early   dynamic with early push (dispatch counters)

for the Llama-3-8B bs=1 step and the Qwen3-30B-A3B bs=1 step (S=1024).
One process per variant; prints one JSON line each.

    python scripts/sched_ablation.py [llama|moe|both]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import json, statistics, sys
sys.path.insert(0, sys.argv[1])
model, kw = sys.argv[2], json.loads(sys.argv[3])
if model == "llama3-8b":
    from paper_2604_13327_b200.decode import CONFIGS, DecodeModel
    m = DecodeModel(CONFIGS["llama3-8b"], samples=(1024,), **kw)
    m.fill_cache(1024); m.set_token(1)
    b = {"s": 1024}
else:
    from paper_2604_13327_b200.moe import MOE_CONFIGS, MoEDecodeModel
    m = MoEDecodeModel(MOE_CONFIGS["qwen3-30b-a3b"], samples=(1024,), **kw)
    m.fill_cache(1024, seed=1); m.set_token([1])
    b = m._binding(1024, 1)
ts = [m.executor.run(b)["kernel_ms"] for _ in range(12)]
st = m.last_stats if hasattr(m, "last_stats") else {}
print(json.dumps({"median_ms": round(statistics.median(ts[2:]), 4), "min_ms": round(min(ts[2:]), 4)}))
'''
VARIANTS = [("static", {"scheduler": "static"}), ("static-barrier", {"scheduler": "static", "stage_barriers": True}),
            ("dynamic", {"scheduler": "dynamic"}), ("dynamic-early", {"scheduler": "dynamic", "early_push": True})]


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "both"
    models = {"llama": ["llama3-8b"], "moe": ["qwen3-30b-a3b"], "both": ["llama3-8b", "qwen3-30b-a3b"]}[which]
    for model in models:
        for name, kw in VARIANTS:
            out = subprocess.run([sys.executable, "-c", CODE, ROOT, model, json.dumps(kw)], capture_output=True, text=True)
            line = [x for x in out.stdout.splitlines() if x.startswith("{")]
            res = json.loads(line[-1]) if line else {"error": out.stderr[-400:]}
            print(json.dumps({"model": model, "variant": name, "kwargs": kw, **res}), flush=True)


if __name__ == "__main__":
    main()

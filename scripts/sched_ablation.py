"""Scheduler ablation on the Llama-3-8B decode step (bs=1, S=1024), the paper's
static-vs-dynamic comparison on real hardware (measurement script): static
per-SM queues (fine-grained and coarse events) vs the on-GPU dynamic scheduler."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import json, statistics, sys
sys.path.insert(0, sys.argv[1])
from paper_2604_13327_b200.decode import CONFIGS, DecodeModel
kw = json.loads(sys.argv[2])
m = DecodeModel(CONFIGS["llama3-8b"], samples=(1024,), **kw)
m.fill_cache(1024); m.set_token(1)
ts = [m.executor.run({"s": 1024})["kernel_ms"] for _ in range(10)]
print(json.dumps({"median_ms": statistics.median(ts[2:])}))
'''
variants = [{"scheduler": "static"}, {"scheduler": "static", "grouped": False},
            {"scheduler": "static", "grouped": False, "fused_merge": False}, {"scheduler": "dynamic"},
            {"scheduler": "dynamic", "early_push": True}]
for v in variants:
    out = subprocess.run([sys.executable, "-c", CODE, ROOT, json.dumps(v)], capture_output=True, text=True)
    line = [x for x in out.stdout.splitlines() if x.startswith("{")]
    print(json.dumps({"variant": v, **(json.loads(line[-1]) if line else {"error": out.stderr[-300:]})}), flush=True)

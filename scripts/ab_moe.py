"""A/B of MoE decode options (separate processes, same box; timing experiment).
    python scripts/ab_moe.py '{"fused_merge": true}' '{"fused_merge": false}' ..."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import json, statistics, sys
sys.path.insert(0, sys.argv[1])
from paper_2604_13327_b200.moe import MOE_CONFIGS, MoEDecodeModel
import dataclasses
kw = json.loads(sys.argv[2])
cfg = MOE_CONFIGS["qwen3-30b-a3b"]
if "attn_chunk" in kw:
    cfg = dataclasses.replace(cfg, attn_chunk=kw.pop("attn_chunk"))
m = MoEDecodeModel(cfg, samples=(1024,), **kw)
m.fill_cache(1024); m.set_token(1)
ts = [m.executor.run({"s": 1024})["kernel_ms"] for _ in range(12)]
print(json.dumps({"median_ms": statistics.median(ts[3:])}))
'''
for rnd in range(2):
    for a in sys.argv[1:]:
        out = subprocess.run([sys.executable, "-c", CODE, ROOT, a], capture_output=True, text=True)
        line = [x for x in out.stdout.splitlines() if x.startswith("{")]
        print(rnd, a, line[-1] if line else out.stderr[-400:], flush=True)

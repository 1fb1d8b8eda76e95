"""Alternate decode-step timings of several package builds (variants/<name>/, made by
scripts/make_variant.sh) in separate processes on the same GPU (timing experiment)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import statistics, sys, json
sys.path.insert(0, sys.argv[1])
from paper_2604_13327_b200.decode import CONFIGS, DecodeModel
m = DecodeModel(CONFIGS[sys.argv[2]], samples=(1024,))
m.fill_cache(1024); m.set_token(1)
ts = [m.executor.run({"s": 1024})["kernel_ms"] for _ in range(15)]
print(json.dumps({"median_ms": statistics.median(ts[3:]), "min_ms": min(ts[3:])}))
'''
CODE_MOE = r'''
import statistics, sys, json
sys.path.insert(0, sys.argv[1])
from paper_2604_13327_b200.moe import MOE_CONFIGS, MoEDecodeModel
m = MoEDecodeModel(MOE_CONFIGS[sys.argv[2]], samples=(1024,), scheduler="static")
m.fill_cache(1024); m.set_token(1)
ts = [m.executor.run({"s": 1024})["kernel_ms"] for _ in range(15)]
print(json.dumps({"median_ms": statistics.median(ts[3:]), "min_ms": min(ts[3:])}))
'''
names = sys.argv[1:] or sorted(os.listdir(os.path.join(ROOT, "variants")))
cfg = os.environ.get("AB_CONFIG", "llama3-8b")
if cfg.startswith("qwen"):  # AB_CONFIG=qwen3-30b-a3b: the MoE decode step (static scheduler)
    CODE = CODE_MOE
for rnd in range(3):
    for n in names:
        out = subprocess.run([sys.executable, "-c", CODE, os.path.join(ROOT, "variants", n), cfg],
                             capture_output=True, text=True)
        line = [x for x in out.stdout.splitlines() if x.startswith("{")]
        print(rnd, n, line[-1] if line else out.stderr[-300:], flush=True)

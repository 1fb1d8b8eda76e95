"""A/B timing of decode-step variants in one process on the same weights (timing experiment).
    python scripts/ab_decode.py [config]"""
import os
import statistics
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_13327_b200.decode import CONFIGS, DecodeModel, init_weights  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"]
W = init_weights(cfg, torch.device("cuda:0"), 0)
variants = [dict(residual="split"), dict(residual="double")]
models = []
for kw in variants:
    m = DecodeModel(cfg, samples=(1024,), weights=W, **kw)
    m.fill_cache(1024)
    m.set_token(1)
    models.append((kw, m))


def clocks():
    try:
        return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                              capture_output=True, text=True).stdout.strip()
    except Exception:
        return "?"


for rnd in range(3):
    for kw, m in models:
        ts = [m.executor.run({"s": 1024})["kernel_ms"] for _ in range(12)]
        print(rnd, kw, "median ms %.4f" % statistics.median(ts[2:]), "min %.4f" % min(ts[2:]), "sm_mhz", clocks(),
              flush=True)

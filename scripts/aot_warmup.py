"""Warmup with and without the ahead-of-time program image (measurement script):
lowering + flatten/upload of the Llama-3-8B bs=1 static program vs loading its
saved image (Executor.save_program / load_program), and the first step after each.

    python scripts/aot_warmup.py [config]
"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2604_13327_b200.decode import CONFIGS, DecodeModel, init_weights  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"]
W = init_weights(cfg, "cuda:0", 0)
path = os.path.join(tempfile.mkdtemp(), "prog.etprog")
out = {}
for label in ("lower+save", "load"):
    t0 = time.perf_counter()
    m = DecodeModel(cfg, samples=(1024,), weights=W, program=path)
    t1 = time.perf_counter()
    m.fill_cache(1024)
    m.set_token(1)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    m.step(1024)
    t3 = time.perf_counter()
    out[label] = {"program_loaded": m.program_loaded, "lower_ms": round(m.lower_ms, 2),
                  "upload_or_load_ms": round(m.upload_ms, 2), "model_ctor_ms": round((t1 - t0) * 1e3, 1),
                  "first_step_ms": round((t3 - t2) * 1e3, 2)}
    del m
    torch.cuda.empty_cache()
out["image_bytes"] = os.path.getsize(path)
print(json.dumps({"config": cfg.name, **out}))

"""Dynamic-shape sweep over the sequence length on ONE compiled artifact (Llama-3-8B
shape, bs=1): the static program is lowered once for the sampled lengths, then
decode steps at arbitrary s <= the largest sample run on the next-larger sample
with masked attention tasks (selection + masking on the device), no recompile or
relaunch of anything but the step kernel.  Prints warmup (lowering + upload +
first step) and per-step latency for each s.  (Measurement script.)"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

t_start = time.perf_counter()
import torch  # noqa: E402

from paper_2604_13327_b200.decode import CONFIGS, DecodeModel  # noqa: E402

samples = (128, 256, 512, 1024, 2048, 4096, 8192)
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"]
m = DecodeModel(cfg, samples=samples, seed=0)
m.fill_cache(8192, seed=1)
m.set_token(1)
m.step(128)
torch.cuda.synchronize()
warm = time.perf_counter() - t_start
print(json.dumps({"workload": f"{cfg.name} bs=1 seq sweep, one artifact", "samples": samples,
                  "warmup_s_first_token": warm, "lower_ms": m.lower_ms, "upload_ms": m.upload_ms}), flush=True)
for s in (3, 128, 200, 1000, 1024, 3000, 5000, 8000, 8192):
    ts = [m.executor.run({"s": s})["kernel_ms"] for _ in range(8)]
    st = m.last_stats if hasattr(m, "last_stats") else {}
    stats = m.executor.run({"s": s})
    print(json.dumps({"s": s, "sample": samples[stats["sample_index"]], "us_per_token": statistics.median(ts[2:]) * 1e3,
                      "tasks": stats["tasks_executed"], "masked_noops": stats["noop_tasks"],
                      "hbm_frac_of_measured": cfg.step_bytes(s) / (statistics.median(ts[2:]) * 1e-3) / 6546.6e9}),
          flush=True)

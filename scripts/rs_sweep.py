"""Qwen3-MoE bs=1 static step time vs expert row splits RS (tasks per routed tile)."""
import dataclasses
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_13327_b200.moe import QWEN3_30B_A3B, MoEDecodeModel, init_moe_weights  # noqa: E402

W = init_moe_weights(QWEN3_30B_A3B, torch.device("cuda:0"), 0)
for rs in [int(x) for x in sys.argv[1:]] or [12, 24, 6]:
    cfg = dataclasses.replace(QWEN3_30B_A3B, row_splits=rs)
    m = MoEDecodeModel(cfg, samples=(1024,), weights=W, scheduler="static")
    m.fill_cache(1024)
    m.set_token(1)
    ts = [m.executor.run({"s": 1024})["kernel_ms"] for _ in range(12)]
    print(f"RS={rs:3d} tasks/tile={rs} median {statistics.median(ts[2:]):.3f} ms", flush=True)
    del m
    torch.cuda.empty_cache()

"""Llama-3-8B-shaped batched decode on the tensor-core GEMV path: one lowered
artifact (batch symbol b <= --max-batch, position symbol s <= max(--seq)) timed
at every (b, s) asked for -- µs/step, tokens/s and the HBM roofline fraction
(algorithmic bytes = weights + b x KV).  One JSON line per (b, s).

    python scripts/bench_batch.py [--batch 1 8 16 32 64] [--seq 1024] [--steps K]
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2604_13327_b200.batch import BatchDecodeModel  # noqa: E402
from paper_2604_13327_b200.decode import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama3-8b")
    ap.add_argument("--batch", type=int, nargs="+", default=[1, 8, 16, 32, 64])
    ap.add_argument("--seq", type=int, nargs="+", default=[1024])
    ap.add_argument("--max-batch", type=int, default=None)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--scheduler", default="static")
    ap.add_argument("--kp", type=int, default=None, help="activation piece length (default: fill 16 KB)")
    ap.add_argument("--attn-per-sm", type=int, default=2, help="attention split budget: tasks per SM")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
    mb = args.max_batch or max(args.batch)
    t0 = time.perf_counter()
    m = BatchDecodeModel(cfg, samples=tuple(sorted(set(args.seq))), max_batch=mb, scheduler=args.scheduler,
                         kp=args.kp, attn_tasks_per_sm=args.attn_per_sm)
    setup = time.perf_counter() - t0
    stream = torch.cuda.Stream()
    for s in args.seq:
        m.fill_cache(s, seed=1)
        m.set_token([(1 + 7 * i) % cfg.vocab for i in range(mb)])
        for b in args.batch:
            t1 = time.perf_counter()
            m.launch(s, b, stream.cuda_stream)
            torch.cuda.synchronize()
            first = time.perf_counter() - t1
            m.executor.sync()
            for _ in range(args.warmup):
                m.launch(s, b, stream.cuda_stream)
            torch.cuda.synchronize()
            evs = []
            for _ in range(args.steps):
                a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                m.launch(s, b, stream.cuda_stream)
                e.record(stream)
                evs.append((a, e))
            torch.cuda.synchronize()
            st = m.executor.sync()
            ms = statistics.median(x.elapsed_time(y) for x, y in evs)
            nbytes = cfg.step_bytes(s, b)
            ach = nbytes / (ms * 1e-3) / 1e9
            print(json.dumps({"workload": f"{cfg.name} decode bs={b} seq {s}", "scheduler": args.scheduler,
                              "path": "tcgen05 GEMV", "kp": m.kp, "batch": b, "seq": s, "max_batch": mb,
                              "us_per_step": ms * 1e3, "tokens_per_s": b / (ms * 1e-3), "bytes_per_step": nbytes,
                              "achieved_gbs": ach, "frac_of_measured_hbm": ach / peak,
                              "tasks_executed": st["tasks_executed"], "first_step_s": first,
                              "model_setup_s": setup, "lower_ms": m.lower_ms, "upload_ms": m.upload_ms}),
                  flush=True)


if __name__ == "__main__":
    main()

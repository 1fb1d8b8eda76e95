"""Qwen3-30B-A3B-shaped MoE decode (bs=1, S=1024) on the megakernel: µs/token
under the static and dynamic schedulers, routing computed on the GPU, plus the
HBM roofline fraction from the device expert counts (algorithmic bytes = dense
weights + the touched experts' weights + KV).  Prints one JSON line per scheduler.

    python scripts/bench_moe.py [--steps K] [--warmup W] [--seq S] [--batch B ...]

--batch lists the batch sizes to time; all of them run on ONE lowered artifact
(batch symbol b <= max(--batch)), as a serving loop would.
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2604_13327_b200.moe import MOE_CONFIGS, MoEDecodeModel, init_moe_weights  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="qwen3-30b-a3b")
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--schedulers", nargs="+", default=["static", "dynamic", "dynamic-early"])
    ap.add_argument("--batch", type=int, nargs="+", default=[1])
    ap.add_argument("--attn-cap", type=int, default=None, help="attention splits per (sequence, kv head)")
    args = ap.parse_args()
    if len(args.schedulers) > 1:  # one process per scheduler
        import subprocess
        for sched in args.schedulers:
            subprocess.run([sys.executable, __file__, "--config", args.config, "--steps", str(args.steps), "--warmup",
                            str(args.warmup), "--seq", str(args.seq), "--schedulers", sched, "--batch",
                            *map(str, args.batch)] + (["--attn-cap", str(args.attn_cap)] if args.attn_cap else []),
                           check=False)
        return
    cfg = MOE_CONFIGS[args.config]
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
    dev = torch.device("cuda:0")
    t0 = time.perf_counter()
    W = init_moe_weights(cfg, dev, 0)
    init_s = time.perf_counter() - t0
    mb = max(args.batch)
    for sched in args.schedulers:
        t1 = time.perf_counter()
        m = MoEDecodeModel(cfg, samples=(args.seq,), weights=W, scheduler=sched.split("-")[0],
                           early_push=sched.endswith("early"), max_batch=mb,
                           batch_samples=tuple(sorted(set(args.batch) | {1, mb})) if mb > 1 else None,
                           attn_cap=args.attn_cap)
        m.fill_cache(args.seq, seed=1)
        m.set_token([1 + 7 * i for i in range(mb)])
        stream = torch.cuda.Stream()
        lower_s = time.perf_counter() - t1
        for b in args.batch:
            t2 = time.perf_counter()
            m.launch(args.seq, stream.cuda_stream, b)
            torch.cuda.synchronize()
            first = time.perf_counter() - t2
            m.executor.sync()
            for _ in range(args.warmup):
                m.launch(args.seq, stream.cuda_stream, b)
            torch.cuda.synchronize()
            m.executor.sync()
            evs = []
            for _ in range(args.steps):
                a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                m.launch(args.seq, stream.cuda_stream, b)
                e.record(stream)
                evs.append((a, e))
            torch.cuda.synchronize()
            st = m.executor.sync()
            ms = statistics.median(x.elapsed_time(y) for x, y in evs)
            active = m.active_experts()
            nbytes = cfg.step_bytes(args.seq, active, b)
            achieved = nbytes / (ms * 1e-3) / 1e9
            print(json.dumps({"workload": f"{cfg.name} decode bs={b} seq {args.seq}", "scheduler": sched,
                              "batch": b, "max_batch": mb, "us_per_step": ms * 1e3,
                              "tokens_per_s": b / (ms * 1e-3), "bytes_per_step": nbytes,
                              "achieved_gbs": achieved, "frac_of_measured_hbm": achieved / peak,
                              "active_experts_per_layer": active, "tasks_executed": st["tasks_executed"],
                              "noop_tasks": st["noop_tasks"], "pushes": st["pushes"], "pops": st["pops"],
                              "first_step_s": first, "model_setup_s": lower_s, "lower_ms": m.lower_ms,
                              "upload_ms": m.upload_ms, "weight_init_s": init_s}), flush=True)
        del m
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

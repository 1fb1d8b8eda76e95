"""Qwen3-30B-A3B-shaped MoE decode (bs=1, S=1024) on the megakernel: µs/token
under the static and dynamic schedulers, routing computed on the GPU, plus the
HBM roofline fraction from the device expert counts (algorithmic bytes = dense
weights + the touched experts' weights + KV).  Prints one JSON line per scheduler.

    python scripts/bench_moe.py [--steps K] [--warmup W] [--seq S]
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
    args = ap.parse_args()
    if len(args.schedulers) > 1:  # one process per scheduler
        import subprocess
        for sched in args.schedulers:
            subprocess.run([sys.executable, __file__, "--config", args.config, "--steps", str(args.steps), "--warmup",
                            str(args.warmup), "--seq", str(args.seq), "--schedulers", sched], check=False)
        return
    cfg = MOE_CONFIGS[args.config]
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
    dev = torch.device("cuda:0")
    t0 = time.perf_counter()
    W = init_moe_weights(cfg, dev, 0)
    init_s = time.perf_counter() - t0
    for sched in args.schedulers:
        t1 = time.perf_counter()
        m = MoEDecodeModel(cfg, samples=(args.seq,), weights=W, scheduler=sched.split("-")[0],
                           early_push=sched.endswith("early"))
        m.fill_cache(args.seq, seed=1)
        m.set_token(1)
        stream = torch.cuda.Stream()
        m.launch(args.seq, stream.cuda_stream)
        torch.cuda.synchronize()
        first = time.perf_counter() - t1
        m.executor.sync()
        for _ in range(args.warmup):
            m.launch(args.seq, stream.cuda_stream)
        torch.cuda.synchronize()
        m.executor.sync()
        evs = []
        for _ in range(args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            m.launch(args.seq, stream.cuda_stream)
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
        st = m.executor.sync()
        ms = statistics.median(x.elapsed_time(y) for x, y in evs)
        active = m.active_experts()
        nbytes = cfg.step_bytes(args.seq, active)
        achieved = nbytes / (ms * 1e-3) / 1e9
        print(json.dumps({"workload": f"{cfg.name} decode bs=1 seq {args.seq}", "scheduler": sched,
                          "us_per_token": ms * 1e3, "bytes_per_step": nbytes, "achieved_gbs": achieved,
                          "frac_of_measured_hbm": achieved / peak, "active_experts_per_layer": active,
                          "tasks_executed": st["tasks_executed"], "noop_tasks": st["noop_tasks"],
                          "pushes": st["pushes"], "pops": st["pops"], "first_step_s": first,
                          "lower_ms": m.lower_ms, "upload_ms": m.upload_ms, "weight_init_s": init_s}), flush=True)
        del m
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

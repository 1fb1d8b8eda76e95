#!/usr/bin/env python3
"""Decode benchmark: Llama-3-8B-shaped bs=1 decode at seq 1024 on the Event
Tensor megakernel (one persistent launch per step).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  metric = decode µs/token (lower is better).
`value` is device time with every input already in HBM; `e2e` goes through
the public API with the token id copied host->device and the logits copied
device->host inside each timed step.  Weights (15 GB) exceed L2 (126 MB), so
no L2 flush is needed between steps.  With N > 1 every rank runs an
independent replica ("replicas only" for the dense 8B path).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode µs/token (Llama-3-8B bs=1) and HBM roofline fraction; warmup time"
UNIT = "µs/token"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def profiled_traffic(cfg_name):
    """dram bytes per launch from the committed ncu capture, if one exists."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(cfg_name)
    except Exception:
        return None


class ClockSampler:
    def __init__(self, device_index):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        self.idx = device_index

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
            sm = [float(r[0]) for r in rows]
            mx = max(float(r[1]) for r in rows)
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].strip().lower() == "active"})
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows)}
        except Exception:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}


def cpu_reference_steps_us(cfg, seq, steps=5, budget_s=12.0):
    """The reference's own CPU path for this step, timed on this host, `steps` samples.

    Per sample:
    (1) the reference executor (etsim, built from its sources into oracle/_ref)
        running the static schedule of the same Llama-3-8B decode graph (one
        `simulate` call, 1 thread);
    (2) the numerics of the step (the reference has none): the CPU
        fp32 oracle on layer 0, scaled by the layer count, plus lm_head.
    Setup (graph lowering, weight init) happens once; each sample is ~30 ms, so
    100 samples stay within a few seconds.  Returns (list of us_per_token, detail)."""
    import torch

    from paper_2604_13327_b200 import etsim
    from paper_2604_13327_b200.decode import decode_graph_spec

    steps = max(1, steps)
    detail = {}
    sims = None
    # The reference module registers pybind types with the same names as this
    # framework's module, so it runs in its own interpreter.
    code = (
        "import json, sys, time\n"
        f"sys.path.insert(0, {os.path.join(ROOT, 'oracle', '_ref')!r})\n"
        "import etsim\n"
        "g = etsim.Graph.from_json(sys.stdin.read())\n"
        f"k = etsim.lower_static(g, [{{'s': {seq}}}], num_sms=148)\n"
        f"etsim.simulate(k, {{'s': {seq}}})\n"
        "ts = []\n"
        f"for _ in range({steps}):\n"
        "    t0 = time.perf_counter()\n"
        f"    etsim.simulate(k, {{'s': {seq}}})\n"
        "    ts.append((time.perf_counter() - t0) * 1e6)\n"
        "print(json.dumps({'us': ts}))\n"
    )
    try:
        # the same decode graph DecodeModel lowers (148 workers)
        g = etsim.Graph.from_json(json.dumps(decode_graph_spec(cfg, 148, seq)[0]))
        detail["graph_tasks"] = g.instantiate({"s": seq}).num_tasks
        out = subprocess.run([sys.executable, "-c", code], input=g.to_json(),
                             capture_output=True, text=True, timeout=budget_s * 5 + 60)
        sims = json.loads(out.stdout.strip().splitlines()[-1])["us"]
        detail["reference_simulate_us"] = statistics.median(sims)
        detail["reference_runs"] = len(sims)
    except Exception as exc:  # reference build absent on this host
        detail["reference_error"] = (str(exc) + " " + (out.stderr[-200:] if "out" in dir() else ""))[:300]
    # numerics: one layer + lm_head in fp32 on CPU
    torch.manual_seed(0)
    H, I, V = cfg.hidden, cfg.intermediate, cfg.vocab
    q_rows, kv_rows = cfg.q_rows, cfg.kv_rows
    w = lambda *s: (torch.randn(*s) * 0.02)  # noqa: E731
    wqkv, wo, wg, wu, wd = w(q_rows + 2 * kv_rows, H), w(H, q_rows), w(I, H), w(I, H), w(H, I)
    lm = w(V, H)
    K = torch.randn(cfg.kv_heads, seq, cfg.head_dim)
    Vc = torch.randn(cfg.kv_heads, seq, cfg.head_dim)
    x = torch.randn(H)
    G = cfg.heads // cfg.kv_heads

    def layer():
        qkv = wqkv @ x
        q = qkv[:q_rows].view(cfg.heads, cfg.head_dim).view(cfg.kv_heads, G, cfg.head_dim)
        sc = torch.einsum("kgd,ksd->kgs", q, K) / cfg.head_dim ** 0.5
        a = torch.einsum("kgs,ksd->kgd", torch.softmax(sc, -1), Vc).reshape(-1)
        h = x + wo @ a
        return h + wd @ (torch.nn.functional.silu(wg @ h) * (wu @ h))

    layer()
    lm @ x
    vals, lay, lms = [], [], []
    for i in range(steps):
        t0 = time.perf_counter()
        layer()
        t1 = time.perf_counter()
        lm @ x
        t2 = time.perf_counter()
        lay.append((t1 - t0) * 1e6)
        lms.append((t2 - t1) * 1e6)
        vals.append(lay[-1] * cfg.layers + lms[-1] + (sims[i] if sims else 0.0))
    detail.update({"numerics_layer_us": statistics.median(lay), "numerics_lm_head_us": statistics.median(lms),
                   "numerics_us": statistics.median(lay) * cfg.layers + statistics.median(lms)})
    return vals, detail


def run_reference(args):
    """--impl reference: the reference's CPU implementation of the path."""
    import torch

    from paper_2604_13327_b200.decode import CONFIGS

    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    threads = torch.get_num_threads()
    # W warm-up samples, then K timed samples (each one simulate + one layer + lm_head)
    vals, detail = cpu_reference_steps_us(cfg, args.seq, steps=args.warmup + max(1, args.steps),
                                          budget_s=args.ref_budget)
    vals = vals[args.warmup:]
    value = statistics.median(vals)
    kind = "reference" if "reference_simulate_us" in detail else "port"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": value / 1e3, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (random-init weights, N(0,1) KV)",
        "config": {"workload": f"{cfg.name} decode bs=1 seq {args.seq}", "seq_len": args.seq, "batch": 1},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": "reference etsim.simulate of the static schedule of this framework's Llama-3-8B "
                                   "decode graph (1 thread) + fp32 torch-CPU numerics of layer 0 scaled x32 + lm_head",
                         "detail": detail},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch

    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    torch.cuda.set_device(local)
    from paper_2604_13327_b200.decode import CONFIGS, DecodeModel

    t_start = time.perf_counter()
    cfg = CONFIGS[args.config]
    tp_mode = args.tp > 0 or cfg.name == "llama3-70b"
    tp = args.tp or world
    if tp_mode:
        # tensor parallel over all ranks: in-megakernel NVLink allreduce tasks;
        # NCCL (torch.distributed) only exchanges the peer buffers' IPC handles
        from paper_2604_13327_b200.tp import TPDecodeModel, exchange_peers

        assert tp == world, "tensor parallelism spans every rank of the launch"
        model = TPDecodeModel(cfg, rank, world, device=f"cuda:{local}", samples=tuple(args.samples), seed=0)
        peers = exchange_peers(model.local_buffers(), rank, world) if world > 1 else [model.local_buffers()]
        model.connect(peers)
        model.vocab_local = model.local.vocab
    else:
        model = DecodeModel(cfg, device=f"cuda:{local}", samples=tuple(args.samples), seed=0)
        model.vocab_local = cfg.vocab
    model.fill_cache(args.seq, seed=1)
    model.set_token(1)
    # a dedicated (non-default) stream: the executor launches on exactly this
    # stream, so the CUDA events below time the megakernel itself
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream
    # first completed step = end of warmup-to-first-token
    model.launch(args.seq, sh)
    torch.cuda.synchronize()
    first_token_s = time.perf_counter() - t_start
    model.executor.sync()

    for _ in range(args.warmup):
        model.launch(args.seq, sh)
    torch.cuda.synchronize()
    model.executor.sync()

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timing -------------------------------------------------
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    per_step = []
    barrier()
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            e_a = torch.cuda.Event(enable_timing=True)
            e_b = torch.cuda.Event(enable_timing=True)
            e_a.record(stream)
            model.launch(args.seq, sh)
            e_b.record(stream)
            per_step.append((e_a, e_b))
        ev1.record(stream)
        barrier()
    model.executor.sync()  # raises if the device reported an error
    total_ms = ev0.elapsed_time(ev1)
    step_ms = [a.elapsed_time(b) for a, b in per_step]
    if world > 1:
        t = torch.tensor([total_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = t.item()
    ms_per_step = total_ms / args.steps

    # ---- end-to-end through the public API (host buffers) ------------------------
    tok_host = torch.ones(1, dtype=torch.int32).pin_memory()
    logits_host = torch.empty(1, model.vocab_local, dtype=torch.float32).pin_memory()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        model.tokens.copy_(tok_host, non_blocking=True)
        model.launch(args.seq, sh)
        logits_host.copy_(model.logits, non_blocking=True)
    e1.record(stream)
    barrier()
    model.executor.sync()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = t.item()

    peak, peak_src = measured_peak()
    step_bytes = cfg.step_bytes(args.seq)
    if tp_mode:  # per-GPU algorithmic bytes: the rank's weight shard plus its kv heads' cache
        step_bytes = model.local.step_bytes(args.seq)
    med_ms = statistics.median(step_ms)
    achieved = step_bytes / (med_ms * 1e-3) / 1e9
    tokens_total = args.steps * (1 if tp_mode else world)  # TP: all ranks serve one token per step
    value = total_ms * 1e3 / tokens_total
    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            import torch as _t

            vals, detail = cpu_reference_steps_us(cfg, args.seq, steps=8, budget_s=args.ref_budget)
            v = statistics.median(vals)
            cpu = {"value": v, "unit": UNIT, "cores": _t.get_num_threads(),
                   "kind": "reference" if "reference_simulate_us" in detail else "port",
                   "sample": "reference etsim.simulate of the static Llama-3-8B decode schedule (1 thread) + fp32 "
                             "torch-CPU numerics of layer 0 scaled x32 + lm_head",
                   "detail": detail}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": False,
            "scaling": "strong" if tp_mode else "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init bf16 weights N(0,0.02), KV cache N(0,1) for positions [0,s))",
            "config": {"workload": f"{cfg.name} decode bs=1 seq {args.seq}", "seq_len": args.seq, "batch": 1,
                       "samples": list(args.samples),
                       "parallelism": f"tp{world}" if tp_mode else f"replicas{world}",
                       "l2": "inputs larger than L2 (15 GB of weights per step), no flush",
                       "step_us_median": med_ms * 1e3, "step_us_p10": sorted(step_ms)[len(step_ms) // 10] * 1e3,
                       "step_us_p90": sorted(step_ms)[(len(step_ms) * 9) // 10] * 1e3,
                       "tasks_per_step": int(model.kernel.to_json().count('"id"')) if args.count_tasks else None,
                       "warmup_s": {"first_token": first_token_s, "lower_ms": model.lower_ms,
                                    "upload_ms": model.upload_ms}},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": profiled_traffic(cfg.name),
                         "bytes_per_step": step_bytes, "peak_source": peak_src,
                         "frac_of_8TBps": achieved / 8000.0},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_ms * 1e3 / tokens_total, "unit": UNIT, "h2d_bytes_per_step": 4,
                    "d2h_bytes_per_step": 4 * model.vocab_local},
            "gpu_launches": args.steps,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="llama3-8b")
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--samples", type=int, nargs="+", default=[1024])
    ap.add_argument("--ref-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--count-tasks", action="store_true")
    ap.add_argument("--tp", type=int, default=0, help="tensor-parallel degree (default: world for llama3-70b, else 1)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

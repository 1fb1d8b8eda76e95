"""Generates tests/golden/reference_golden.json from the UNMODIFIED reference
(arxiv/paper_2604_13327 proj/, built from its own sources into oracle/_ref by
oracle/Makefile).  Run in the development container, where /root/reference
exists:

    make -C oracle && python tests/golden/make_golden.py

The fixtures pin (1) the oracle restatement (oracle/etsim_oracle.py) and (2)
this framework's host library and GPU executor accounting to the reference's
own outputs: graph JSON, instantiation structure and counts, seeded durations,
compiled static kernels (queues, initial counts), no-op masking, dynamic-queue
accounting, routing realizations and the critical-path / list-schedule values.
"""

import hashlib
import importlib.util
import json
import os
import sys
import types

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
import etsim  # noqa: E402  (the reference module)

spec = importlib.util.spec_from_file_location("graphs", os.path.join(ROOT, "paper_2604_13327_b200", "graphs.py"))
graphs = importlib.util.module_from_spec(spec)
spec.loader.exec_module(graphs)


def sha(s):
    return hashlib.sha256(s.encode()).hexdigest()


def mat(m, full=True):
    d = {"num_tasks": m.num_tasks, "num_events": m.num_events, "call_task_counts": m.call_task_counts,
         "initial_counts": m.initial_counts}
    return d


def trace_acc(t):
    return {"final_counters": t.final_counters, "noop_records": t.noop_records, "num_records": t.num_records,
            "makespan": t.makespan}


cases = {}

# --- split-K row sum (paper 2.2)
g = etsim.splitk_rowsum()
k = etsim.lower_static(g, [{"n": 2}, {"n": 4}, {"n": 8}], num_sms=3)
cases["splitk"] = {
    "graph": g.to_json(),
    "instantiate": {str(n): mat(g.instantiate({"n": n})) for n in (1, 2, 3, 5)},
    "samples": [{"n": 2}, {"n": 4}, {"n": 8}], "num_sms": 3,
    "kernel": k.to_json(),
    "simulate": {str(n): trace_acc(etsim.simulate(k, {"n": n})) for n in (1, 3, 4, 5, 8)},
}

# --- gemm + reduce-scatter with shape sampling (acceptance criterion 8)
g = etsim.gemm_reduce_scatter("b * 2", 2)
samples = [{"b": 1}, {"b": 2}, {"b": 4}, {"b": 8}]
k = etsim.lower_static(g, samples, num_sms=2)
cases["gemm_rs"] = {
    "graph": g.to_json(), "samples": samples, "num_sms": 2, "kernel": k.to_json(),
    "instantiate": {str(b): mat(g.instantiate({"b": b})) for b in range(1, 9)},
    "simulate": {str(b): trace_acc(etsim.simulate(k, {"b": b}, seed=b)) for b in range(1, 9)},
}

# --- all-gather ring with a DMA queue
g = etsim.all_gather_gemm(4, 3)
k = etsim.lower_static(g, [{}], num_sms=3)
cases["all_gather"] = {"graph": g.to_json(), "samples": [{}], "num_sms": 3, "kernel": k.to_json(),
                       "instantiate": {"": mat(g.instantiate({}))}, "simulate": {"": trace_acc(etsim.simulate(k, {}))}}

# --- MoE layer, data-dependent (worst-case rewrite + dynamic)
routing = etsim.moe_realization(tokens=16, experts=4, top_k=2, tile_size=2, hot_fraction=0.6, hot_expert=1, seed=3)
g = etsim.moe_layer(tokens=16, experts=4, top_k=2, tile_size=2)
wg = etsim.worst_case_rewrite(g)
k = etsim.lower_static(wg, [{"tokens": 16}], num_sms=4)
dk = etsim.lower_dynamic(g)
td = etsim.simulate(dk, {"tokens": 16}, routing=routing, seed=3)
md = etsim.metrics(td)
cases["moe"] = {
    "graph": g.to_json(), "rewritten": wg.to_json(), "routing": routing, "samples": [{"tokens": 16}], "num_sms": 4,
    "kernel": k.to_json(),
    "instantiate": {"16": mat(g.instantiate({"tokens": 16}, routing=routing, seed=3))},
    "simulate": {"16": trace_acc(etsim.simulate(k, {"tokens": 16}, routing=routing, seed=3))},
    "dynamic": {"pushes": md["pushes"], "pops": md["pops"], "real_tasks": md["real_tasks"],
                "final_counters": td.final_counters},
    "dynamic_kernel": dk.to_json(),
    "early_kernel": etsim.lower_dynamic(g, early_push=True).to_json(),
}

# --- random DAGs (graph JSON, seeded durations, oracles)
cases["random_dag"] = {}
for seed in range(12):
    nodes, edges = 5 + seed % 16, 8 + seed % 20
    g = etsim.random_dag(nodes, edges, seed)
    m = g.instantiate({}, seed=seed)
    sms = 1 + seed % 4
    k = etsim.lower_static(g, [{}], num_sms=sms)
    cases["random_dag"][str(seed)] = {"nodes": nodes, "edges": edges, "graph": g.to_json(), "num_sms": sms,
                                      "kernel": k.to_json(), "instantiate": mat(m),
                                      "critical_path": m.critical_path(), "list_schedule": m.list_schedule(sms)}

# --- seeded uniform durations and the list-schedule oracle (acceptance criterion 6)
spec_j = json.loads(etsim.gemm_reduce_scatter("16", 2).to_json())
spec_j["duration_models"]["mm"] = {"kind": "uniform", "lo": 5, "hi": 9}
spec_j["duration_models"]["rs"] = {"kind": "uniform", "lo": 5, "hi": 9}
g = etsim.Graph.from_json(json.dumps(spec_j))
cases["uniform"] = {"graph": g.to_json(), "seeds": {}}
for seed in range(4):
    m = g.instantiate({}, seed=seed)
    t = etsim.simulate(etsim.lower_static(g, [{}], num_sms=4), {}, seed=seed)
    cases["uniform"]["seeds"][str(seed)] = {"critical_path": m.critical_path(), "list_schedule": m.list_schedule(4),
                                            "static_makespan": t.makespan,
                                            "barrier_makespan": etsim.simulate_barrier(g, {}, num_sms=4, seed=seed).makespan}

# --- routing realizations (golden vectors)
cases["realizations"] = []
for kw in [dict(tokens=1, experts=128, top_k=8, seed=0), dict(tokens=4, experts=8, top_k=2, tile_size=2, seed=7),
           dict(tokens=8, experts=128, top_k=8, seed=1), dict(tokens=32, experts=128, top_k=8, seed=2),
           dict(tokens=64, experts=8, top_k=2, tile_size=4, hot_fraction=0.5, hot_expert=1, seed=11),
           dict(tokens=128, experts=8, top_k=1, tile_size=4, hot_fraction=0.7, hot_expert=0, seed=5)]:
    cases["realizations"].append({"args": kw, "out": etsim.moe_realization(**kw)})

# --- decode graphs (this framework's workloads, lowered by the reference)
for name, cfg_kw, tasks, samples in [
        ("tiny", dict(attn_chunk=64, kv_heads=2, layers=2), 16, [16, 64]),
        ("llama8b", dict(attn_chunk=64, kv_heads=8, layers=32), 148, [1024])]:
    cfg = types.SimpleNamespace(**cfg_kw)
    spec_d = graphs.graph_spec(cfg, tasks, tasks)
    g = etsim.Graph.from_json(json.dumps(spec_d))
    k = etsim.lower_static(g, [{"s": s} for s in samples], num_sms=tasks)
    kj = k.to_json()
    entry = {"spec": spec_d, "num_sms": tasks, "samples": [{"s": s} for s in samples], "kernel_sha256": sha(kj),
             "instantiate": {str(s): mat(g.instantiate({"s": s})) for s in samples}}
    if name == "tiny":
        entry["kernel"] = kj
        entry["simulate"] = {str(s): trace_acc(etsim.simulate(k, {"s": s})) for s in (0, 10, 16, 40, 64)}
    else:
        entry["simulate"] = {str(s): trace_acc(etsim.simulate(k, {"s": s})) for s in (1000, 1024)}
    cases[name] = entry

# --- the graphs bench.py actually lowers (tests/golden/bench_graphs.json.gz, pinned to the
# live layout functions by tests/test_bench_graphs.py): the headline Llama-3-8B step
# (balanced / grouped / fused-merge spec) and the Qwen3-30B-A3B bs=1 step on both schedulers
import gzip  # noqa: E402

with gzip.open(os.path.join(HERE, "bench_graphs.json.gz"), "rt") as f:
    BENCH = json.load(f)
fx = BENCH["llama3-8b|b1|static|s1024|tp0"]
g = etsim.Graph.from_json(json.dumps(fx["spec"]))
k = etsim.lower_static(g, fx["bindings"], num_sms=fx["num_sms"])
cases["llama8b_bench"] = {"spec": fx["spec"], "num_sms": fx["num_sms"], "samples": fx["bindings"],
                          "kernel_sha256": sha(k.to_json()),
                          "instantiate": {str(s): mat(g.instantiate({"s": s})) for s in (1000, 1024)},
                          "simulate": {str(s): trace_acc(etsim.simulate(k, {"s": s})) for s in (1000, 1024)}}
for sched in ("static", "dynamic"):
    fx = BENCH[f"qwen3-30b-a3b|b1|{sched}|s1024|tp0"]
    g = etsim.Graph.from_json(json.dumps(fx["spec"]))
    routing = {}
    for l in range(fx["moe"]["layers"]):
        r = etsim.moe_realization(tokens=1, experts=128, top_k=8, tile_size=8, seed=l)
        routing.update({f"topk{l}": r["topk"], f"cnt{l}": r["expert_counts"], f"ind{l}": r["exp_indptr"],
                        f"tind{l}": [12 * v for v in r["exp_indptr"]]})
    if sched == "static":
        k = etsim.lower_static(etsim.worst_case_rewrite(g), fx["bindings"], num_sms=fx["num_sms"])
        t = etsim.simulate(k, fx["binding"], routing=routing)
        extra = {}
    else:
        k = etsim.lower_dynamic(g)
        t = etsim.simulate(k, fx["binding"], routing=routing, num_sms=fx["num_sms"])
        md = etsim.metrics(t)
        extra = {"pushes": md["pushes"], "pops": md["pops"], "real_tasks": md["real_tasks"]}
    m = g.instantiate(fx["binding"], routing=routing)
    cases[f"qwen3_bench_{sched}"] = dict({"spec": fx["spec"], "bindings": fx["bindings"], "routing": routing,
                                          "kernel_sha256": sha(k.to_json()), "instantiate": mat(m),
                                          "simulate": trace_acc(t)}, **extra)

out = os.path.join(HERE, "reference_golden.json")
with open(out, "w") as f:
    json.dump(cases, f, sort_keys=True)
print("wrote", out, os.path.getsize(out), "bytes")

"""This framework's host library (the C++ lowering behind the drop-in API) vs
the reference's outputs: bit-exact artifacts, structures and counts
(tests/golden/reference_golden.json), plus the reference's own Python smoke
tests (ref proj/tests/python/test_smoke.py) for the parts that need no GPU."""

import json
import os

import pytest

from oracle import etsim_oracle as O
from paper_2604_13327_b200 import etsim

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def _mk(case):
    if case == "splitk":
        return etsim.splitk_rowsum()
    if case == "gemm_rs":
        return etsim.gemm_reduce_scatter("b * 2", 2)
    if case == "all_gather":
        return etsim.all_gather_gemm(4, 3)
    raise KeyError(case)


@pytest.mark.parametrize("case", ["splitk", "gemm_rs", "all_gather"])
def test_generators_and_kernels_bit_exact(case):
    c = GOLD[case]
    g = _mk(case)
    assert g.to_json() == c["graph"]
    k = etsim.lower_static(g, c["samples"], num_sms=c["num_sms"])
    assert k.to_json() == c["kernel"]  # queues, waits, notifies, initial counts, layout
    for key, want in c["instantiate"].items():
        b = {} if key == "" else {g.symbols[0]: int(key)}
        m = g.instantiate(b)
        assert (m.num_tasks, m.num_events) == (want["num_tasks"], want["num_events"])
        assert m.call_task_counts == want["call_task_counts"]
        assert m.initial_counts == want["initial_counts"]


def test_moe_paths_bit_exact():
    c = GOLD["moe"]
    g = etsim.moe_layer(tokens=16, experts=4, top_k=2, tile_size=2)
    assert g.to_json() == c["graph"]
    routing = etsim.moe_realization(tokens=16, experts=4, top_k=2, tile_size=2, hot_fraction=0.6, hot_expert=1,
                                    seed=3)
    assert routing == c["routing"]
    wg = etsim.worst_case_rewrite(g)
    assert wg.to_json() == c["rewritten"]
    assert etsim.lower_static(wg, [{"tokens": 16}], num_sms=4).to_json() == c["kernel"]
    m = g.instantiate({"tokens": 16}, routing=routing, seed=3)
    assert m.call_task_counts == c["instantiate"]["16"]["call_task_counts"]
    assert m.initial_counts == c["instantiate"]["16"]["initial_counts"]
    assert etsim.lower_dynamic(g).to_json() == c["dynamic_kernel"]
    assert etsim.lower_dynamic(g, early_push=True).to_json() == c["early_kernel"]
    assert etsim.enable_early_push(etsim.lower_dynamic(g)).to_json() == c["early_kernel"]


def test_random_dags_bit_exact():
    for seed, c in GOLD["random_dag"].items():
        g = etsim.random_dag(c["nodes"], c["edges"], int(seed))
        assert g.to_json() == c["graph"]
        assert etsim.lower_static(g, [{}], num_sms=c["num_sms"]).to_json() == c["kernel"]
        m = g.instantiate({}, seed=int(seed))
        assert m.critical_path() == c["critical_path"]
        assert m.list_schedule(c["num_sms"]) == c["list_schedule"]


def test_seeded_durations_and_oracles():
    c = GOLD["uniform"]
    g = etsim.Graph.from_json(c["graph"])
    assert g.to_json() == c["graph"]
    for seed, want in c["seeds"].items():
        m = g.instantiate({}, seed=int(seed))
        assert m.critical_path() == want["critical_path"]
        assert m.list_schedule(4) == want["list_schedule"]
        o = O.instantiate(json.loads(c["graph"]), {}, seed=int(seed))
        assert m.durations == [t["duration"] for t in o["tasks"]]


def test_realizations_bit_exact():
    for case in GOLD["realizations"]:
        assert etsim.moe_realization(**case["args"]) == case["out"]


@pytest.mark.parametrize("name", ["tiny", "llama8b", "llama8b_bench"])
def test_decode_graph_lowering_bit_exact(name):
    import hashlib

    c = GOLD[name]
    g = etsim.Graph.from_json(json.dumps(c["spec"]))
    k = etsim.lower_static(g, c["samples"], num_sms=c["num_sms"])
    kj = k.to_json()
    assert hashlib.sha256(kj.encode()).hexdigest() == c["kernel_sha256"]
    for s, want in c["instantiate"].items():
        m = g.instantiate({"s": int(s)})
        assert m.num_tasks == want["num_tasks"] and m.initial_counts == want["initial_counts"]


def test_select_queues_masks_match_oracle():
    c = GOLD["gemm_rs"]
    g = etsim.gemm_reduce_scatter("b * 2", 2)
    k = etsim.lower_static(g, c["samples"], num_sms=2)
    samples = O.lower_static(json.loads(c["graph"]), c["samples"], 2)
    for b in range(1, 9):
        sel = etsim.select_queues(k, {"b": b})
        pick, masked, real = O.select_queues(json.loads(c["graph"]), samples, {"b": b})
        assert (sel["sample_index"], sel["masked"], sel["real_tasks"]) == (pick, masked, real)
        assert len(masked) - real == c["simulate"][str(b)]["noop_records"]
    with pytest.raises(etsim.GraphError):
        etsim.select_queues(k, {"b": 9})


def test_random_graphs_vs_oracle():
    """Differential: random layered DAGs with symbolic grids and maps."""
    import random

    rnd = random.Random(0)
    for it in range(25):
        ncalls = rnd.randint(2, 6)
        spec = {"symbols": ["b"], "size_symbol": "b", "duration_models": {"u": {"kind": "uniform", "lo": 1, "hi": 9}},
                "device_functions": [], "event_tensors": [], "calls": []}
        for ci in range(ncalls):
            grid = [rnd.choice(["b", "b * 2", "(b + 1) // 2", "3"]), rnd.choice(["1", "2", "b"])]
            spec["device_functions"].append({"name": f"f{ci}", "grid": grid, "resource": "sm", "duration": "u"})
            spec["event_tensors"].append({"name": f"e{ci}", "shape": ["1"]})
            c = {"fn": f"f{ci}", "out": [{"event": f"e{ci}", "map": ["0"]}]}
            deps = [d for d in range(ci) if rnd.random() < 0.6]
            if deps:
                c["in"] = [{"event": f"e{d}", "map": ["0"]} for d in deps]
            spec["calls"].append(c)
        text = json.dumps(spec)
        g = etsim.Graph.from_json(text)
        assert g.validate() == []
        for b in (1, 2, 3):
            m = g.instantiate({"b": b}, seed=it)
            o = O.instantiate(spec, {"b": b}, seed=it)
            assert m.num_tasks == len(o["tasks"])
            assert m.initial_counts == o["initial_counts"]
            assert m.task_waits == o["waits"] and m.task_notifies == o["notifies"]
            assert m.event_consumers == o["consumers"] and m.event_producers == o["producers"]
            assert m.durations == [t["duration"] for t in o["tasks"]]
        k = etsim.lower_static(g, [{"b": 1}, {"b": 4}], num_sms=3)
        ok = O.lower_static(spec, [{"b": 1}, {"b": 4}], 3)
        for i in range(2):
            q = k.sample_queues(i)
            assert [[t["id"] for t in qq] for qq in q["sm_queues"]] == ok[i]["sm_queues"]


# ---- the reference's own python smoke tests (ref tests/python/test_smoke.py), CPU parts ----

def test_ref_smoke_splitk_structure():
    g = etsim.splitk_rowsum()
    assert g.validate() == []
    m = g.instantiate({"n": 2})
    assert m.num_tasks == 10 and m.call_task_counts == [8, 2] and m.initial_counts == [4, 4]


def test_ref_smoke_kernel_round_trip():
    g = etsim.gemm_reduce_scatter("b * 2", 2)
    k = etsim.lower_static(g, [{"b": 1}, {"b": 2}, {"b": 4}], num_sms=2)
    assert k.sample_bindings == [{"b": 1}, {"b": 2}, {"b": 4}]
    k2 = etsim.load_kernel(k.to_json())
    assert isinstance(k2, etsim.StaticKernel) and k2.to_json() == k.to_json()
    dk = etsim.lower_dynamic(g)
    assert isinstance(etsim.load_kernel(dk.to_json()), etsim.DynamicKernel)


def test_ref_smoke_moe_summary():
    routing = etsim.moe_realization(tokens=16, experts=4, top_k=2, tile_size=2, hot_fraction=0.6, hot_expert=1, seed=3)
    assert sum(routing["expert_counts"]) == 32
    indptr = routing["exp_indptr"]
    assert indptr[0] == 0 and indptr[-1] == sum((c + 1) // 2 for c in routing["expert_counts"])
    g = etsim.moe_layer(tokens=16, experts=4, top_k=2, tile_size=2)
    assert g.summary()["has_data_dependent"]
    sk = etsim.lower_static(etsim.worst_case_rewrite(g), [{"tokens": 16}], num_sms=4)
    assert sk.graph.summary()["has_data_dependent"] is False


def test_ref_smoke_graph_json_round_trip():
    g = etsim.random_dag(10, 14, seed=5)
    text = g.to_json()
    assert etsim.Graph.from_json(text).to_json() == text


def test_ref_smoke_errors_are_typed():
    with pytest.raises(etsim.GraphError):
        etsim.Graph.from_json("not a graph")
    with pytest.raises(etsim.GraphError):
        etsim.lower_static(etsim.moe_layer(tokens=4), [{"tokens": 4}])


def test_no_cpu_fallback_without_gpu():
    if etsim.gpu_available():
        pytest.skip("GPU present")
    k = etsim.lower_static(etsim.gemm_reduce_scatter("4", 2), [{}], num_sms=2)
    with pytest.raises(etsim.GraphError):
        etsim.simulate(k)


@pytest.mark.parametrize("sched", ["static", "dynamic"])
def test_qwen3_bench_graph_lowering_bit_exact(sched):
    """The Qwen3-30B-A3B bs=1 graph bench.py lowers: this framework's lowering and
    routed instantiation equal the reference's (tests/golden/make_golden.py)."""
    import hashlib

    c = GOLD[f"qwen3_bench_{sched}"]
    g = etsim.Graph.from_json(json.dumps(c["spec"]))
    if sched == "static":
        k = etsim.lower_static(etsim.worst_case_rewrite(g), c["bindings"], num_sms=148)
    else:
        k = etsim.lower_dynamic(g)
    assert hashlib.sha256(k.to_json().encode()).hexdigest() == c["kernel_sha256"]
    m = g.instantiate(c["bindings"][0], routing=c["routing"])
    want = c["instantiate"]
    assert (m.num_tasks, m.num_events) == (want["num_tasks"], want["num_events"])
    assert m.call_task_counts == want["call_task_counts"] and m.initial_counts == want["initial_counts"]

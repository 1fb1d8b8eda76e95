"""Pins the CPU oracle (oracle/etsim_oracle.py) to the reference's own outputs
(tests/golden/reference_golden.json, produced by tests/golden/make_golden.py
from the unmodified reference built in oracle/_ref)."""

import json
import os

import pytest

from oracle import etsim_oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def _ref_queue_ids(kernel_json, sample=0):
    k = json.loads(kernel_json)
    s = k["samples"][sample]
    return [[t["id"] for t in q] for q in s["sm_queues"]], [t["id"] for t in s["dma_queue"]], s["initial_counts"]


@pytest.mark.parametrize("case", ["splitk", "gemm_rs", "all_gather"])
def test_oracle_instantiate_and_queues(case):
    c = GOLD[case]
    g = json.loads(c["graph"])
    for key, want in c["instantiate"].items():
        b = {} if key == "" else {g["symbols"][0]: int(key)}
        m = O.instantiate(g, b)
        assert len(m["tasks"]) == want["num_tasks"]
        assert m["call_task_counts"] == want["call_task_counts"]
        assert m["initial_counts"] == want["initial_counts"]
    samples = O.lower_static(g, c["samples"], c["num_sms"])
    ref = json.loads(c["kernel"])
    for i, s in enumerate(samples):
        sm, dma, init = _ref_queue_ids(c["kernel"], i)
        assert s["sm_queues"] == sm and s["dma_queue"] == dma and s["initial_counts"] == init
        assert s["binding"] == ref["samples"][i]["binding"]


@pytest.mark.parametrize("case", ["splitk", "gemm_rs", "all_gather"])
def test_oracle_static_accounting(case):
    c = GOLD[case]
    g = json.loads(c["graph"])
    samples = O.lower_static(g, c["samples"], c["num_sms"])
    for key, want in c["simulate"].items():
        b = {} if key == "" else {g["symbols"][0]: int(key)}
        acc = O.static_accounting(g, samples, b)
        assert acc["noops"] == want["noop_records"]
        assert acc["executed"] + acc["noops"] == want["num_records"]
        assert acc["final_counters"] == want["final_counters"]


def test_oracle_moe_worst_case_and_masking():
    c = GOLD["moe"]
    g = json.loads(c["graph"])
    r = c["routing"]
    m = O.instantiate(g, {"tokens": 16}, r, seed=3)
    assert m["call_task_counts"] == c["instantiate"]["16"]["call_task_counts"]
    assert m["initial_counts"] == c["instantiate"]["16"]["initial_counts"]
    wg = O.worst_case_rewrite(g)
    assert wg == json.loads(c["rewritten"])
    samples = O.lower_static(wg, [{"tokens": 16}], 4)
    sm, dma, init = _ref_queue_ids(c["kernel"])
    assert samples[0]["sm_queues"] == sm and samples[0]["initial_counts"] == init
    acc = O.static_accounting(wg, samples, {"tokens": 16}, r)
    assert acc["noops"] == c["simulate"]["16"]["noop_records"]
    assert acc["final_counters"] == c["simulate"]["16"]["final_counters"]
    # dynamic scheduler accounting: every instantiated task pushed and popped once
    assert c["dynamic"]["pushes"] == c["dynamic"]["pops"] == len(m["tasks"]) == c["dynamic"]["real_tasks"]
    dk = json.loads(c["dynamic_kernel"])
    assert [t["wait_edges"] for t in dk["templates"]] == O.lower_dynamic_arming(g)
    ek = json.loads(c["early_kernel"])
    assert [t["wait_edges"] for t in ek["templates"]] == O.lower_dynamic_arming(g, early_push=True)


def test_oracle_random_dags():
    for seed, c in GOLD["random_dag"].items():
        g = json.loads(c["graph"])
        arcs, durs = O.random_dag_edges(c["nodes"], c["edges"], int(seed))
        assert [g["duration_models"][f"d{v}"]["value"] for v in range(c["nodes"])] == durs
        ins = sorted((int(e["event"][1:]), v) for v, call in enumerate(g["calls"]) for e in call.get("in", []))
        assert ins == sorted(arcs)
        m = O.instantiate(g, {}, seed=int(seed))
        assert m["initial_counts"] == c["instantiate"]["initial_counts"]
        sm, _, _ = _ref_queue_ids(c["kernel"])
        assert O.lower_static(g, [{}], c["num_sms"])[0]["sm_queues"] == sm


def test_oracle_seeded_uniform_durations():
    c = GOLD["uniform"]
    g = json.loads(c["graph"])
    for seed, want in c["seeds"].items():
        m = O.instantiate(g, {}, seed=int(seed))
        # critical path of the two-stage pipeline from the restated durations
        mm = [t["duration"] for t in m["tasks"] if t["call"] == 0]
        rs = [t["duration"] for t in m["tasks"] if t["call"] == 1]
        cp = max(max(mm[2 * r], mm[2 * r + 1]) + rs[r] for r in range(len(rs)))
        assert cp == want["critical_path"]


def test_oracle_routing_realizations():
    for case in GOLD["realizations"]:
        assert O.moe_realization(**case["args"]) == case["out"]
    # SURVEY 8c golden vector
    assert O.moe_realization(tokens=1, experts=128, top_k=8, seed=0)["topk"] == [48, 27, 76, 93, 3, 125, 57, 63]


def test_oracle_expressions():
    e = O.parse("(s + 63) // 64")
    assert O.evaluate(e, {"s": 1000}) == 16 and O.evaluate(e, {"s": 0}) == 0
    assert O.evaluate(O.parse("min(b * 2, 7) % 4 + max(1, t0)"), {"b": 3, "t0": 0}) == 2 + 1
    with pytest.raises(O.ExprError):
        O.evaluate(O.parse("4 // (b % 1)"), {"b": 2})
    with pytest.raises(O.ExprError):
        O.parse("3 +")


def test_oracle_decode_graphs():
    for name in ("tiny", "llama8b"):
        c = GOLD[name]
        for s, want in c["instantiate"].items():
            m = O.instantiate(c["spec"], {"s": int(s)})
            assert len(m["tasks"]) == want["num_tasks"]
            assert m["initial_counts"] == want["initial_counts"]
    c = GOLD["tiny"]
    samples = O.lower_static(c["spec"], c["samples"], c["num_sms"])
    for s, want in c["simulate"].items():
        acc = O.static_accounting(c["spec"], samples, {"s": int(s)})
        assert acc["noops"] == want["noop_records"]


def test_moe_oracle_routing_algebra_matches_reference_realizations():
    """oracle/moe_oracle.moe_routing_tensors (what the device route task computes)
    reproduces the reference's counts and tile indptr (ref workloads.cpp:137-144)
    on every golden realization generated from the reference."""
    import json
    import os

    from oracle.moe_oracle import moe_routing_tensors

    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))
    for case in gold["realizations"]:
        a, out = case["args"], case["out"]
        got = moe_routing_tensors(out["topk"], a["experts"], a.get("tile_size", 1), 3)
        assert got["cnt"] == out["expert_counts"], a
        assert got["ind"] == out["exp_indptr"], a
        assert got["tind"] == [3 * v for v in out["exp_indptr"]]
        # elist groups the slots by expert in slot order
        assert [out["topk"][sl] for sl in got["elist"]] == sorted(out["topk"])

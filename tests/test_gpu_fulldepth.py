"""Parity at the configurations bench.py measures, at full depth.

* Llama-3-8B (32 layers, the exact balanced / grouped / fused-merge graph the
  headline bench lowers): logits and every layer's appended K/V row against the
  CPU oracle fed layer by layer (oracle/parity.py), task counts equal to the
  reference's instantiate() of the same graph (golden `llama8b_bench`), every
  Event Tensor counter back to zero.
* Qwen3-30B-A3B (48 layers, 128 experts, top-8, routing computed on the GPU),
  both schedulers: logits / K/V against the oracle, and the device's top-8 in
  every layer against the ORACLE's own top-8 computed from the oracle's router
  logits (a mismatch is tolerated only at a near tie within 2x the router-logit
  error; counted).
* Qwen3-30B-A3B with the reference's own routing injected (golden
  `qwen3_bench_*`, drawn by the reference's moe_realization): device counts /
  exp_indptr / task indptr, executed and masked task counts, and (dynamic)
  pushes and pops bit-exact against the reference's simulate() of the same
  graph.
Tolerances are the ones stated in oracle/parity.py."""
import json
import os

import pytest
import torch

from oracle.parity import dense_parity, moe_parity
from paper_2604_13327_b200.decode import LLAMA3_8B, DecodeModel
from paper_2604_13327_b200.moe import QWEN3_30B_A3B, MoEDecodeModel

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def _report(name, r):
    print(name, json.dumps({k: v for k, v in r.items() if k != "seqs"}), flush=True)
    for t, x in r["seqs"].items():
        print("  seq", t, json.dumps(x), flush=True)


@pytest.fixture(scope="module")
def llama():
    m = DecodeModel(LLAMA3_8B, samples=(1024,), seed=0)
    yield m
    del m
    torch.cuda.empty_cache()


@pytest.mark.parametrize("s", [1024, 1000])
def test_llama8b_full_depth_bench_graph(llama, s):
    m = llama
    gold = GOLD["llama8b_bench"]
    m.fill_cache(s, seed=1)
    m.set_token(1)
    m.step(s)
    st = m.last_stats
    want = gold["simulate"][str(s)]
    assert st["tasks_executed"] + st["noop_tasks"] == want["num_records"]
    assert st["noop_tasks"] == want["noop_records"]
    assert st["tasks_executed"] == gold["instantiate"][str(s)]["num_tasks"]
    assert all(c == 0 for c in m.executor.final_counters())
    r = dense_parity(m.cfg, 0, m.device, [1], s, m.inv_freq, m.kcache, m.vcache, m.logits)
    _report(f"llama3-8b full depth s={s}", r)
    assert r["pass"], r


@pytest.mark.parametrize("scheduler", ["static", "dynamic"])
def test_qwen3_full_depth_computed_routing(scheduler):
    cfg, s = QWEN3_30B_A3B, 1024
    m = MoEDecodeModel(cfg, samples=(s,), seed=0, scheduler=scheduler)
    try:
        m.fill_cache(s, seed=1)
        m.set_token(1)
        m.step(s)
        assert all(c == 0 for c in m.executor.final_counters())
        mg = m.kernel.graph.instantiate({"s": s}, routing=m.realization())
        assert m.last_stats["tasks_executed"] == mg.num_tasks
        r = moe_parity(cfg, 0, m.device, [1], s, m.inv_freq, m.kcache, m.vcache, m.logits, m.logits_r,
                       lambda l, t: m.routing(l, 1)["topk"], xn_taps=m.xn)
    finally:
        del m
        torch.cuda.empty_cache()
    _report(f"qwen3-30b-a3b full depth ({scheduler})", r)
    # teacher-forced: the device router logits equal router @ the device's own
    # normalised activations in every layer (fp32 GEMV, ~1e-6 relative)
    assert max(r["seqs"]["0"]["per_layer"]["router_local_rel"]) <= 1e-4
    assert r["routing"]["mismatch"] == 0, r["routing"]
    assert r["pass"], r


@pytest.mark.parametrize("scheduler", ["static", "dynamic"])
def test_qwen3_bench_graph_reference_routing_accounting(scheduler):
    cfg, s = QWEN3_30B_A3B, 1024
    gold = GOLD[f"qwen3_bench_{scheduler}"]
    m = MoEDecodeModel(cfg, samples=(s,), seed=0, scheduler=scheduler)
    try:
        m.fill_cache(s, seed=1)
        m.set_token(1)
        m.inject_routing([gold["routing"][f"topk{l}"] for l in range(cfg.layers)])
        m.step(s)
        routing = [m.routing(l, 1) for l in range(cfg.layers)]
        st, counters = m.last_stats, m.executor.final_counters()
    finally:
        del m
        torch.cuda.empty_cache()
    for l in range(cfg.layers):
        for key in ("topk", "cnt", "ind", "tind"):
            assert routing[l][key] == gold["routing"][f"{key}{l}"], (l, key)
    want = gold["simulate"]
    assert st["tasks_executed"] + st["noop_tasks"] == want["num_records"]
    assert st["noop_tasks"] == want["noop_records"]
    assert st["tasks_executed"] == gold["instantiate"]["num_tasks"]
    if scheduler == "dynamic":
        assert st["pushes"] == gold["pushes"] and st["pops"] == gold["pops"]
    assert all(c == 0 for c in counters)
    assert want["final_counters"] == [0] * len(want["final_counters"])

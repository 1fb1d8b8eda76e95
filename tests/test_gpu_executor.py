"""GPU executor parity: the persistent megakernel runs the reference's
workloads; Event Tensor accounting (final counters, masked no-ops, executed
task counts) must equal the reference's, and every GPU trace must pass the
dependency checker (ref materialize.cpp:442-547)."""

import json

import numpy as np
import pytest
import torch

from paper_2604_13327_b200 import etsim
from paper_2604_13327_b200.ops import OP_SPLITK_FINAL, OP_SPLITK_PARTIAL, make_op, pack, ptr

pytestmark = pytest.mark.gpu


def test_splitk_rowsum_int32_bit_exact():
    n, parts, L = 37, 4, 1000
    g = etsim.splitk_rowsum()
    k = etsim.lower_static(g, [{"n": 16}, {"n": 64}], num_sms=8)
    rng = np.random.default_rng(0)
    data = rng.integers(-2**31, 2**31 - 1, size=(64, parts * L), dtype=np.int64).astype(np.int32)
    d_data = torch.from_numpy(data).cuda()
    d_part = torch.zeros(64 * parts, dtype=torch.int32, device="cuda")
    d_out = torch.zeros(64, dtype=torch.int32, device="cuda")
    ex = etsim.Executor(k, num_workers=8)
    ex.bind_ops(pack([make_op(OP_SPLITK_PARTIAL, i=[L, parts], p=[ptr(d_data), ptr(d_part)]),
                      make_op(OP_SPLITK_FINAL, i=[0, parts], p=[0, ptr(d_part), ptr(d_out)])]))
    stats = ex.run({"n": n})
    assert stats["sample_index"] == 1  # next-larger sample (64)
    want = data[:n].astype(np.int64).sum(axis=1)
    want = ((want + 2**31) % 2**32 - 2**31).astype(np.int32)  # int32 wraparound
    got = d_out[:n].cpu().numpy()
    assert np.array_equal(got, want)
    t = ex.trace()
    m = g.instantiate({"n": n})
    assert m.check(t) == []
    assert all(c == 0 for c in ex.final_counters())
    assert stats["tasks_executed"] == m.num_tasks
    assert stats["noop_tasks"] == (64 - n) * 5


def test_shape_sampling_masks_on_device():
    g = etsim.gemm_reduce_scatter("b * 2", 2)
    k = etsim.lower_static(g, [{"b": 1}, {"b": 2}, {"b": 4}, {"b": 8}], num_sms=2)
    for b in range(1, 9):
        t = etsim.simulate(k, {"b": b}, seed=b)
        m = g.instantiate({"b": b})
        assert m.check(t) == [], b
        assert t.num_records - t.noop_records == m.num_tasks
        assert all(c == 0 for c in t.final_counters)
    assert etsim.simulate(k, {"b": 3}).noop_records == 3
    with pytest.raises(etsim.GraphError):
        etsim.simulate(k, {"b": 9})


def test_random_dags_and_dma():
    for seed in range(12):
        g = etsim.random_dag(5 + seed % 16, 8 + seed % 20, seed)
        sms = 1 + seed % 4
        t = etsim.simulate(etsim.lower_static(g, [{}], num_sms=sms), {}, num_sms=sms, seed=seed)
        assert g.instantiate({}, seed=seed).check(t) == []
        assert all(c == 0 for c in t.final_counters)
    g = etsim.all_gather_gemm(4, 3)
    t = etsim.simulate(etsim.lower_static(g, [{}], num_sms=3), {})
    assert g.instantiate({}).check(t) == []


def test_moe_static_worst_case_masking():
    routing = etsim.moe_realization(tokens=16, experts=4, top_k=2, tile_size=2, hot_fraction=0.6, hot_expert=1, seed=3)
    g = etsim.moe_layer(tokens=16, experts=4, top_k=2, tile_size=2)
    sk = etsim.lower_static(etsim.worst_case_rewrite(g), [{"tokens": 16}], num_sms=4)
    t = etsim.simulate(sk, {"tokens": 16}, routing=routing, seed=3)
    tiles = routing["exp_indptr"][-1]
    assert t.noop_records == 16 * 2 - tiles
    assert all(c == 0 for c in t.final_counters)


def test_corrupted_queue_deadlock_detected():
    g = etsim.random_dag(8, 14, 0)
    k = etsim.lower_static(g, [{}], num_sms=1)
    m = g.instantiate({})
    doc = json.loads(k.to_json())
    q = doc["samples"][0]["sm_queues"][0]
    pi = ci = None
    for j in range(len(q)):
        for i in range(j):
            if pi is None and any(p == q[i]["id"] for el in m.task_waits[q[j]["id"]] for p in m.event_producers[el]):
                pi, ci = i, j
    moved = q.pop(pi)
    q.insert(ci, moved)
    bad = etsim.load_kernel(json.dumps(doc))
    with pytest.raises(etsim.SimulationError):
        etsim.simulate(bad, {}, num_sms=1)


def test_step_limit_is_typed():
    k = etsim.lower_static(etsim.gemm_reduce_scatter("4", 2), [{}], num_sms=2)
    with pytest.raises(etsim.SimulationError):
        etsim.simulate(k, step_limit=2)

"""MoE decode with data-dependent routing resolved on the GPU (tiny Qwen3-MoE-style
model, 16 experts, top-4) under both schedulers.

Bit-exact checks:
  * device top-k == CPU top-k (larger logit first, lower index on ties) on the
    device's own router logits, every layer;
  * expert counts, exp_indptr (tiles of TS tokens, ref workloads.cpp:137-144),
    task_indptr, eoff and elist == the CPU routing algebra of that top-k;
  * injected routing (etsim.moe_realization, the reference's seeded routing):
    device counts / exp_indptr == the realization's, bit for bit;
  * executed + masked task counts and the Event Tensor accounting == the
    reference instantiate() of the same graph with the device routing
    (check_trace clean, final counters 0).
Logits: max |err| <= 2e-3 * max|logit| + 2e-3 against the bf16-emulating
oracle (oracle/moe_oracle.py) run with the device's routing."""

import pytest
import torch

from oracle.moe_oracle import moe_decode_step, moe_routing_tensors, topk_ref
from oracle.decoder_oracle import weights_to_cpu
from paper_2604_13327_b200 import etsim
from paper_2604_13327_b200.moe import TINY_MOE, MoEDecodeModel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["static", "dynamic"])
def model(request):
    return MoEDecodeModel(TINY_MOE, samples=(16, 64), num_workers=16, seed=0, scheduler=request.param,
                          record_trace=True, keep_logical=True)


def _cpu_cache(m, seq=0):
    """CPU copy of one sequence's caches ([kv][cap][dh] per layer)."""
    return [k[seq].cpu() for k in m.kcache], [v[seq].cpu() for v in m.vcache]


@pytest.mark.parametrize("s,token", [(16, 3), (40, 11), (0, 5)])
def test_moe_logits_and_routing(model, s, token):
    m, cfg = model, model.cfg
    m.fill_cache(s, seed=2)
    m.set_token(token)
    ck, cv = _cpu_cache(m)
    logits = m.step(s)[0].cpu()
    K = cfg.top_k
    dev_topk = []
    for l in range(cfg.layers):
        r = m.routing(l)
        lg = m.logits_r[l, 0].cpu().tolist()
        assert r["topk"] == topk_ref(lg, K), (l, r["topk"], lg)           # routing indices
        want = moe_routing_tensors(r["topk"], cfg.experts, cfg.tile_tokens, cfg.row_splits)
        for key in ("cnt", "ind", "tind", "eoff", "elist"):
            assert r[key] == want[key], (l, key, r[key], want[key])       # counts / indptr bit-exact
        dev_topk.append(r["topk"])
    Wc = weights_to_cpu(m.W_logical)
    ref, ref_lg, ref_topk = moe_decode_step(cfg, Wc, ck, cv, token, s, m.inv_freq.cpu(), routing=dev_topk)
    err = (logits - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 2e-3 * scale + 2e-3, (err, scale)
    for l in range(cfg.layers):  # the device router logits agree with the oracle's
        d = (m.logits_r[l, 0].cpu() - ref_lg[l]).abs().max().item()
        assert d <= 2e-3 * ref_lg[l].abs().max().item() + 2e-3
    # Event Tensor accounting against the reference instantiate() with the device routing
    t = m.executor.trace()
    mg = m.kernel.graph.instantiate({"s": s}, routing=m.realization())
    assert mg.check(t) == [], mg.check(t)[:3]
    assert all(c == 0 for c in m.executor.final_counters())
    assert m.last_stats["tasks_executed"] == mg.num_tasks
    if not m.batched:  # the greedy token decided on the device
        assert m.greedy_token() == int(logits.argmax())


def test_moe_injected_routing_matches_reference_realization():
    cfg = TINY_MOE
    m = MoEDecodeModel(cfg, samples=(16,), num_workers=16, seed=0, scheduler="dynamic", record_trace=True)
    m.fill_cache(16, seed=2)
    m.set_token(7)
    reals = [etsim.moe_realization(tokens=1, experts=cfg.experts, top_k=cfg.top_k, tile_size=cfg.tile_tokens,
                                   seed=100 + l) for l in range(cfg.layers)]
    m.inject_routing([r["topk"] for r in reals])
    logits = m.step(16)
    assert torch.isfinite(logits).all()
    for l, real in enumerate(reals):
        r = m.routing(l)
        assert r["topk"] == list(real["topk"])
        assert r["cnt"] == list(real["expert_counts"])
        assert r["ind"] == list(real["exp_indptr"])
    t = m.executor.trace()
    mg = m.kernel.graph.instantiate({"s": 16}, routing=m.realization())
    assert mg.check(t) == []
    assert m.last_stats["tasks_executed"] == mg.num_tasks


@pytest.mark.parametrize("scheduler,max_batch,cases", [
    ("static", 8, ((1, 16), (3, 40), (8, 64))),
    ("dynamic", 8, ((1, 16), (3, 40), (8, 64))),
    ("static", 16, ((1, 16), (5, 40), (16, 64))),    # tensor-core projections (batch above 8)
    ("dynamic", 16, ((2, 16), (11, 64), (16, 40))),
])
def test_moe_batched_decode_no_recompile(scheduler, max_batch, cases):
    """One lowered artifact (batch symbol b <= max_batch) runs several batches, each
    sequence with its own KV cache and token: per-token routing bit-exact, per-sequence
    logits vs the oracle, and the Event Tensor accounting of the exact (s, b).  Above
    8 the dense projections run on tcgen05 (GEMV_TC) and the router logits come from
    a tensor-core GEMV before the route task."""
    cfg = TINY_MOE
    m = MoEDecodeModel(cfg, samples=(64,), num_workers=16, seed=0, scheduler=scheduler, record_trace=True,
                       keep_logical=True, max_batch=max_batch, batch_samples=(2, max_batch))
    Wc = weights_to_cpu(m.W_logical)
    toks = [(3 ** i + 7 * i) % cfg.vocab for i in range(max_batch)]
    for b, s in cases:
        m.fill_cache(s, seed=b)
        m.set_token(toks)
        from paper_2604_13327_b200.batch import cache_swizzle

        sw = cache_swizzle if m.tc else (lambda x: x)  # the tensor-core variant stores rows swizzled
        kc = [sw(k).cpu() for k in m.kcache]
        vc = [sw(v).cpu() for v in m.vcache]
        logits = m.step(s, b).cpu()
        for l in range(cfg.layers):
            r = m.routing(l, b)
            want_topk = []
            for t in range(b):
                want_topk += topk_ref(m.logits_r[l, t].cpu().tolist(), cfg.top_k)
            assert r["topk"] == want_topk, (b, l)
            want = moe_routing_tensors(r["topk"], cfg.experts, cfg.tile_tokens, cfg.row_splits)
            for key in ("cnt", "ind", "tind", "eoff", "elist"):
                assert r[key] == want[key], (b, l, key)
        for t in range(b):
            routing = [m.routing(l, b)["topk"][t * cfg.top_k:(t + 1) * cfg.top_k] for l in range(cfg.layers)]
            ref, _, _ = moe_decode_step(cfg, Wc, [k[t] for k in kc], [v[t] for v in vc], toks[t], s,
                                        m.inv_freq.cpu(), routing=routing)
            err = (logits[t] - ref).abs().max().item()
            scale = ref.abs().max().item()
            assert err <= 2e-3 * scale + 2e-3, (b, t, err, scale)
        mg = m.kernel.graph.instantiate(m._binding(s, b), routing=m.realization())
        assert mg.check(m.executor.trace()) == []
        assert m.last_stats["tasks_executed"] == mg.num_tasks
        assert all(c == 0 for c in m.executor.final_counters())


@pytest.mark.parametrize("scheduler", ["static", "dynamic"])
def test_moe_attention_head_split(scheduler):
    """head_split=2: each (kv head, split) runs as two tasks over half the q heads each
    (scalar split, output-projection merge); logits and routing as in the unsplit case."""
    m = MoEDecodeModel(TINY_MOE, samples=(16, 64), num_workers=16, seed=0, scheduler=scheduler,
                       keep_logical=True, head_split=2)
    assert m.head_split == 2
    for s, token in ((40, 11), (1, 5)):
        m.fill_cache(s, seed=2)
        m.set_token(token)
        ck, cv = _cpu_cache(m)
        logits = m.step(s)[0].cpu()
        dev_topk = [m.routing(l)["topk"] for l in range(m.cfg.layers)]
        ref, _, _ = moe_decode_step(m.cfg, weights_to_cpu(m.W_logical), ck, cv, token, s, m.inv_freq.cpu(),
                                    routing=dev_topk)
        err = (logits - ref).abs().max().item()
        scale = ref.abs().max().item()
        assert err <= 2e-3 * scale + 2e-3, (s, err, scale)

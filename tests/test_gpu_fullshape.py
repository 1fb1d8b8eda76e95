"""Parity at the real benchmark shapes (2 layers each, full hidden / heads /
intermediate / vocab): Llama-3-8B-shaped dense decode and Qwen3-30B-A3B-shaped
MoE decode (128 experts, top-8, routing computed on the GPU), against the CPU
oracles on the same weights.  These exercise what the tiny models cannot:
148-task GEMVs with balanced / split-K spans, K = 14336 activations, 16 attention
splits per kv head, 8 q heads per kv head, E/16 router tasks.
Tolerance: max|err| <= 1e-2 * max|logit| against the bf16-emulating oracle.  At
these sizes the kernel and the oracle round the bf16 activations (attention
output, SiLU product, normalised x) at the same points but from fp32 values
summed in a different order, so single-ulp flips of those activations (2^-8
relative) are expected and propagate; measured: ~2.5e-3 relative per layer
(1 layer) and ~4e-3 (2 layers) -- the tolerance is 2.5 bf16 epsilons.  The
attention output itself matches the oracle to 1 bf16 ulp (scripts/dbg_attn_num.py).
The greedy token (argmax) must agree whenever the oracle's top-2 margin exceeds
twice the error."""
import dataclasses

import pytest
import torch

from oracle.decoder_oracle import decode_step, weights_to_cpu
from oracle.moe_oracle import moe_decode_step, topk_ref
from paper_2604_13327_b200.decode import LLAMA3_8B, DecodeModel
from paper_2604_13327_b200.moe import QWEN3_30B_A3B, MoEDecodeModel

pytestmark = pytest.mark.gpu


def _check(logits, ref):
    err = (logits - ref).abs().max().item()
    scale = ref.abs().max().item()
    print(f"logits max abs err {err:.3e}, max rel err {err / scale:.3e} (scale {scale:.3f})")
    assert err <= 1e-2 * scale, (err, scale)
    top2 = ref.topk(2).values
    if (top2[0] - top2[1]).item() > 2 * err:
        assert logits.argmax().item() == ref.argmax().item()


def _cpu(m):
    """CPU caches of the (first) sequence, [kv][cap][dh] per layer."""
    pick = (lambda t: t[0]) if m.kcache[0].dim() == 4 else (lambda t: t)
    return [pick(k).cpu() for k in m.kcache], [pick(v).cpu() for v in m.vcache]


@pytest.mark.parametrize("s", [1024, 777])
def test_llama8b_shape_two_layers(s):
    cfg = dataclasses.replace(LLAMA3_8B, name="llama3-8b-2L", layers=2)
    m = DecodeModel(cfg, samples=(1024,), seed=0, record_trace=True, keep_logical=True)
    m.fill_cache(s, seed=1)
    m.set_token(123)
    ck, cv = _cpu(m)
    logits = m.step(s)[0].cpu()
    ref, _, _ = decode_step(cfg, weights_to_cpu(m.W_logical), ck, cv, 123, s, m.inv_freq.cpu())
    _check(logits, ref)
    assert m.graph.instantiate({"s": s}).check(m.executor.trace()) == []


@pytest.mark.parametrize("scheduler", ["static", "dynamic"])
def test_qwen3_moe_shape_two_layers(scheduler):
    cfg = dataclasses.replace(QWEN3_30B_A3B, name="qwen3-moe-2L", layers=2)
    s = 1024
    m = MoEDecodeModel(cfg, samples=(s,), seed=0, scheduler=scheduler, record_trace=True, keep_logical=True)
    m.fill_cache(s, seed=2)
    m.set_token(77)
    ck, cv = _cpu(m)
    logits = m.step(s)[0].cpu()
    dev_topk = []
    for l in range(cfg.layers):
        r = m.routing(l)
        assert r["topk"] == topk_ref(m.logits_r[l, 0].cpu().tolist(), cfg.top_k)
        assert sum(r["cnt"]) == cfg.top_k and r["ind"][-1] == cfg.top_k
        dev_topk.append(r["topk"])
    ref, _, _ = moe_decode_step(cfg, weights_to_cpu(m.W_logical), ck, cv, 77, s, m.inv_freq.cpu(), routing=dev_topk)
    _check(logits, ref)
    mg = m.kernel.graph.instantiate({"s": s}, routing=m.realization())
    assert mg.check(m.executor.trace()) == []
    assert m.last_stats["tasks_executed"] == mg.num_tasks


@pytest.mark.parametrize("b,s,scheduler", [(9, 1024, "static"), (64, 333, "static"), (24, 700, "dynamic")])
def test_llama8b_shape_batched_tensor_core(b, s, scheduler):
    """The tensor-core batch path at the real shapes (2 layers): 128-row blocks of the
    6144 / 4096 / 2x14336 / 128256-row projections, K = 14336 pieces, split-K adds,
    flat batch-dependent attention grid; sequences 0 and b-1 against the oracle."""
    from paper_2604_13327_b200.batch import BatchDecodeModel, cache_swizzle

    cfg = dataclasses.replace(LLAMA3_8B, name="llama3-8b-2L", layers=2)
    m = BatchDecodeModel(cfg, samples=(1024,), max_batch=64, seed=0, record_trace=True, keep_logical=True,
                         scheduler=scheduler)
    m.fill_cache(s, seed=1)
    toks = [(101 * i + 7) % cfg.vocab for i in range(b)]
    m.set_token(toks)
    kc = [cache_swizzle(k).cpu() for k in m.kcache]
    vc = [cache_swizzle(v).cpu() for v in m.vcache]
    logits = m.step(s, b).cpu()
    Wc = weights_to_cpu(m.W_logical)
    for t in (0, b - 1):
        ref, _, _ = decode_step(cfg, Wc, [k[t] for k in kc], [v[t] for v in vc], toks[t], s, m.inv_freq.cpu())
        _check(logits[t], ref)
    assert m.graph.instantiate({"s": s, "b": b}).check(m.executor.trace()) == []


@pytest.mark.parametrize("scheduler", ["static", "dynamic"])
def test_qwen3_moe_shape_batch32_tensor_core(scheduler):
    """Qwen3-MoE shape (2 layers) at batch 32 on the tensor-core variant: per-token
    routing bit-exact against the CPU top-k of the device logits, two sequences'
    logits against the oracle."""
    from paper_2604_13327_b200.batch import cache_swizzle

    cfg = dataclasses.replace(QWEN3_30B_A3B, name="qwen3-moe-2L", layers=2)
    b, s = 32, 200
    m = MoEDecodeModel(cfg, samples=(256,), seed=0, scheduler=scheduler, keep_logical=True, max_batch=32,
                       batch_samples=(32,))
    m.fill_cache(s, seed=1)
    toks = [(977 * i + 5) % cfg.vocab for i in range(b)]
    m.set_token(toks)
    kc = [cache_swizzle(k).cpu() for k in m.kcache]
    vc = [cache_swizzle(v).cpu() for v in m.vcache]
    logits = m.step(s, b).cpu()
    for l in range(cfg.layers):
        r = m.routing(l, b)
        want = []
        for t in range(b):
            want += topk_ref(m.logits_r[l, t].cpu().tolist(), cfg.top_k)
        assert r["topk"] == want
    Wc = weights_to_cpu(m.W_logical)
    for t in (0, b - 1):
        routing = [m.routing(l, b)["topk"][t * cfg.top_k:(t + 1) * cfg.top_k] for l in range(cfg.layers)]
        ref, _, _ = moe_decode_step(cfg, Wc, [k[t] for k in kc], [v[t] for v in vc], toks[t], s, m.inv_freq.cpu(),
                                    routing=routing)
        _check(logits[t], ref)

"""Decode-step numerics: megakernel logits vs the CPU fp32 oracle on the same
random-init weights (oracle/decoder_oracle.py).  Tolerances (bf16 weights,
fp32 accumulation):
  * vs the bf16-emulating oracle: max |err| <= 2e-3 * max|logit| + 2e-3
  * vs the pure fp32 oracle:      max |err| <= 5e-2 * max|logit| + 5e-2
and the appended K/V rows must equal the oracle's bf16 rows to 1 bf16 ulp."""

import pytest
import torch

from oracle.decoder_oracle import decode_step, weights_to_cpu
from paper_2604_13327_b200.decode import TINY, DecodeModel

pytestmark = pytest.mark.gpu


def _errs(got, want):
    err = (got - want).abs().max().item()
    scale = want.abs().max().item()
    return err, scale


@pytest.fixture(scope="module")
def tiny():
    return DecodeModel(TINY, samples=(16, 64), num_workers=16, seed=0, record_trace=True, keep_logical=True)


@pytest.mark.parametrize("s", [16, 10, 40, 0, 64])
def test_tiny_logits_match_oracle(tiny, s):
    m = tiny
    m.fill_cache(s, seed=1)
    m.set_token(7)
    cpu_k = [k.cpu() for k in m.kcache]
    cpu_v = [v.cpu() for v in m.vcache]
    logits = m.step(s)[0].cpu()
    Wc = weights_to_cpu(m.W_logical)
    inv = m.inv_freq.cpu()
    ref, nk, nv = decode_step(m.cfg, Wc, cpu_k, cpu_v, 7, s, inv, emulate_bf16=True)
    err, scale = _errs(logits, ref)
    assert err <= 2e-3 * scale + 2e-3, (s, err, scale)
    ref32, _, _ = decode_step(m.cfg, Wc, cpu_k, cpu_v, 7, s, inv, emulate_bf16=False)
    err32, scale32 = _errs(logits, ref32)
    assert err32 <= 5e-2 * scale32 + 5e-2, (s, err32, scale32)
    for l in range(m.cfg.layers):
        dk = m.kcache[l][:, s].float().cpu()
        dv = m.vcache[l][:, s].float().cpu()
        assert torch.allclose(dk, nk[l], rtol=1e-2, atol=1e-2)
        assert torch.allclose(dv, nv[l], rtol=1e-2, atol=1e-2)
    t = m.executor.trace()
    mg = m.graph.instantiate({"s": s})
    assert mg.check(t) == []
    assert all(c == 0 for c in m.executor.final_counters())
    assert m.last_stats["tasks_executed"] == mg.num_tasks
    # greedy token decided on the device (lm_head argmax words) == argmax of the logits
    assert m.greedy_token() == int(logits.argmax())


def test_greedy_token_on_device_across_steps(tiny):
    """The argmax word restarts every step (the embed zeroes it) and ET_OP_ARGMAX-style
    decoding follows the logits step after step (tokens fed back by the host)."""
    m = tiny
    m.fill_cache(20, seed=3)
    tok = 5
    for step in range(4):
        m.set_token(tok)
        logits = m.step(20 + step)[0]
        got = m.greedy_token()
        assert got == int(logits.argmax()), (step, got)
        tok = got


@pytest.fixture(scope="module")
def tiny_long():
    # 4 workers -> at most 2 attention splits per kv head: every split streams a run
    # of 64-position blocks with the online softmax (flash-decoding across blocks)
    return DecodeModel(TINY, samples=(512,), num_workers=4, seed=0, record_trace=True, keep_logical=True)


@pytest.mark.parametrize("s", [300, 512, 65, 1])
def test_tiny_multi_block_splits_match_oracle(tiny_long, s):
    m = tiny_long
    assert m.max_splits == 2
    m.fill_cache(s, seed=3)
    m.set_token(11)
    cpu_k = [k.cpu() for k in m.kcache]
    cpu_v = [v.cpu() for v in m.vcache]
    logits = m.step(s)[0].cpu()
    ref, _, _ = decode_step(m.cfg, weights_to_cpu(m.W_logical), cpu_k, cpu_v, 11, s, m.inv_freq.cpu(),
                            emulate_bf16=True)
    err, scale = _errs(logits, ref)
    assert err <= 2e-3 * scale + 2e-3, (s, err, scale)
    mg = m.graph.instantiate({"s": s})
    assert mg.check(m.executor.trace()) == []
    assert all(c == 0 for c in m.executor.final_counters())


@pytest.mark.parametrize("early", [False, True])
def test_tiny_dynamic_scheduler_matches_oracle(early):
    """The same decode graph under the on-GPU dynamic scheduler (push/pop ready
    queues, optional early push): logits and Event Tensor accounting."""
    m = DecodeModel(TINY, samples=(16, 64), num_workers=16, seed=0, record_trace=True, keep_logical=True,
                    scheduler="dynamic", early_push=early)
    for s in (16, 40):
        m.fill_cache(s, seed=1)
        m.set_token(5)
        cpu_k = [k.cpu() for k in m.kcache]
        cpu_v = [v.cpu() for v in m.vcache]
        logits = m.step(s)[0].cpu()
        ref, _, _ = decode_step(m.cfg, weights_to_cpu(m.W_logical), cpu_k, cpu_v, 5, s, m.inv_freq.cpu())
        err, scale = _errs(logits, ref)
        assert err <= 2e-3 * scale + 2e-3, (s, err, scale)
        mg = m.graph.instantiate({"s": s})
        assert mg.check(m.executor.trace()) == []
        assert m.last_stats["pushes"] == m.last_stats["pops"] == mg.num_tasks

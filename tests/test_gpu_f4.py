"""f4 (ref workloads.cpp:30-54): GEMM + reduce-scatter with real data on
the persistent kernel -- tcgen05 GEMM tiles into per-rank partials, reduce tiles gated by
their output tile's Event Tensor element.  Checked against torch's fp32 product of the
same bf16 operands (tolerance: bf16 output rounding + fp32 accumulation order)."""
import pytest
import torch

from paper_2604_13327_b200.f4 import GemmReduceScatter

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tokens,n,k,ranks", [(256, 256, 512, 2), (384, 512, 1024, 4), (1024, 1024, 2048, 2)])
def test_gemm_reduce_scatter_matches_torch(tokens, n, k, ranks):
    m = GemmReduceScatter(tokens=tokens, n=n, k=k, ranks=ranks, record_trace=True)
    out = m.step().float()
    ref = m.reference()
    err = (out - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 1e-2 * scale, (err, scale)
    # the per-rank partials sum to the product too (each is X[:, K_r] W[:, K_r]^T)
    assert torch.allclose(m.partials.sum(0), ref, rtol=1e-3, atol=1e-3 * scale)
    st = m.last_stats
    mg = m.graph.instantiate({})
    assert st["tasks_executed"] == mg.num_tasks
    assert mg.check(m.executor.trace()) == []
    assert all(c == 0 for c in m.executor.final_counters())


@pytest.mark.parametrize("push", [False, True])
def test_all_gather_gemm_matches_torch(push):
    from paper_2604_13327_b200.f4 import AllGatherGemm

    m = AllGatherGemm(tokens=1024, n=512, k=512, chunks=4, record_trace=True, push=push)
    out = m.step()
    ref = m.reference()
    err = (out - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 1e-3 * scale, (err, scale)
    if push:
        assert torch.equal(m.x_gather, m.x_src)
    mg = m.graph.instantiate({})
    assert m.last_stats["tasks_executed"] == mg.num_tasks
    assert mg.check(m.executor.trace()) == []
    assert all(c == 0 for c in m.executor.final_counters())

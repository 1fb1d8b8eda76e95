"""Tensor-parallel decode with the in-megakernel allreduce, TP=2 on ONE GPU:
two ranks = two runtimes in one process, each a persistent kernel on its own
stream (16 SMs each), peers mapped by plain device pointers (same address
space).  Exercises the cross-rank Event Tensor elements (st.release.sys /
ld.acquire.sys) and the P2P reads; the multi-process IPC exchange is covered
on CPU in test_tp_host.py.  The gathered logits must match the CPU oracle of
the full model (same tolerance as the single-GPU decode)."""
import pytest
import torch

from oracle.decoder_oracle import decode_step, weights_to_cpu
from paper_2604_13327_b200.decode import TINY, init_weights
from paper_2604_13327_b200.tp import TPDecodeModel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("s,token", [(16, 3), (40, 9)])
def test_tp2_logits_match_full_model_oracle(s, token):
    cfg, world = TINY, 2
    dev = torch.device("cuda:0")
    W = init_weights(cfg, dev, 0)
    ranks = [TPDecodeModel(cfg, r, world, device=dev, samples=(64,), num_workers=16, weights=W, record_trace=True)
             for r in range(world)]
    peers = [m.local_buffers() for m in ranks]
    for m in ranks:
        m.connect(peers)
        m.fill_cache(s, seed=1)
        m.set_token(token)
    streams = [torch.cuda.Stream() for _ in ranks]
    for step in range(3):  # several steps: epochs advance, no reset between steps
        for m, st in zip(ranks, streams):
            m.launch(s, st.cuda_stream)
        torch.cuda.synchronize()
        for m in ranks:
            m.executor.sync()  # raises on a device-reported deadlock / underflow
    logits = torch.cat([m.logits[0].cpu() for m in ranks])
    # oracle on the full weights and the full cache (rank caches are slices of it)
    full_k = [torch.cat([m.kcache[l] for m in ranks]).cpu() for l in range(cfg.layers)]
    full_v = [torch.cat([m.vcache[l] for m in ranks]).cpu() for l in range(cfg.layers)]
    for l in range(cfg.layers):  # undo this step's append (the oracle appends itself)
        full_k[l][:, s] = 0
        full_v[l][:, s] = 0
    ref, _, _ = decode_step(cfg, weights_to_cpu(W), full_k, full_v, token, s, ranks[0].inv_freq.cpu())
    err = (logits - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 2e-3 * scale + 2e-3, (err, scale)
    for m in ranks:
        t = m.executor.trace()
        assert m.graph.instantiate({"s": s}).check(t) == []
        assert all(c == 0 for c in m.executor.final_counters())


def test_tp2_llama70b_shape_two_layers_on_one_gpu():
    """Llama-3-70B-shaped layers (hidden 8192, 64 q / 8 kv heads, intermediate 28672,
    vocab 128256), 2 of the 80, TP=2 as two concurrent persistent kernels on one GPU
    (74 SMs each, tp.LocalTPGroup): the gathered logits against the full-model CPU
    oracle at the full-depth tolerance (oracle/parity.py), appended K/V per layer."""
    import dataclasses

    from oracle.parity import dense_parity
    from paper_2604_13327_b200.decode import LLAMA3_70B
    from paper_2604_13327_b200.tp import LocalTPGroup

    cfg, s, token = dataclasses.replace(LLAMA3_70B, layers=2), 300, 11
    dev = torch.device("cuda:0")
    g = LocalTPGroup(cfg, 2, device=dev, samples=(512,), seed=0)
    try:
        g.fill_cache(s, seed=1)
        g.set_token(token)
        g.launch(s)
        torch.cuda.synchronize()
        g.executor.sync()
        full_k = [torch.cat([m.kcache[l] for m in g.ranks]) for l in range(cfg.layers)]
        full_v = [torch.cat([m.vcache[l] for m in g.ranks]) for l in range(cfg.layers)]
        rep = dense_parity(cfg, 0, dev, [token], s, g.ranks[0].inv_freq, full_k, full_v, g.logits)
        print("llama3-70b 2L TP=2 on one GPU", rep)
        assert rep["pass"], rep
        for m in g.ranks:
            assert all(c == 0 for c in m.executor.final_counters())
    finally:
        del g
        torch.cuda.empty_cache()

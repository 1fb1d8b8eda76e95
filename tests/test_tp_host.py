"""Tensor-parallel host logic on CPU (no GPU): weight sharding covers the full
model exactly once, and the setup-time peer exchange over torch.distributed
(gloo, world_size 2) hands every rank the peers' buffers."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_2604_13327_b200.decode import TINY, frag16
from paper_2604_13327_b200.tp import exchange_peers, shard_weights


def _full_weights(cfg):
    g = torch.Generator().manual_seed(0)
    w = lambda *s: torch.randn(*s, generator=g).to(torch.bfloat16)  # noqa: E731
    W = {"embed": w(cfg.vocab, cfg.hidden), "final_norm": torch.ones(cfg.hidden), "lm_head": w(cfg.vocab, cfg.hidden),
         "layers": []}
    for _ in range(cfg.layers):
        W["layers"].append({"attn_norm": torch.ones(cfg.hidden), "ffn_norm": torch.ones(cfg.hidden),
                            "wqkv": w(cfg.q_rows + 2 * cfg.kv_rows, cfg.hidden), "wo": w(cfg.hidden, cfg.q_rows),
                            "wgate": w(cfg.intermediate, cfg.hidden), "wup": w(cfg.intermediate, cfg.hidden),
                            "wdown": w(cfg.hidden, cfg.intermediate)})
    return W


@pytest.mark.parametrize("world", [1, 2])
def test_shards_partition_the_model(world):
    cfg = TINY
    W = _full_weights(cfg)
    shards = [shard_weights(cfg, W, r, world) for r in range(world)]
    for name in ("wqkv", "wgate", "wup", "lm_head"):  # column-parallel: rows partitioned
        for l in range(cfg.layers if name != "lm_head" else 1):
            parts = [s["layers"][l][name] if name != "lm_head" else s["lm_head"] for s in shards]
            full = W["layers"][l][name] if name != "lm_head" else W["lm_head"]
            assert sum(p.shape[0] for p in parts) == full.shape[0]
            assert sum(p.float().sum().item() for p in parts) == pytest.approx(full.float().sum().item(), rel=1e-5)
    for l in range(cfg.layers):  # row-parallel: columns partitioned
        assert sum(s["layers"][l]["wo"].shape[1] for s in shards) == cfg.q_rows
        # the frag16 shard of Wo columns equals frag16 of the column slice
        cols = cfg.q_rows // world
        assert torch.equal(shards[-1]["layers"][l]["wo"], frag16(W["layers"][l]["wo"][:, (world - 1) * cols:].contiguous()))


def _worker(rank, world, port, out):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    local = (1000 + rank, 2000 + rank)
    peers = exchange_peers(local, rank, world, get_handle=lambda p: f"h{p}".encode(),
                           opener=lambda h: ("mapped", h.decode()))
    out[rank] = peers
    dist.destroy_process_group()


def test_peer_exchange_gloo_two_ranks():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0] == [(1000, 2000), (("mapped", "h1001"), ("mapped", "h2001"))]
    assert out[1] == [(("mapped", "h1000"), ("mapped", "h2000")), (1001, 2001)]


def test_streaming_shard_init_equals_sharding_the_full_model():
    from paper_2604_13327_b200.decode import init_weights
    from paper_2604_13327_b200.tp import init_shard

    cfg = TINY
    full = init_weights(cfg, torch.device("cpu"), 0)
    for r in range(2):
        a = init_shard(cfg, r, 2, torch.device("cpu"), 0)
        b = shard_weights(cfg, full, r, 2)
        assert torch.equal(a["lm_head"], b["lm_head"])
        for la, lb in zip(a["layers"], b["layers"]):
            for k in la:
                assert torch.equal(la[k], lb[k]), k

"""Tensor-parallel decode (Megatron sharding) on the megakernel: one rank per GPU,
row-parallel reductions as in-megakernel allreduce tasks over NVLink peer memory.

Rank r of TP holds:
- the q/k/v rows of its heads (nq/TP q heads, nkv/TP kv heads; column parallel);
- the Wo columns of those heads (row parallel);
- I/TP gate/up rows and the matching Wd columns;
- vocab/TP lm_head rows.

The embedding and the norms are replicated. Per layer the graph is

    qkv -> attn (fused merge) -> oproj -> ar_o -> gateup -> down -> ar_d

`oproj` and `down` store the rank's partial product into its own `part` slot.
The ALLREDUCE tasks (csrc/kernels/megakernel.cu body_allreduce) add every
rank's slot into the replicated residual stream. They wait on cross-GPU Event
Tensor elements (epoch = step id) that peers store into this rank's `flags`
with st.release.sys.

torch.distributed (NCCL or gloo) is used only at setup, to exchange the CUDA
IPC handles of `part` and `flags` (`exchange_peers`). The reference models TP
only as task graphs (ref workloads.cpp:30-79).
"""

import dataclasses
import json
import math
import time

import torch

from . import etsim
from .decode import attn_split_cap, frag16, init_weights, rope_inv_freq
from .graphs import graph_spec
from .ops import (
    EPI_F32,
    EPI_QKV_ROPE,
    EPI_SILU_MUL,
    OP_ALLREDUCE,
    OP_ATTN_SPLIT,
    OP_EMBED,
    OP_GEMV,
    make_op,
    pack,
    ptr,
)


def _shard_layer(cfg, L, rank, world):
    dh = cfg.head_dim
    hq, hk = cfg.heads // world, cfg.kv_heads // world
    I = cfg.intermediate // world
    nq, nkv = cfg.heads * dh, cfg.kv_heads * dh
    q = L["wqkv"][rank * hq * dh:(rank + 1) * hq * dh]
    k = L["wqkv"][nq + rank * hk * dh: nq + (rank + 1) * hk * dh]
    v = L["wqkv"][nq + nkv + rank * hk * dh: nq + nkv + (rank + 1) * hk * dh]
    return {
        "attn_norm": L["attn_norm"], "ffn_norm": L["ffn_norm"],
        "wqkv": frag16(torch.cat([q, k, v]).contiguous()),
        "wo": frag16(L["wo"][:, rank * hq * dh:(rank + 1) * hq * dh].contiguous()),
        "wgate": frag16(L["wgate"][rank * I:(rank + 1) * I].contiguous()),
        "wup": frag16(L["wup"][rank * I:(rank + 1) * I].contiguous()),
        "wdown": frag16(L["wdown"][:, rank * I:(rank + 1) * I].contiguous()),
    }


def init_shard(cfg, rank, world, device, seed=0):
    """This rank's shard of init_weights(cfg, seed) without ever holding the full
    model (layers are sharded as they are drawn: 70B fits a rank at any TP)."""
    V = cfg.vocab // world

    def hook(d):
        if "embed" in d:  # the top-level dict: keep the lm_head slice only
            d["lm_head"] = frag16(d["lm_head"][rank * V:(rank + 1) * V].contiguous())
            return d
        return _shard_layer(cfg, d, rank, world)

    return init_weights(cfg, device, seed, layer_hook=hook)


def shard_weights(cfg, W, rank, world):
    """Rank `rank`'s slices of the full (row-major bf16) weights, in frag16 order."""
    V = cfg.vocab // world
    return {"embed": W["embed"], "final_norm": W["final_norm"],
            "lm_head": frag16(W["lm_head"][rank * V:(rank + 1) * V].contiguous()),
            "layers": [_shard_layer(cfg, L, rank, world) for L in W["layers"]]}


def local_config(cfg, world):
    """The per-rank decoder shape (heads, kv heads, intermediate and vocab / TP)."""
    return dataclasses.replace(cfg, heads=cfg.heads // world, kv_heads=cfg.kv_heads // world,
                               intermediate=cfg.intermediate // world, vocab=cfg.vocab // world)


def tp_graph_spec(cfg, world, num_workers, samples, ar_tasks=None):
    """The graph one rank lowers (device-free; the committed bench-graph fixtures use it)."""
    lc = local_config(cfg, world)
    return graph_spec(lc, num_workers, num_workers, fused_merge=True, allreduce_tasks=ar_tasks or num_workers,
                      attn_cap=attn_split_cap(lc, max(samples), num_workers))


class TPDecodeModel:
    """Rank `rank` of a TP-way sharded Llama-style decoder (static scheduler)."""

    def __init__(self, cfg, rank, world, device="cuda:0", samples=(1024,), num_workers=None, seed=0, weights=None,
                 record_trace=False, ar_tasks=None):
        if not etsim.gpu_available():
            raise RuntimeError("TPDecodeModel needs a CUDA device")
        assert cfg.heads % world == 0 and cfg.kv_heads % world == 0 and cfg.intermediate % world == 0
        assert cfg.vocab % world == 0
        self.cfg, self.rank, self.world = cfg, rank, world
        self.device = torch.device(device)
        props = torch.cuda.get_device_properties(self.device)
        self.num_workers = num_workers or props.multi_processor_count
        self.samples = sorted(int(s) for s in samples)
        self.capacity = self.samples[-1] + 1
        self.local = local_config(cfg, world)
        self.ar_tasks = ar_tasks or self.num_workers
        self.max_splits = attn_split_cap(self.local, self.samples[-1], self.num_workers)
        t0 = time.perf_counter()
        spec = tp_graph_spec(cfg, world, self.num_workers, self.samples, self.ar_tasks)
        self.graph = etsim.Graph.from_json(json.dumps(spec))
        self.kernel = etsim.lower_static(self.graph, [{"s": s} for s in self.samples], num_sms=self.num_workers)
        self.lower_ms = (time.perf_counter() - t0) * 1e3
        dev = self.device
        self.W = shard_weights(cfg, weights, rank, world) if weights is not None else init_shard(cfg, rank, world, dev, seed)
        lc = self.local
        self.kcache = [torch.zeros(lc.kv_heads, self.capacity, cfg.head_dim, dtype=torch.bfloat16, device=dev)
                       for _ in range(cfg.layers)]
        self.vcache = [torch.zeros_like(k) for k in self.kcache]
        self.tokens = torch.zeros(1, dtype=torch.int32, device=dev)
        self.h = torch.zeros(1, cfg.hidden, dtype=torch.float32, device=dev)
        self.q = torch.zeros(lc.q_rows, dtype=torch.float32, device=dev)
        self.attn = torch.zeros(lc.q_rows, dtype=torch.bfloat16, device=dev)
        self.act = torch.zeros(lc.intermediate, dtype=torch.bfloat16, device=dev)
        self.partials = torch.zeros(lc.heads, self.max_splits, cfg.head_dim + 4, dtype=torch.float32, device=dev)
        self.arrive = torch.zeros(cfg.layers, lc.kv_heads, dtype=torch.int32, device=dev)
        self.logits = torch.zeros(1, lc.vocab, dtype=torch.float32, device=dev)   # this rank's vocab slice
        slots = 2 * cfg.layers
        self.part = torch.zeros(slots, cfg.hidden, dtype=torch.float32, device=dev)  # peer-visible partials
        self.flags = torch.zeros(slots, world, dtype=torch.int32, device=dev)        # peer-written Event Tensor elements
        self.once = torch.zeros(slots, dtype=torch.int32, device=dev)
        self.peer_table = torch.zeros(world, 2, dtype=torch.int64, device=dev)
        self.inv_freq = rope_inv_freq(cfg).to(dev)
        t1 = time.perf_counter()
        self.executor = etsim.Executor(self.kernel, device=dev.index or 0, num_workers=self.num_workers,
                                       record_trace=record_trace)
        self.upload_ms = (time.perf_counter() - t1) * 1e3
        self.connected = False

    # ------------------------------------------------------------------
    def local_buffers(self):
        """(part, flags) device addresses other ranks map."""
        return ptr(self.part), ptr(self.flags)

    def connect(self, peers):
        """peers[p] = (part address, flags address) of rank p as mapped in this process."""
        assert len(peers) == self.world
        self.peer_table.copy_(torch.tensor([[int(a), int(b)] for a, b in peers], dtype=torch.int64))
        self.executor.bind_ops(pack(self._ops()))
        self.connected = True

    def _ops(self):
        cfg, lc, W = self.cfg, self.local, self.W
        H, dh, CH = cfg.hidden, cfg.head_dim, cfg.attn_chunk
        G = lc.heads // lc.kv_heads
        scale = 1.0 / math.sqrt(dh)
        ops = [make_op(OP_EMBED, i=[H, -1], p=[ptr(W["embed"]), ptr(self.tokens), ptr(self.h)])]
        ar_p = [ptr(self.h), ptr(self.flags), ptr(self.once), ptr(self.peer_table)]
        for l, L in enumerate(W["layers"]):
            kc, vc = self.kcache[l], self.vcache[l]
            ops.append(make_op(OP_GEMV, i=[lc.q_rows + 2 * lc.kv_rows, H, 1, 1, EPI_QKV_ROPE, -1, 0, 16, dh, H,
                                           lc.q_rows, lc.kv_rows, self.capacity],
                               f=[cfg.eps], p=[ptr(L["wqkv"]), 0, ptr(self.h), ptr(L["attn_norm"]), ptr(self.q), 0,
                                               ptr(kc), ptr(vc), ptr(self.inv_freq)]))
            attn_i = [dh, G, CH, self.capacity, 0, self.max_splits, lc.kv_heads]
            ops.append(make_op(OP_ATTN_SPLIT, i=attn_i, f=[scale], flags=2,
                               p=[ptr(self.q), ptr(kc), ptr(vc), ptr(self.partials), ptr(self.attn),
                                  ptr(self.arrive[l])]))
            ops.append(make_op(OP_GEMV, i=[H, lc.q_rows, 1, 0, EPI_F32, -1, 0, 16],
                               p=[ptr(L["wo"]), 0, ptr(self.attn), 0, ptr(self.part[2 * l])]))
            ops.append(make_op(OP_ALLREDUCE, i=[H, self.world, self.rank, 2 * l], p=ar_p))
            ops.append(make_op(OP_GEMV, i=[lc.intermediate, H, 2, 1, EPI_SILU_MUL, -1, 0, 16, 0, H], f=[cfg.eps],
                               p=[ptr(L["wgate"]), ptr(L["wup"]), ptr(self.h), ptr(L["ffn_norm"]), ptr(self.act)]))
            ops.append(make_op(OP_GEMV, i=[H, lc.intermediate, 1, 0, EPI_F32, -1, 0, 16],
                               p=[ptr(L["wdown"]), 0, ptr(self.act), 0, ptr(self.part[2 * l + 1])]))
            ops.append(make_op(OP_ALLREDUCE, i=[H, self.world, self.rank, 2 * l + 1], p=ar_p))
        ops.append(make_op(OP_GEMV, i=[lc.vocab, H, 1, 1, EPI_F32, -1, 0, 16, 0, H], f=[cfg.eps],
                           p=[ptr(W["lm_head"]), 0, ptr(self.h), ptr(W["final_norm"]), ptr(self.logits)]))
        return ops

    def fill_cache(self, s, seed=1, full_cache=None):
        """Synthetic KV cache: this rank's kv heads of the full-model cache N(0,1) (same seed on every rank)."""
        lc = self.local
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        for l in range(self.cfg.layers):
            k = torch.zeros(self.cfg.kv_heads, self.capacity, self.cfg.head_dim, dtype=torch.bfloat16,
                            device=self.device)
            v = torch.zeros_like(k)
            k[:, :s].normal_(0.0, 1.0, generator=g)
            v[:, :s].normal_(0.0, 1.0, generator=g)
            sl = slice(self.rank * lc.kv_heads, (self.rank + 1) * lc.kv_heads)
            self.kcache[l].copy_(k[sl])
            self.vcache[l].copy_(v[sl])

    def set_token(self, token):
        self.tokens.fill_(int(token))

    def launch(self, s, stream=0):
        assert self.connected, "connect() the peers first"
        self.executor.launch({"s": int(s)}, stream)


def exchange_peers(local_ptrs, rank, world, group=None, get_handle=None, opener=None):
    """Setup-only exchange of every rank's (part, flags) buffers over
    torch.distributed: all-gathers their CUDA IPC handles and opens the peers'
    handles in this process.  Returns peers[p] = (part, flags) addresses usable
    by this rank's kernel (its own buffers for p == rank).  `get_handle` /
    `opener` default to etsim.ipc_handle / etsim.ipc_open (injectable for CPU tests)."""
    import torch.distributed as dist

    get_handle = get_handle or etsim.ipc_handle
    opener = opener or (lambda h: etsim.ipc_open(h, torch.cuda.current_device()))
    mine = tuple(get_handle(p) for p in local_ptrs)
    handles = [None] * world
    dist.all_gather_object(handles, mine, group=group)
    return [tuple(local_ptrs) if p == rank else tuple(opener(h) for h in handles[p]) for p in range(world)]


class LocalTPGroup:
    """All TP ranks of a sharded decoder in ONE process on ONE GPU (a single-GPU
    pool): each rank is its own persistent kernel on its own stream over
    num_workers // world SMs, peers mapped by plain device pointers.  The ranks
    share one token buffer and write their vocab slices into one logits row, so
    the group looks like one model to a caller (launch / executor.sync / logits).
    The cross-rank Event Tensor elements and the peer reads are exactly the
    multi-GPU ones; only NVLink is replaced by the GPU's own memory."""

    class _Sync:
        def __init__(self, ranks):
            self.ranks = ranks

        def sync(self):
            out = {}
            for m in self.ranks:  # per-rank counts summed over the group
                for k, v in m.executor.sync().items():
                    out[k] = out.get(k, 0) + v if isinstance(v, (int, float)) and k != "kernel_ms" else v
            return out

    def __init__(self, cfg, world, device="cuda:0", samples=(1024,), seed=0, weights=None, record_trace=False):
        dev = torch.device(device)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        self.cfg, self.world, self.device = cfg, world, dev
        self.ranks = [TPDecodeModel(cfg, r, world, device=dev, samples=samples, num_workers=sms // world, seed=seed,
                                    weights=weights, record_trace=record_trace) for r in range(world)]
        self.tokens = torch.zeros(1, dtype=torch.int32, device=dev)
        self.logits = torch.zeros(1, cfg.vocab, dtype=torch.float32, device=dev)
        V = cfg.vocab // world
        for r, m in enumerate(self.ranks):
            m.tokens = self.tokens
            m.logits = self.logits[:, r * V:(r + 1) * V]
        peers = [m.local_buffers() for m in self.ranks]
        for m in self.ranks:
            m.connect(peers)
        self.streams = [torch.cuda.Stream(device=dev) for _ in self.ranks]
        self.executor = LocalTPGroup._Sync(self.ranks)
        self.local = self.ranks[0].local
        self.lower_ms = sum(m.lower_ms for m in self.ranks)
        self.upload_ms = sum(m.upload_ms for m in self.ranks)

    def fill_cache(self, s, seed=1):
        for m in self.ranks:
            m.fill_cache(s, seed=seed)

    def set_token(self, token):
        self.tokens.fill_(int(token))

    def launch(self, s, stream=0):
        """Every rank's step, ordered after the work already on `stream`, which then
        waits for all of them (events time the whole TP step on `stream`)."""
        main = torch.cuda.ExternalStream(stream, device=self.device) if stream else torch.cuda.current_stream(self.device)
        start = torch.cuda.Event()
        start.record(main)
        done = []
        for m, st in zip(self.ranks, self.streams):
            st.wait_event(start)
            m.launch(s, st.cuda_stream)
            e = torch.cuda.Event()
            e.record(st)
            done.append(e)
        for e in done:
            main.wait_event(e)

    def step_bytes(self, s):
        return self.world * self.local.step_bytes(s)

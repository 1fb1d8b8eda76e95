"""Large-batch decode: the batch is a graph symbol `b` (1..max_batch, up to 128)
next to the position symbol `s`, and every projection runs on the 5th-generation
tensor cores (ET_OP_GEMV_TC: tcgen05.mma, accumulators in TMEM).

One lowered artifact serves every (s, b) covered by its samples: grids that
depend on `b` (norms, attention) shrink on device, the GEMV tasks read the
batch from the binding, no recompilation or relaunch.

Graph per layer l (Event Tensors, counts derived by the reference lowering):
    norm1_l  [b]                 waits D_{l-1}[0]  notifies N1_l[0]
    qkv_l    [Tq]                waits N1_l[0]     notifies QKV_l[0]
    attn_l   [b*kv*splits(s,b)]  waits QKV_l[0]    notifies M_l[0]   (fused merge; fewer,
                                                                       longer splits as b grows)
    oproj_l  [To]                waits M_l[0]      notifies O_l[0]
    norm2_l  [b]                 waits O_l[0]      notifies N2_l[0]
    gateup_l [Tg]                waits N2_l[0]     notifies G_l[0]
    down_l   [Td]                waits G_l[0]      notifies D_l[0]
then normf [b] and lm_head [Tl].

Device layout (HBM):
  * weights: per projection, pieces of kp input columns; inside a piece, blocks
    of 128 output rows; inside a block, k steps of 16 (4 KB each) holding 16 x 2
    core matrices of 8 rows x 8 bf16 (tc_pack) -- one 16 KB ring chunk is one
    block x 64 k, the A operand of four K=16 MMAs as it lands;
  * activations feeding a projection: bf16 in the matching operand layout
    (ops.cuh xb_offset) written by the producer (norm, attention merge, SiLU-mul
    epilogue), so each piece reaches shared memory with one bulk copy;
  * residual stream fp32 [b][H] (row-parallel projections red.add into it),
    raw q/k/v fp32 [b][rows] (split-K adds; the attention merger zeroes them),
    KV caches bf16 [b][kv][capacity][head_dim] per layer, each row's 16-byte chunks
    XOR-swizzled by position % 8 (cache_swizzle) so the tensor-core attention reads
    8 rows from 8 different bank groups.
"""

import json
import math
import time

import torch

from . import etsim
from .decode import DecoderConfig, attn_split_cap, init_weights, rope_inv_freq
from .ops import (
    EPI_ADD,
    EPI_F32,
    EPI_SILU_MUL,
    OP_ATTN_SPLIT,
    OP_EMBED,
    OP_GEMV_TC,
    OP_NORM,
    make_op,
    pack,
    ptr,
)

TMEM_COLS = 512
XBUF_BYTES = 16384


def tc_npad(b):
    """Batch rounded up to the MMA N dimension (multiple of 16, >= 16); ops.cuh tc_npad."""
    return 16 if b <= 16 else (b + 15) // 16 * 16


def tc_piece(max_batch):
    """Piece length kp: one activation piece (npad x kp bf16) fills a 16 KB x buffer."""
    kp = XBUF_BYTES // (2 * tc_npad(max_batch))
    return min(512, kp // 64 * 64)


def cache_swizzle(t):
    """K/V cache rows with their 16-byte (8-element) chunks XOR-permuted by position % 8
    (attention flags bit 8): the device layout <-> the logical [.., cap, dh] rows.  An
    involution, so the same call converts either way."""
    *lead, cap, dh = t.shape
    pos = torch.arange(cap, device=t.device).view(cap, 1)
    chunk = torch.arange(dh // 8, device=t.device).view(1, dh // 8)
    src = (chunk ^ (pos % 8)).view(*([1] * len(lead)), cap, dh // 8, 1).expand(*lead, cap, dh // 8, 8)
    return torch.gather(t.reshape(*lead, cap, dh // 8, 8), -2, src).reshape(t.shape)


def tc_piece_for(max_batch, ks):
    """tc_piece(max_batch), reduced until it divides every projection input width in ks."""
    kp = tc_piece(max_batch)
    while any(k % kp for k in ks):
        kp -= 64
    assert kp >= 64, ks
    return kp


def tc_pack(w, kp):
    """[N][K] bf16 -> the tensor-core layout [K/kp][N/128][kp/16][16][2][8][8]
    (piece, row block, k step, 8-row group, k half, row, k)."""
    N, K = w.shape
    assert N % 128 == 0 and K % kp == 0 and kp % 64 == 0, (N, K, kp)
    v = w.reshape(N // 128, 16, 8, K // kp, kp // 16, 2, 8)
    return v.permute(3, 0, 4, 1, 5, 2, 6).contiguous().reshape(-1)


def xb_unpack(buf, b, K, npad, kp):
    """Inverse of the activation operand layout (tests): [b][K] fp32 from the bf16 buffer."""
    v = buf[: npad * K].reshape(K // kp, kp // 16, npad // 8, 2, 8, 8)   # piece, kstep, ngroup, khalf, n, k
    return v.permute(2, 4, 0, 1, 3, 5).reshape(npad, K)[:b].float()


def tc_tasks(nblk, workers, splittable, nseg=1, npad=64, pieces=1):
    """(tasks, k splits) of a projection: one 128-row block per group and enough
    k splits to cover the workers when the epilogue adds (split-K: at most one
    wave -- 32 blocks x 5 splits = 160 tasks on 148 SMs put a second task on 12
    of them and doubled the stage's tail; two blocks per task with twice the
    splits, halving the activation re-reads, measured slower: more tasks and
    red.add traffic); otherwise groups of blocks small enough that two MMA
    issuers fit their accumulators in TMEM (ops.cuh kTcIssuers)."""
    if splittable:
        splits = max(1, min(pieces, workers // nblk))
        return nblk * splits, splits
    per = max(1, TMEM_COLS // (2 * nseg * npad))  # blocks per task that leave TMEM for 2 MMA issuers
    groups = max(min(workers, nblk), -(-nblk // per))
    if groups > workers:
        # more than one wave (lm_head: 1002 blocks): one wave of larger tasks with one MMA
        # issuer each (TMEM holds up to 512 / (nseg * npad) blocks) -- a streaming issuer
        # keeps up with the SM's share of HBM, a second wave doubles the stage
        groups = max(workers, -(-nblk // max(1, TMEM_COLS // (nseg * npad))))
    return groups, 1


def attn_budget(cfg, workers, per_sm=2):
    """Per-step split budget of the batched attention: splits per (sequence, kv head)
    <= max(1, budget // b), about `per_sm` attention tasks per SM at any batch."""
    return max(1, per_sm * workers // cfg.kv_heads)


def attn_grid(cfg, attn_cap, budget):
    """Flat attention grid [b * kv * splits] (ops.cuh attn_coord, flags bit 7)."""
    CH = cfg.attn_chunk
    return f"b * {cfg.kv_heads} * max(1, min(min((s + {CH - 1}) // {CH}, {attn_cap}), {budget} // b))"


def batch_graph_spec(cfg, tasks, attn_cap, budget):
    """Reference-format graph spec (ref json_io.cpp:115-230) of one batched decode step."""
    CH, kv = cfg.attn_chunk, str(cfg.kv_heads)
    fns, events, calls = [], [], []

    def fn(name, grid):
        fns.append({"name": name, "grid": grid, "resource": "sm", "duration": "unit"})
        return name

    def call(f, grid, prev, out):
        events.append({"name": out, "shape": ["1"]})
        calls.append({"fn": fn(f, grid), "in": [{"event": prev, "map": ["0"]}] if prev else [],
                      "out": [{"event": out, "map": ["0"]}]})
        return out

    prev = call("embed", ["1"], None, "EMB")
    calls[-1].pop("in")
    for l in range(cfg.layers):
        prev = call(f"L{l}.norm1", ["b"], prev, f"N1{l}")
        prev = call(f"L{l}.qkv", [str(tasks["qkv"])], prev, f"QKV{l}")
        prev = call(f"L{l}.attn", [attn_grid(cfg, attn_cap, budget)], prev, f"M{l}")
        prev = call(f"L{l}.oproj", [str(tasks["oproj"])], prev, f"O{l}")
        prev = call(f"L{l}.norm2", ["b"], prev, f"N2{l}")
        prev = call(f"L{l}.gateup", [str(tasks["gateup"])], prev, f"G{l}")
        prev = call(f"L{l}.down", [str(tasks["down"])], prev, f"D{l}")
    prev = call("normf", ["b"], prev, "NF")
    call("lm_head", [str(tasks["lm"])], prev, "LM")
    return {"symbols": ["s", "b"], "size_symbol": "s", "duration_models": {"unit": {"kind": "constant", "value": 1}},
            "device_functions": fns, "event_tensors": events, "calls": calls}


def batch_layout(cfg, num_workers, samples, max_batch=64, batch_samples=None, kp=None, attn_tasks_per_sm=2):
    """Every layout choice BatchDecodeModel makes before touching the device (graph
    spec, bindings, task counts, piece length).  Device-free, so the committed
    bench-graph fixtures are exactly the graphs the model lowers."""
    assert 1 <= max_batch <= 128
    L = {"max_batch": max_batch}
    # batch samples: powers of two up to max_batch by default, so a small batch runs on a
    # schedule at most twice its size (masked tasks still wait and notify)
    default = [1 << i for i in range(8) if (1 << i) < max_batch]
    L["batch_samples"] = sorted(set(batch_samples or default) | {max_batch})
    L["samples"] = sorted(int(s) for s in samples)
    L["capacity"] = L["samples"][-1] + 1
    # piece length (input columns per activation piece); kp overrides (multiple of 64)
    kp = kp or tc_piece_for(max_batch, (cfg.hidden, cfg.q_rows, cfg.intermediate))
    L["kp"] = kp
    npad = tc_npad(max_batch)
    H, I, nq, nkv = cfg.hidden, cfg.intermediate, cfg.q_rows, cfg.kv_rows
    rows = nq + 2 * nkv
    for k in (H, nq, I):
        assert k % kp == 0, (k, kp)
    tasks, splits = {}, {}
    for name, n, k, add, nseg in (("qkv", rows, H, True, 1), ("oproj", H, nq, True, 1),
                                  ("gateup", I, H, False, 2), ("down", H, I, True, 1),
                                  ("lm", cfg.vocab, H, False, 1)):
        tasks[name], splits[name] = tc_tasks(n // 128, num_workers, add, nseg, npad, k // kp)
    L["tasks"], L["splits"] = tasks, splits
    # attention splits per (sequence, kv head): half the batch-1 cap -- a split runs its
    # blocks two at a time (warps 0-3 / 4-7), so it should own at least two
    L["max_splits"] = max(1, attn_split_cap(cfg, L["samples"][-1], num_workers) // 2)
    L["attn_budget"] = attn_budget(cfg, num_workers, attn_tasks_per_sm)
    L["spec"] = batch_graph_spec(cfg, tasks, L["max_splits"], L["attn_budget"])
    L["bindings"] = [{"s": s, "b": b} for s in L["samples"] for b in L["batch_samples"]]
    return L


class BatchDecodeModel:
    """Llama-style decoder, batch 1..max_batch (<= 128) and sequence length up to the
    largest sample on one lowered artifact; projections on tcgen05 tensor cores."""

    def __init__(self, cfg: DecoderConfig, device="cuda:0", samples=(1024,), max_batch=64, batch_samples=None,
                 num_workers=None, seed=0, weights=None, scheduler="static", record_trace=False, keep_logical=False,
                 kp=None, attn_tasks_per_sm=2):
        if not etsim.gpu_available():
            raise RuntimeError("BatchDecodeModel needs a CUDA device (the executor has no CPU fallback)")
        assert 1 <= max_batch <= 128
        self.cfg = cfg
        self.device = torch.device(device)
        props = torch.cuda.get_device_properties(self.device)
        self.num_workers = num_workers or props.multi_processor_count
        self.scheduler = scheduler
        t0 = time.perf_counter()
        for k, v in batch_layout(cfg, self.num_workers, samples, max_batch, batch_samples, kp,
                                 attn_tasks_per_sm).items():
            setattr(self, k, v)
        kp, npad = self.kp, tc_npad(max_batch)
        H, I, nq, nkv = cfg.hidden, cfg.intermediate, cfg.q_rows, cfg.kv_rows
        rows = nq + 2 * nkv
        self.graph = etsim.Graph.from_json(json.dumps(self.spec))
        if scheduler == "dynamic":
            self.kernel = etsim.lower_dynamic(self.graph)
        else:
            self.kernel = etsim.lower_static(self.graph, self.bindings, num_sms=self.num_workers)
        self.lower_ms = (time.perf_counter() - t0) * 1e3

        dev = self.device
        W = weights if weights is not None else init_weights(cfg, dev, seed)
        self.W_logical = W if keep_logical else None
        self.W = self._layout(W, keep_logical)
        B = max_batch
        self.kcache = [torch.zeros(B, cfg.kv_heads, self.capacity, cfg.head_dim, dtype=torch.bfloat16, device=dev)
                       for _ in range(cfg.layers)]
        self.vcache = [torch.zeros_like(k) for k in self.kcache]
        self.tok = torch.zeros(B, dtype=torch.int32, device=dev)
        self.h = torch.zeros(B, H, dtype=torch.float32, device=dev)
        self.xn = torch.zeros(npad * H, dtype=torch.bfloat16, device=dev)       # normed stream (operand layout)
        self.qkv = torch.zeros(B, rows, dtype=torch.float32, device=dev)        # raw projections (split-K adds)
        self.attn = torch.zeros(npad * nq, dtype=torch.bfloat16, device=dev)    # attention out (operand layout)
        self.act = torch.zeros(npad * I, dtype=torch.bfloat16, device=dev)      # silu(gate)*up (operand layout)
        # split stride max(splits, 8): a lone split leaves its 8 warp partials (flags bit 9)
        self.partials = torch.zeros(B * cfg.heads, max(8, self.max_splits), cfg.head_dim + 4, dtype=torch.float32,
                                    device=dev)
        self.arrive = torch.zeros(cfg.layers, B * cfg.kv_heads, dtype=torch.int32, device=dev)
        self.logits = torch.zeros(B, cfg.vocab, dtype=torch.float32, device=dev)
        self.inv_freq = rope_inv_freq(cfg).to(dev)

        t1 = time.perf_counter()
        if scheduler == "dynamic":
            self.executor = etsim.Executor(self.kernel, self.bindings, device=dev.index or 0,
                                           num_workers=self.num_workers, record_trace=record_trace,
                                           max_batch=max_batch)
        else:
            self.executor = etsim.Executor(self.kernel, device=dev.index or 0, num_workers=self.num_workers,
                                           record_trace=record_trace, max_batch=max_batch)
        self.executor.bind_ops(pack(self._ops()))
        self.upload_ms = (time.perf_counter() - t1) * 1e3

    def _layout(self, W, keep_logical):
        kp = self.kp
        D = {"embed": W["embed"], "final_norm": W["final_norm"], "lm_head": tc_pack(W["lm_head"], kp), "layers": []}
        for L in W["layers"]:
            D["layers"].append({"attn_norm": L["attn_norm"], "ffn_norm": L["ffn_norm"],
                                **{k: tc_pack(L[k], kp) for k in ("wqkv", "wo", "wgate", "wup", "wdown")}})
            if not keep_logical:
                for k in ("wqkv", "wo", "wgate", "wup", "wdown"):
                    L[k] = None
        if not keep_logical:
            W["lm_head"] = None
        return D

    def _ops(self):
        cfg, W, kp = self.cfg, self.W, self.kp
        H, I, nq, dh, CH = cfg.hidden, cfg.intermediate, cfg.q_rows, cfg.head_dim, cfg.attn_chunk
        rows = nq + 2 * cfg.kv_rows
        G = cfg.heads // cfg.kv_heads
        bs = 1  # binding slot of `b`
        sp = self.splits

        def tc(n, k, nseg, epi, w0, w1, x, out, splits, kp_out=0):
            return make_op(OP_GEMV_TC, i=[n, k, nseg, splits, epi, bs, kp, kp_out],
                           p=[ptr(w0), ptr(w1), ptr(x), 0, ptr(out)])

        def norm(gamma):
            return make_op(OP_NORM, i=[H, 0, 0, 0, 0, bs, kp], f=[cfg.eps], p=[ptr(self.h), ptr(gamma), ptr(self.xn)])

        ops = [make_op(OP_EMBED, i=[H, bs], p=[ptr(W["embed"]), ptr(self.tok), ptr(self.h)])]
        for l, L in enumerate(W["layers"]):
            ops.append(norm(L["attn_norm"]))
            ops.append(tc(rows, H, 1, EPI_ADD, L["wqkv"], None, self.xn, self.qkv, sp["qkv"]))
            # flags: 1 q/k fused mode, 2 fused merge, 32 zero the raw q/k/v after use, 64 RoPE only,
            # 128 flat batch-dependent grid, 256 chunk-swizzled cache rows (cache_swizzle),
            # 512 a lone split leaves its 8 warp partials to the merge
            ops.append(make_op(OP_ATTN_SPLIT,
                               i=[dh, G, CH, self.capacity, 0, self.max_splits, cfg.kv_heads, rows,
                                  cfg.kv_heads * self.capacity * dh, kp, bs, self.attn_budget],
                               f=[1.0 / math.sqrt(dh), cfg.eps], flags=1 | 2 | 32 | 64 | 128 | 256 | 512,
                               p=[ptr(self.qkv), ptr(self.kcache[l]), ptr(self.vcache[l]), ptr(self.partials),
                                  ptr(self.attn), ptr(self.arrive[l]), 0, ptr(self.inv_freq),
                                  ptr(self.qkv) + 4 * nq, 0]))
            ops.append(tc(H, nq, 1, EPI_ADD, L["wo"], None, self.attn, self.h, sp["oproj"]))
            ops.append(norm(L["ffn_norm"]))
            ops.append(tc(I, H, 2, EPI_SILU_MUL, L["wgate"], L["wup"], self.xn, self.act, 1, kp_out=kp))
            ops.append(tc(H, I, 1, EPI_ADD, L["wdown"], None, self.act, self.h, sp["down"]))
        ops.append(norm(W["final_norm"]))
        ops.append(tc(cfg.vocab, H, 1, EPI_F32, W["lm_head"], None, self.xn, self.logits, 1))
        return ops

    def fill_cache(self, s, seed=1):
        """Synthetic prefilled caches, N(0, 1) bf16 for positions [0, s) of every sequence."""
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        for k, v in zip(self.kcache, self.vcache):
            k.zero_()
            v.zero_()
            k[..., :s, :].normal_(0.0, 1.0, generator=g)
            v[..., :s, :].normal_(0.0, 1.0, generator=g)

    def set_token(self, token):
        if isinstance(token, (list, tuple)):
            self.tok[: len(token)].copy_(torch.tensor(token, dtype=torch.int32))
        else:
            self.tok.fill_(int(token))

    def step(self, s, b):
        self.last_stats = self.executor.run({"s": int(s), "b": int(b)})
        return self.logits[:b]

    def launch(self, s, b, stream=0):
        self.executor.launch({"s": int(s), "b": int(b)}, stream)

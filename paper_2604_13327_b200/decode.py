"""Event Tensor graphs for LLM decode and their GPU runtime.

The reference has no transformer template (ref SPEC.md:515); this module
expresses one decode step of a Llama-style decoder in the reference's own
graph-spec format (the JSON schema of ref src/json_io.cpp:115-230), lowers it
with the reference-compatible static scheduler (`lower_static`), binds every
call to a tile operation of the megakernel and runs it with one persistent
launch per step.

Graph per layer l (all events are Event Tensors; counts are derived):
    qkv_l   [T]            waits D_{l-1}[0]      notifies QKV_l[0]
    attn_l  [kv, ceil(s/CH)] waits QKV_l[0]      notifies A_l[t0]
    merge_l [kv]           waits A_l[t0], QKV_l[0] notifies M_l[0]
    oproj_l [T]            waits M_l[0]          notifies O_l[0]
    gateup_l[T]            waits O_l[0]          notifies G_l[0]
    down_l  [T]            waits G_l[0]          notifies D_l[0]
followed by lm_head [T_lm] waiting on D_{L-1}[0].  `s` (cached positions) is
the graph's symbolic size: one compiled artifact serves every sequence length
covered by its samples, with out-of-range attention splits masked on device.

Device layout (HBM): GEMV weights bf16 in mma-fragment tile order (`frag16`,
row ranges of whole 16-row tiles are contiguous); the q and k rows of
Wqkv are stored so that rotary pairs are adjacent (GPT-J style rotation on
(2j, 2j+1), frequency theta^(-2j/head_dim)), which is Llama's rotate-half
RoPE up to a fixed permutation of the q/k rows; the residual stream is fp32;
KV caches are bf16 [kv_heads][capacity][head_dim] per layer.
"""

import dataclasses
import json
import math

import torch

from . import etsim
from .graphs import graph_spec  # noqa: F401  (re-exported)
from .ops import (
    EPI_BF16,
    EPI_F32,
    EPI_QKV_ROPE,
    EPI_ADD,
    EPI_RESID,
    EPI_SILU_MUL,
    GEMV_ARGMAX,
    OP_ATTN_MERGE,
    OP_ATTN_SPLIT,
    OP_EMBED,
    OP_GEMV,
    make_op,
    pack,
    ptr,
)


@dataclasses.dataclass
class DecoderConfig:
    name: str
    hidden: int
    layers: int
    heads: int
    kv_heads: int
    head_dim: int
    intermediate: int
    vocab: int
    rope_theta: float = 500000.0
    eps: float = 1e-5
    attn_chunk: int = 64      # cached positions per attention split task

    @property
    def q_rows(self):
        return self.heads * self.head_dim

    @property
    def kv_rows(self):
        return self.kv_heads * self.head_dim

    def weight_bytes(self):
        h, i = self.hidden, self.intermediate
        per_layer = 2 * (h * (self.q_rows + 2 * self.kv_rows) + self.q_rows * h + 3 * h * i + 2 * h)
        return self.layers * per_layer + 2 * self.vocab * h + 4 * h

    def kv_bytes(self, s, b=1):
        """Algorithmic KV traffic of one step: read s cached positions, write one."""
        per_pos = self.layers * 2 * self.kv_rows * 2 * b
        return per_pos * s + per_pos

    def step_bytes(self, s, b=1):
        return self.weight_bytes() + self.kv_bytes(s, b)


TINY = DecoderConfig("tiny-2L-h256", hidden=256, layers=2, heads=4, kv_heads=2, head_dim=64, intermediate=768,
                     vocab=1024, rope_theta=10000.0)
LLAMA3_8B = DecoderConfig("llama3-8b", hidden=4096, layers=32, heads=32, kv_heads=8, head_dim=128,
                          intermediate=14336, vocab=128256)
LLAMA3_70B = DecoderConfig("llama3-70b", hidden=8192, layers=80, heads=64, kv_heads=8, head_dim=128,
                           intermediate=28672, vocab=128256)
CONFIGS = {c.name: c for c in (TINY, LLAMA3_8B, LLAMA3_70B)}


def build_graph(cfg, tasks, lm_tasks, fused_merge=False, call_tasks=None, attn_cap=None):
    return etsim.Graph.from_json(json.dumps(graph_spec(cfg, tasks, lm_tasks, fused_merge, call_tasks=call_tasks,
                                                       attn_cap=attn_cap)))


def decode_graph_spec(cfg, workers, max_seq, lm_tasks=None, residual="split", fused_merge=True, balance=True,
                      grouped=True, attn_cap=None, head_split=1):
    """The decode-step graph DecodeModel lowers (reference JSON spec) and the
    layout choices it implies: per-call task counts, kv-head grouping, the
    attention split cap."""
    call_tasks = None
    if balance:  # whole-row GEMVs get a task count that divides their row tiles evenly
        call_tasks = {"qkv": balanced_tasks(cfg.q_rows + 2 * cfg.kv_rows, workers),
                      "gateup": balanced_tasks(cfg.intermediate, workers)}
        if residual == "double":  # whole-row residual GEMVs too (split-K spans are balanced already)
            call_tasks.update(oproj=balanced_tasks(cfg.hidden, workers), down=balanced_tasks(cfg.hidden, workers))
    grouped = bool(grouped and fused_merge and residual == "split" and balance and
                   call_tasks["qkv"] % cfg.kv_heads == 0)
    og = max(1, workers // cfg.kv_heads)
    while (cfg.hidden // 16) % og:
        og -= 1
    cap = attn_cap or attn_split_cap(cfg, max_seq, workers)
    head_split = head_split if grouped else 1
    spec = graph_spec(cfg, workers, lm_tasks or workers, fused_merge, call_tasks=call_tasks, attn_cap=cap,
                      grouped=grouped, oproj_group_tasks=og, head_split=head_split)
    return spec, {"call_tasks": call_tasks, "grouped": grouped, "oproj_group_tasks": og, "attn_cap": cap,
                  "head_split": head_split}


def attn_split_cap(cfg, max_seq, workers):
    """Splits per kv head: one per 64-position block up to ~one task per SM."""
    return max(1, min((max_seq + cfg.attn_chunk - 1) // cfg.attn_chunk, workers // cfg.kv_heads))


def balanced_tasks(rows, workers, tile=16):
    """Largest task count <= workers that splits rows into equal whole tiles (a stage
    ends with its slowest task: 384 tiles over 148 tasks leaves 3-tile tasks beside
    2-tile ones, over 128 tasks every task streams 3 tiles)."""
    tiles = rows // tile
    best = workers
    for t in range(workers, max(1, workers // 2) - 1, -1):
        if tiles % t == 0:
            return t
        if tiles / t <= 1:
            continue
    return best


def rope_inv_freq(cfg):
    j = torch.arange(0, cfg.head_dim // 2, dtype=torch.float64)
    return (cfg.rope_theta ** (-2.0 * j / cfg.head_dim)).to(torch.float32)


def frag16(w):
    """Device layout of a GEMV weight [N][K] (N % 16 == 0, K % 32 == 0): m16n8k16
    A-fragment tiles (see body_gemv in csrc/kernels/megakernel.cu).  Tile (t, j)
    covers rows [16t, 16t+16) and k-step j; tiles are row-tile major, so a row
    range of whole tiles is one contiguous byte range.  Inside a tile lane
    (g, q) = (lane // 4, lane % 4) holds 8 bf16: rows (g, g+8) x k = 32p + 8q + 4e
    + {0, 1, 2, 3} of the 32-wide block p = j // 2, e = j % 2, ordered
    (k-pair c, row-half h, d) -- its a0..a3 registers under the k permutation
    that makes the matching activation fragment 16 contiguous bytes."""
    N, K = w.shape
    assert N % 16 == 0 and K % 32 == 0, (N, K)
    # (t, h, g, p, q, e, c, d) -> (t, p, e, g, q, c, h, d)
    return (w.reshape(N // 16, 2, 8, K // 32, 4, 2, 2, 2).permute(0, 3, 5, 2, 4, 6, 1, 7).contiguous()
            .reshape(N, K))


GEMV_WEIGHTS = ("wqkv", "wo", "wgate", "wup", "wdown")


def group_qkv_rows(w, cfg):
    """Wqkv rows reordered per kv head: (its G q heads, its k head, its v head)."""
    dh, G, nkv = cfg.head_dim, cfg.heads // cfg.kv_heads, cfg.kv_heads
    q = w[: cfg.q_rows].reshape(nkv, G * dh, -1)
    k = w[cfg.q_rows: cfg.q_rows + cfg.kv_rows].reshape(nkv, dh, -1)
    v = w[cfg.q_rows + cfg.kv_rows:].reshape(nkv, dh, -1)
    return torch.cat([q, k, v], dim=1).reshape(w.shape[0], -1)


def group_wo(w, cfg):
    """Wo split by kv-head group along its input columns: [kv][H][G*dh], each frag16."""
    cols = (cfg.heads // cfg.kv_heads) * cfg.head_dim
    return torch.stack([frag16(w[:, g * cols:(g + 1) * cols].contiguous()) for g in range(cfg.kv_heads)])


def device_layout(W, keep_logical=False, cfg=None, grouped=False):
    """Weight dict the megakernel reads: every GEMV matrix in frag16 order (grouped:
    Wqkv rows per kv head, Wo split per kv-head group).  With keep_logical the
    row-major originals stay referenced (the CPU oracle reads them); otherwise
    they are dropped as each layer is converted."""
    D = {"embed": W["embed"], "final_norm": W["final_norm"], "lm_head": frag16(W["lm_head"]), "layers": []}
    if not keep_logical:
        W["lm_head"] = None
    for L in W["layers"]:
        d = {}
        for k, v in L.items():
            if grouped and k == "wqkv":
                d[k] = frag16(group_qkv_rows(v, cfg).contiguous())
            elif grouped and k == "wo":
                d[k] = group_wo(v, cfg)
            else:
                d[k] = frag16(v) if k in GEMV_WEIGHTS else v
        D["layers"].append(d)
        if not keep_logical:
            for k in GEMV_WEIGHTS:
                L[k] = None
    return D


def init_weights(cfg: DecoderConfig, device, seed=0, std=0.02, layer_hook=None):
    """Random-init weights of the architecture (bf16, N(0, std)); norms ~ 1 + N(0, 0.01).
    `layer_hook(d)` (optional) may replace each layer dict as soon as it is drawn
    (tensor-parallel ranks keep only their shard; the draw order is unchanged)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)

    def w(*shape):
        t = torch.empty(*shape, dtype=torch.bfloat16, device=device)
        t.normal_(0.0, std, generator=g)
        return t

    def norm():
        t = torch.empty(cfg.hidden, dtype=torch.float32, device=device)
        t.normal_(1.0, 0.01, generator=g)
        return t

    W = {"embed": w(cfg.vocab, cfg.hidden), "final_norm": norm(), "lm_head": w(cfg.vocab, cfg.hidden), "layers": []}
    if layer_hook is not None:
        W = layer_hook(W)
    for _ in range(cfg.layers):
        d = {
            "attn_norm": norm(),
            "wqkv": w(cfg.q_rows + 2 * cfg.kv_rows, cfg.hidden),
            "wo": w(cfg.hidden, cfg.q_rows),
            "ffn_norm": norm(),
            "wgate": w(cfg.intermediate, cfg.hidden),
            "wup": w(cfg.intermediate, cfg.hidden),
            "wdown": w(cfg.hidden, cfg.intermediate),
        }
        W["layers"].append(layer_hook(d) if layer_hook is not None else d)
    return W


class DecodeModel:
    """One decoder + its lowered megakernel, ready to run decode steps.

    `samples` are the sequence lengths the static program is lowered for; any
    `s` up to the largest runs on the next-larger sample without re-lowering.
    """

    def __init__(self, cfg: DecoderConfig, device="cuda:0", samples=(1024,), num_workers=None, capacity=None,
                 seed=0, weights=None, record_trace=False, prefetch=True, lm_tasks=None, keep_logical=False,
                 l2_prefetch=512 << 10, residual="split", fused_merge=True, balance=True, grouped=True,
                 scheduler="static", early_push=False, stage_barriers=False, program=None, attn_cap=None,
                 head_split=1):
        if not etsim.gpu_available():
            raise RuntimeError("DecodeModel needs a CUDA device (the executor has no CPU fallback)")
        self.cfg = cfg
        self.device = torch.device(device)
        props = torch.cuda.get_device_properties(self.device)
        self.num_workers = num_workers or props.multi_processor_count
        self.tasks = self.num_workers
        self.lm_tasks = lm_tasks or self.num_workers
        self.samples = sorted(int(s) for s in samples)
        self.capacity = capacity or (self.samples[-1] + 1)
        # attention splits per kv head (attn_cap overrides the default: one per 64-position
        # block up to about one task per SM)
        self.max_splits = attn_cap or attn_split_cap(cfg, self.samples[-1], self.num_workers)
        self.residual = residual

        import time
        t0 = time.perf_counter()
        self.fused_merge = fused_merge
        spec, self.layout = decode_graph_spec(cfg, self.tasks, self.samples[-1], lm_tasks=self.lm_tasks,
                                              residual=residual, fused_merge=fused_merge, balance=balance,
                                              grouped=grouped, attn_cap=attn_cap, head_split=head_split)
        self.call_tasks = self.layout["call_tasks"]
        self.grouped = self.layout["grouped"]
        self.oproj_group_tasks = self.layout["oproj_group_tasks"]
        if stage_barriers:  # ablation: every call waits for the whole previous call (graphs.add_stage_barriers)
            from .graphs import add_stage_barriers
            spec = add_stage_barriers(spec)
        self.graph = etsim.Graph.from_json(json.dumps(spec))
        self.scheduler = scheduler
        # program: path of an ahead-of-time program image (Executor.save_program): loaded
        # when it exists (no lowering), else written after lowering
        import os
        self.program_loaded = bool(program) and scheduler == "static" and os.path.exists(program)
        if self.program_loaded:
            self.kernel = None
        elif scheduler == "dynamic":  # on-GPU ready queues (Algorithm 2) instead of per-SM queues
            self.kernel = etsim.lower_dynamic(self.graph, early_push=early_push)
        else:
            self.kernel = etsim.lower_static(self.graph, [{"s": s} for s in self.samples], num_sms=self.num_workers)
        self.lower_ms = (time.perf_counter() - t0) * 1e3

        dev = self.device
        W = weights if weights is not None else init_weights(cfg, dev, seed)
        self.W_logical = W if keep_logical else None           # row-major bf16; the CPU oracle reads these
        self.W = device_layout(W, keep_logical=keep_logical or weights is not None, cfg=cfg,
                               grouped=self.grouped)  # what the megakernel reads
        self.kcache = [torch.zeros(cfg.kv_heads, self.capacity, cfg.head_dim, dtype=torch.bfloat16, device=dev)
                       for _ in range(cfg.layers)]
        self.vcache = [torch.zeros_like(k) for k in self.kcache]
        self.tokens = torch.zeros(1, dtype=torch.int32, device=dev)
        self.h_a = torch.zeros(1, cfg.hidden, dtype=torch.float32, device=dev)
        self.q = torch.zeros(cfg.q_rows, dtype=torch.float32, device=dev)
        self.attn = torch.zeros(cfg.q_rows, dtype=torch.bfloat16, device=dev)
        self.act = torch.zeros(cfg.intermediate, dtype=torch.bfloat16, device=dev)
        self.logits = torch.zeros(1, cfg.vocab, dtype=torch.float32, device=dev)
        # greedy decoding on the device: the lm_head tasks fold their rows into one argmax
        # word per step (zeroed by the step's embed); 8 bytes to read instead of the logits
        self.best = torch.zeros(1, dtype=torch.int64, device=dev)
        self.h_b = torch.zeros_like(self.h_a) if residual == "double" else self.h_a
        self.partials = torch.zeros(cfg.heads, self.max_splits, cfg.head_dim + 4, dtype=torch.float32, device=dev)
        self.arrive = torch.zeros(cfg.layers, cfg.kv_heads, dtype=torch.int32, device=dev)  # split arrivals (fused merge)
        self.inv_freq = rope_inv_freq(cfg).to(dev)

        t1 = time.perf_counter()
        if scheduler == "dynamic":
            self.executor = etsim.Executor(self.kernel, [{"s": s} for s in self.samples], device=self.device.index or 0,
                                           num_workers=self.num_workers, record_trace=record_trace, prefetch=prefetch)
        elif self.program_loaded:
            self.executor = etsim.Executor.load_program(program, device=self.device.index or 0,
                                                        record_trace=record_trace, prefetch=prefetch,
                                                        l2_prefetch=l2_prefetch)
        else:
            self.executor = etsim.Executor(self.kernel, device=self.device.index or 0, num_workers=self.num_workers,
                                           record_trace=record_trace, prefetch=prefetch, l2_prefetch=l2_prefetch)
            if program and scheduler == "static":
                self.executor.save_program(program)
        self.executor.bind_ops(pack(self._ops()))
        self.upload_ms = (time.perf_counter() - t1) * 1e3

    # ------------------------------------------------------------------
    def _ops(self):
        cfg, W = self.cfg, self.W
        H, dh, CH = cfg.hidden, cfg.head_dim, cfg.attn_chunk
        ops = [make_op(OP_EMBED, i=[H, -1], p=[ptr(W["embed"]), ptr(self.tokens), ptr(self.h_a), ptr(self.best)],
                       flags=1)]
        s_slot = 0
        scale = 1.0 / math.sqrt(dh)
        G = cfg.heads // cfg.kv_heads
        for l, L in enumerate(W["layers"]):
            kc, vc = self.kcache[l], self.vcache[l]
            ops.append(make_op(OP_GEMV, i=[cfg.q_rows + 2 * cfg.kv_rows, H, 1, 1, EPI_QKV_ROPE, -1, s_slot, 16, dh, H,
                                           cfg.q_rows, cfg.kv_rows, self.capacity], flags=8 if self.grouped else 0,
                               f=[cfg.eps], p=[ptr(L["wqkv"]), 0, ptr(self.h_a), ptr(L["attn_norm"]), ptr(self.q), 0,
                                               ptr(kc), ptr(vc), ptr(self.inv_freq)]))
            attn_i = [dh, G, CH, self.capacity, s_slot, self.max_splits, cfg.kv_heads]
            attn_p = [ptr(self.q), ptr(kc), ptr(vc), ptr(self.partials), ptr(self.attn), ptr(self.arrive[l])]
            if self.grouped:
                # flags bit 10: the last split folds in the new token; the output projection's
                # prologue merges each group's partials (no merge task, one hop less)
                # i13: q-head split (graphs.graph_spec head_split)
                ops.append(make_op(OP_ATTN_SPLIT, i=attn_i + [0] * 6 + [self.layout.get("head_split", 1)], f=[scale],
                                   p=attn_p, flags=1024))
            elif self.fused_merge:  # flags bit 1: the last split of a kv head merges it
                ops.append(make_op(OP_ATTN_SPLIT, i=attn_i, f=[scale], p=attn_p, flags=2))
            else:
                ops.append(make_op(OP_ATTN_SPLIT, i=attn_i, f=[scale], p=attn_p))
                ops.append(make_op(OP_ATTN_MERGE, i=attn_i, f=[scale], p=attn_p))
            if self.grouped:
                # per kv-head group: h += Wo[:, group cols] a_group (red.global.add), each
                # group's tasks released by its own merge
                # x mode 2: the activations are the merge of the group's attention partials
                ops.append(make_op(OP_GEMV, i=[H, G * dh, 1, 2, EPI_ADD, -1, s_slot, 16, dh, 0, self.max_splits, CH,
                                               self.max_splits, self.oproj_group_tasks],
                                   flags=16, p=[ptr(L["wo"]), 0, ptr(self.partials), 0, ptr(self.h_a)]))
            elif self.residual == "split":
                # row-parallel products add into the residual stream in place: split-K
                # spans (every task streams the same bytes), red.global.add epilogue
                ops.append(make_op(OP_GEMV, i=[H, cfg.q_rows, 1, 0, EPI_ADD, -1, 0, 16, 0, 0, 0, 0, 0, 1],
                                   p=[ptr(L["wo"]), 0, ptr(self.attn), 0, ptr(self.h_a)]))
            else:  # whole-row tasks, residual ping-pong h_a -> h_b -> h_a
                ops.append(make_op(OP_GEMV, i=[H, cfg.q_rows, 1, 0, EPI_RESID, -1, 0, 16],
                                   p=[ptr(L["wo"]), 0, ptr(self.attn), 0, ptr(self.h_b), ptr(self.h_a)]))
            ops.append(make_op(OP_GEMV, i=[cfg.intermediate, H, 2, 1, EPI_SILU_MUL, -1, 0, 16, 0, H],
                               f=[cfg.eps], p=[ptr(L["wgate"]), ptr(L["wup"]), ptr(self.h_b), ptr(L["ffn_norm"]),
                                               ptr(self.act)]))
            if self.residual == "split":
                ops.append(make_op(OP_GEMV, i=[H, cfg.intermediate, 1, 0, EPI_ADD, -1, 0, 16, 0, 0, 0, 0, 0, 1],
                                   p=[ptr(L["wdown"]), 0, ptr(self.act), 0, ptr(self.h_a)]))
            else:
                ops.append(make_op(OP_GEMV, i=[H, cfg.intermediate, 1, 0, EPI_RESID, -1, 0, 16],
                                   p=[ptr(L["wdown"]), 0, ptr(self.act), 0, ptr(self.h_a), ptr(self.h_b)]))
        ops.append(make_op(OP_GEMV, i=[cfg.vocab, H, 1, 1, EPI_F32, -1, 0, 16, 0, H], f=[cfg.eps], flags=GEMV_ARGMAX,
                           p=[ptr(W["lm_head"]), 0, ptr(self.h_a), ptr(W["final_norm"]), ptr(self.logits), 0,
                              ptr(self.best)]))
        return ops

    def greedy_token(self):
        """The last step's greedy token, computed on the device (reads 8 bytes)."""
        from .ops import argmax_token
        return argmax_token(self.best.item())

    def fill_cache(self, s, seed=1):
        """Synthetic prefilled KV cache: N(0, 1) bf16 for positions [0, s)."""
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        for k, v in zip(self.kcache, self.vcache):
            k.zero_()
            v.zero_()
            k[:, :s].normal_(0.0, 1.0, generator=g)
            v[:, :s].normal_(0.0, 1.0, generator=g)

    def set_token(self, token):
        self.tokens.fill_(int(token))

    def step(self, s):
        """One synchronous decode step at position s; returns device logits [1, vocab]."""
        stats = self.executor.run({"s": int(s)})
        self.last_stats = stats
        return self.logits

    def launch(self, s, stream=0):
        self.executor.launch({"s": int(s)}, stream)

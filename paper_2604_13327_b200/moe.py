"""Qwen3-MoE-style decode on the Event Tensor megakernel, with routing resolved
on the GPU.

The reference models an MoE layer as the graph route(1) -> group(tokens*top_k)
-> expert_mm (ref workloads.cpp:81-114):

- `group` notifies EXP[topk[f]] through a data-dependent notify;
- `expert_mm` is range-triggered on `exp_indptr` and sizes itself with
  `extent_from`.

The routing is a seeded RNG (`moe_realization`, ref workloads.cpp:116-150).
Here the same structure runs inside each decoder layer of one decode step:

    qkv[T] -> attn[kv, ceil(s/CH)] -> merge[kv] -> oproj[T] -> route[E/16]
      -> group[b*K]      (routed notify EXP_l[topk_l[f]]; EXP_l has data-dependent
                          counts = cnt_l, written by route_l)
      -> expert[b*K*RS]  (range trigger on tind_l = exp_indptr_l * RS, extent_from tind_l)
      -> next layer's qkv

The route tasks run the router GEMV. The last task to arrive computes on the
device:

- softmax and top-k;
- expert counts, `exp_indptr` (tiles of TS tokens, the reference's routing
  algebra);
- `task_indptr`, the per-expert slot lists and the weights.

These become the runtime tensors the Event Tensors read. No host round trip,
recompile or relaunch is involved. Routing can also be injected from the host
(`inject_routing`): route then skips its top-k, as in the reference's
realization.

Each expert task (tile, r) computes SiLU(gate)*up for rows [r*IR, r*IR+IR) of
its expert on the tile's tokens. It then adds the matching column block of the
down projection, times the routing weight, into the fp32 residual stream with
red.global.add, so no combine stage exists. Attention uses Qwen3's per-head
q/k RMSNorm before RoPE, applied inside the attention tasks (ATTN flags bit 0).
"""

import dataclasses
import json
import math
import time

import torch

from . import etsim
from .decode import frag16, rope_inv_freq
from .ops import (
    EPI_ADD,
    EPI_F32,
    GEMV_ARGMAX,
    OP_ATTN_MERGE,
    OP_ATTN_SPLIT,
    OP_EMBED,
    OP_GEMV,
    OP_MOE_EXPERT,
    OP_MOE_ROUTE,
    OP_NONE,
    make_op,
    pack,
    ptr,
)


@dataclasses.dataclass
class MoEConfig:
    name: str
    hidden: int
    layers: int
    heads: int
    kv_heads: int
    head_dim: int
    experts: int
    top_k: int
    expert_inter: int
    vocab: int
    rope_theta: float = 1000000.0
    eps: float = 1e-6
    attn_chunk: int = 64
    row_splits: int = 12       # expert row splits (expert_inter / row_splits % 32 == 0)
    tile_tokens: int = 8       # tokens per expert tile (<= 8: the mma N dimension)
    # Router init scale.  0.02 like every projection: round 1 drew the router from
    # N(0, 0.1), whose logits (std ~4.5) make the renormalised top-k softmax so sharp
    # that a bf16-ulp difference in the hidden state grows ~12% per layer (measured:
    # 0.4% after layer 0, 66% after layer 47, profiles/r2_diag_moe_depth.txt) -- a
    # property of that synthetic function, not of any implementation, which made a
    # 48-layer logits comparison meaningless.
    router_std: float = 0.02

    @property
    def q_rows(self):
        return self.heads * self.head_dim

    @property
    def kv_rows(self):
        return self.kv_heads * self.head_dim

    def dense_bytes(self):
        h = self.hidden
        per_layer = 2 * (h * (self.q_rows + 2 * self.kv_rows) + self.q_rows * h + self.experts * h + 2 * h
                         + 2 * self.head_dim)
        return self.layers * per_layer + 2 * self.vocab * h + 4 * h

    def expert_bytes(self):
        return 3 * self.expert_inter * self.hidden * 2

    def step_bytes(self, s, active_experts_per_layer, b=1):
        """Algorithmic bytes: dense weights + touched experts (from the device counts) + KV."""
        kv = self.layers * 2 * self.kv_rows * 2 * b * (s + 1)
        return self.dense_bytes() + sum(active_experts_per_layer) * self.expert_bytes() + kv


TINY_MOE = MoEConfig("tiny-moe-2L", hidden=256, layers=2, heads=4, kv_heads=2, head_dim=64, experts=16, top_k=4,
                     expert_inter=64, vocab=1024, row_splits=2, rope_theta=10000.0)
QWEN3_30B_A3B = MoEConfig("qwen3-30b-a3b", hidden=2048, layers=48, heads=32, kv_heads=4, head_dim=128, experts=128,
                          top_k=8, expert_inter=768, vocab=151936, row_splits=12)
MOE_CONFIGS = {c.name: c for c in (TINY_MOE, QWEN3_30B_A3B)}

RT_PER_LAYER = ("topk", "cnt", "ind", "tind", "elist", "eoff")


def moe_graph_spec(cfg, tasks, lm_tasks, tokens=1, fused_merge=False, qkv_tasks=None, route_tasks=1,
                   group_stage=True, attn_cap=None, oproj_group_tasks=None, tc=None, head_split=1):
    """Reference-format graph spec (ref json_io.cpp:115-230) of one MoE decode step.

    tokens: an int (fixed batch) or "b" -- the batch is then a graph symbol next
    to `s`, and the attention, group and expert grids scale with it at run time
    (one lowered artifact serves every batch up to the largest sample).
    oproj_group_tasks: the output projection runs per kv-head group (grid [kv, n]),
    each group released by its own attention merge (needed for batch > 4: the
    full attention row would not fit the staged activations).
    tc: task counts of the tensor-core projections (batches above 8): every
    RMSNorm becomes its own [b] call feeding the tensor-core operand layout, and
    the router logits come from a tensor-core GEMV call before the route task."""
    CH = cfg.attn_chunk
    E, K, RS = cfg.experts, cfg.top_k, cfg.row_splits
    fns, events, calls, rts = [], [], [], []

    def fn(name, grid):
        fns.append({"name": name, "grid": grid, "resource": "sm", "duration": "unit"})
        return name

    def ev(name, shape, **kw):
        events.append(dict({"name": name, "shape": shape}, **kw))
        return name

    T, kv = str(tasks), str(cfg.kv_heads)
    ev("EMB", ["1"])
    calls.append({"fn": fn("embed", ["1"]), "out": [{"event": "EMB", "map": ["0"]}]})
    prev = "EMB"
    for l in range(cfg.layers):
        rt = {n: f"{n}{l}" for n in RT_PER_LAYER}
        route = f"L{l}.route"
        rts += [{"name": rt["topk"], "shape": [str(tokens), str(K)], "role": "routing", "writer": route},
                {"name": rt["cnt"], "shape": [str(E)], "role": "counts", "writer": route},
                {"name": rt["ind"], "shape": [str(E + 1)], "role": "indptr", "writer": route},
                {"name": rt["tind"], "shape": [str(E + 1)], "role": "indptr", "writer": route},
                {"name": rt["elist"], "shape": [f"{tokens} * {K}"], "role": "routing", "writer": route},
                {"name": rt["eoff"], "shape": [str(E + 1)], "role": "indptr", "writer": route}]
        qkv, a, m, o, r, x, d = (f"{n}{l}" for n in ("QKV", "A", "M", "O", "R", "EXP", "D"))
        ev(qkv, ["1"])
        if not fused_merge:
            ev(a, [kv])
        ev(m, [kv] if oproj_group_tasks else ["1"])
        ev(o, ["1"])
        ev(r, ["1"])
        if group_stage:
            ev(x, [str(E)], data_dependent=True, counts=rt["cnt"], writer=route)
        ev(d, ["1"])
        nsplit = f"(s + {CH - 1}) // {CH}" if not attn_cap else f"min((s + {CH - 1}) // {CH}, {attn_cap})"
        if tc:  # RMSNorm of the stream into the tensor-core operand layout, one task per token
            n1 = ev(f"N1{l}", ["1"])
            calls.append({"fn": fn(f"L{l}.norm1", [str(tokens)]), "in": [{"event": prev, "map": ["0"]}],
                          "out": [{"event": n1, "map": ["0"]}]})
            prev = n1
        calls.append({"fn": fn(f"L{l}.qkv", [str(tc["qkv"] if tc else qkv_tasks or tasks)]),
                      "in": [{"event": prev, "map": ["0"]}], "out": [{"event": qkv, "map": ["0"]}]})
        if tc:  # flat grid, split count shrinking with the batch (batch.attn_grid)
            from .batch import attn_grid

            calls.append({"fn": fn(f"L{l}.attn", [attn_grid(cfg, attn_cap, tc["attn_budget"])]),
                          "in": [{"event": qkv, "map": ["0"]}], "out": [{"event": m, "map": ["0"]}]})
        elif fused_merge and head_split > 1:  # q heads of a group shared by head_split tasks per split
            calls.append({"fn": fn(f"L{l}.attn", [f"{tokens} * {kv} * {head_split}", f"max({nsplit}, 1)"]),
                          "in": [{"event": qkv, "map": ["0"]}],
                          "out": [{"event": m, "map": [f"(t0 // {head_split}) % {kv}"]}]})
        elif fused_merge:  # the last split of each (sequence, kv head) merges the group
            calls.append({"fn": fn(f"L{l}.attn", [f"{tokens} * {kv}", f"max({nsplit}, 1)"]),
                          "in": [{"event": qkv, "map": ["0"]}],
                          "out": [{"event": m, "map": [f"t0 % {kv}" if oproj_group_tasks else "0"]}]})
        else:
            calls += [
                {"fn": fn(f"L{l}.attn", [kv, nsplit]), "in": [{"event": qkv, "map": ["0"]}],
                 "out": [{"event": a, "map": ["t0"]}]},
                {"fn": fn(f"L{l}.merge", [kv]), "in": [{"event": a, "map": ["t0"]}, {"event": qkv, "map": ["0"]}],
                 "out": [{"event": m, "map": ["0"]}]}]
        if oproj_group_tasks:
            calls.append({"fn": fn(f"L{l}.oproj", [kv, str(oproj_group_tasks)]), "in": [{"event": m, "map": ["t0"]}],
                          "out": [{"event": o, "map": ["0"]}]})
        else:
            calls.append({"fn": fn(f"L{l}.oproj", [str(tc["oproj"]) if tc else T]), "in": [{"event": m, "map": ["0"]}],
                          "out": [{"event": o, "map": ["0"]}]})
        rin = o
        if tc:  # norm2 -> router logits (tensor cores) -> route (top-k, counts, indptr)
            n2, rl = ev(f"N2{l}", ["1"]), ev(f"RL{l}", ["1"])
            calls += [{"fn": fn(f"L{l}.norm2", [str(tokens)]), "in": [{"event": o, "map": ["0"]}],
                       "out": [{"event": n2, "map": ["0"]}]},
                      {"fn": fn(f"L{l}.router", [str(tc["router"])]), "in": [{"event": n2, "map": ["0"]}],
                       "out": [{"event": rl, "map": ["0"]}]}]
            rin = rl
        calls += [
            {"fn": fn(route, [str(1 if tc else route_tasks)]), "in": [{"event": rin, "map": ["0"]}],
             "out": [{"event": r, "map": ["0"]}]}]
        if group_stage:  # the reference structure: routed notify + range trigger (dynamic scheduler)
            calls += [
                {"fn": fn(f"L{l}.group", [f"{tokens} * {K}"]), "in": [{"event": r, "map": ["0"]}],
                 "out": [{"event": x, "routed_by": rt["topk"]}]},
                {"fn": fn(f"L{l}.expert", [f"{tokens} * {K * RS}"]), "extent_from": rt["tind"],
                 "in": [{"event": x, "indptr": rt["tind"]}], "out": [{"event": d, "map": ["0"]}]}]
        else:  # static scheduler: the worst-case rewrite makes EXP a barrier over the no-op
            # group tasks anyway; the expert tiles wait on the routing itself (extent_from masks)
            calls.append({"fn": fn(f"L{l}.expert", [f"{tokens} * {K * RS}"]), "extent_from": rt["tind"],
                          "in": [{"event": r, "map": ["0"]}], "out": [{"event": d, "map": ["0"]}]})
        prev = d
    if tc:
        ev("NF", ["1"])
        calls.append({"fn": fn("normf", [str(tokens)]), "in": [{"event": prev, "map": ["0"]}],
                      "out": [{"event": "NF", "map": ["0"]}]})
        prev = "NF"
    ev("LM", ["1"])
    calls.append({"fn": fn("lm_head", [str(tc["lm"] if tc else lm_tasks)]), "in": [{"event": prev, "map": ["0"]}],
                  "out": [{"event": "LM", "map": ["0"]}]})
    symbols = ["s", "b"] if tokens == "b" else ["s"]
    return {"symbols": symbols, "size_symbol": "s", "duration_models": {"unit": {"kind": "constant", "value": 1}},
            "device_functions": fns, "event_tensors": events, "runtime_tensors": rts, "calls": calls}


def init_moe_weights(cfg: MoEConfig, device, seed=0, std=0.02, layer_hook=None):
    """Random-init weights (bf16 N(0, std), router N(0, cfg.router_std), norms ~ 1 + N(0, 0.01)).
    `layer_hook(d)` (optional) may replace the top-level dict and each layer dict as
    soon as it is drawn (the draw order is unchanged)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)

    def w(*shape, s=std):
        t = torch.empty(*shape, dtype=torch.bfloat16, device=device)
        t.normal_(0.0, s, generator=g)
        return t

    def norm(n):
        t = torch.empty(n, dtype=torch.float32, device=device)
        t.normal_(1.0, 0.01, generator=g)
        return t

    H, I, E = cfg.hidden, cfg.expert_inter, cfg.experts
    W = {"embed": w(cfg.vocab, H), "final_norm": norm(H), "lm_head": w(cfg.vocab, H), "layers": []}
    if layer_hook is not None:
        W = layer_hook(W)
    for _ in range(cfg.layers):
        d = {
            "attn_norm": norm(H), "wqkv": w(cfg.q_rows + 2 * cfg.kv_rows, H), "q_norm": norm(cfg.head_dim),
            "k_norm": norm(cfg.head_dim), "wo": w(H, cfg.q_rows), "ffn_norm": norm(H),
            "router": w(E, H, s=cfg.router_std),
            "wgate": w(E, I, H), "wup": w(E, I, H), "wdown": w(E, H, I),
        }
        W["layers"].append(layer_hook(d) if layer_hook is not None else d)
    return W


def moe_device_layout(cfg, W, kp=0):
    """frag16 tiles for every GEMV matrix; expert down projections cut into RS
    column blocks [E][RS][H][IR], each its own frag16 matrix.  kp > 0 (batches
    above 8): the dense projections in the tensor-core layout instead (batch.tc_pack;
    router rows padded to a 128-row block)."""
    E, H, I, RS = cfg.experts, cfg.hidden, cfg.expert_inter, cfg.row_splits
    IR = I // RS
    if kp:
        from .batch import tc_pack

        def pad128(w):
            n = -(-w.shape[0] // 128) * 128
            return w if n == w.shape[0] else torch.cat([w, w.new_zeros(n - w.shape[0], w.shape[1])])
    D = {"embed": W["embed"], "final_norm": W["final_norm"],
         "lm_head": tc_pack(W["lm_head"], kp) if kp else frag16(W["lm_head"]), "layers": []}
    for L in W["layers"]:
        d = dict(L)
        for k in ("wqkv", "wo", "router"):
            d[k] = tc_pack(pad128(L[k]), kp) if kp else frag16(L[k])
        d["wgate"] = torch.stack([frag16(L["wgate"][e]) for e in range(E)])
        d["wup"] = torch.stack([frag16(L["wup"][e]) for e in range(E)])
        blocks = L["wdown"].reshape(E, H, RS, IR).permute(0, 2, 1, 3)  # [E][RS][H][IR]
        d["wdown"] = torch.stack([torch.stack([frag16(blocks[e, r].contiguous()) for r in range(RS)])
                                  for e in range(E)])
        if not kp:
            cols = (cfg.heads // cfg.kv_heads) * cfg.head_dim  # Wo per kv-head group (batched decode)
            d["wo_grouped"] = torch.stack([frag16(L["wo"][:, g * cols:(g + 1) * cols].contiguous())
                                           for g in range(cfg.kv_heads)])
        D["layers"].append(d)
    return D


def moe_layout(cfg, num_workers, samples, scheduler, max_batch=1, batch_samples=None, attn_cap=None,
               fused_merge=True, balance=False, route_tasks=None, group_stage=None, qkv_split=True,
               oproj_merge=True, head_split=None):
    """Every layout choice MoEDecodeModel makes before touching the device: the graph
    spec it lowers, its bindings (samples) and task counts.  Pure (no device, no
    extension), so the committed bench-graph fixtures (tests/golden/make_bench_graphs.py)
    are exactly the graphs the model runs.

    batch: a graph symbol `b`; every (s, b) at or below a sample runs on the lowered
    artifact.  Up to 8 the projections carry the batch in the mma.sync N dimension;
    above, they run on the tcgen05 tensor cores (batch.py layouts)."""
    from .decode import attn_split_cap, balanced_tasks

    assert cfg.expert_inter % cfg.row_splits == 0 and (cfg.expert_inter // cfg.row_splits) % 32 == 0
    # the expert body's accumulators (gate / up for 8 tokens + activations) fit 2048 floats
    assert cfg.expert_inter // cfg.row_splits <= 96, "expert row split wider than 96 rows"
    assert 1 <= max_batch <= 64
    L = {"max_batch": max_batch, "batched": max_batch > 1, "tc": max_batch > 8}
    L["tokens"] = "b" if L["batched"] else 1
    default = [1 << i for i in range(7) if (1 << i) < max_batch] if L["tc"] else [1]
    L["batch_samples"] = sorted(set(batch_samples or default) | {max_batch}) if L["batched"] else [1]
    L["samples"] = sorted(int(s) for s in samples)
    L["capacity"] = L["samples"][-1] + 1
    ms = attn_cap or attn_split_cap(cfg, L["samples"][-1], num_workers)
    if not attn_cap and max_batch == 1 and oproj_merge and fused_merge:
        # the output projection stages each group's partials in shared memory with bulk
        # copies (G * splits * (dh + 4) * 4 bytes <= ~35 KB): at most 8 splits of 8 heads
        ms = min(ms, max(1, (35 * 1024) // ((cfg.heads // cfg.kv_heads) * (cfg.head_dim + 4) * 4)))
    if max_batch > 8 and not attn_cap:  # tensor-core attention: a split runs two blocks at a time (batch.py)
        ms = max(1, ms // 2)
    L["max_splits"] = ms
    L["fused_merge"] = fused_merge
    # q-head split of the scalar attention (one sequence, output projection merge only): by
    # default 4 tasks per (kv head, split) for groups of >= 8 q heads (Qwen3-30B-A3B bs=1:
    # 3.80 -> 3.57 ms static, 5.37 -> 5.21 ms dynamic; 2: 3.59 ms, 8: 4.09 ms)
    G = cfg.heads // cfg.kv_heads
    if head_split is None:
        head_split = 4 if G >= 8 else 1
    L["head_split"] = head_split if (max_batch == 1 and oproj_merge and fused_merge) else 1
    assert (cfg.heads // cfg.kv_heads) % L["head_split"] == 0
    L["group_stage"] = (scheduler == "dynamic") if group_stage is None else group_stage
    L["qkv_split"] = qkv_split and fused_merge
    L["route_tasks"] = route_tasks or max(1, cfg.experts // 16)
    assert fused_merge or not L["batched"], "batched decode uses the fused attention merge"
    og = None
    # one sequence: the attention splits leave partials and the per-group output
    # projection merges them in its prologue (no merge task; GEMV x mode 2)
    L["oproj_merge"] = bool(oproj_merge and not L["batched"] and fused_merge)
    if L["batched"] or L["oproj_merge"]:  # per kv-head-group output projection (a batch of full attention rows would not fit)
        og = max(1, num_workers // cfg.kv_heads)
        while (cfg.hidden // 16) % og:
            og -= 1
    # the lm_head task's rows x batch accumulate in shared memory (2048 fp32): a large
    # vocabulary at batch 8 needs more, smaller row spans than one per worker
    tiles, cap_tiles = cfg.vocab // 16, max(1, 2048 // (16 * max_batch))
    L["lm_tasks"] = max(num_workers, -(-tiles // cap_tiles))
    kp, tct, tcs = 0, None, None
    if L["tc"]:
        from .batch import attn_budget, tc_npad, tc_piece_for, tc_tasks

        assert fused_merge
        og = None
        H, nq = cfg.hidden, cfg.q_rows
        kp = tc_piece_for(max_batch, (H, nq))
        npad = tc_npad(max_batch)
        tct, tcs = {}, {}
        for name, n, k, add in (("qkv", nq + 2 * cfg.kv_rows, H, True), ("oproj", H, nq, True),
                                ("router", -(-cfg.experts // 128) * 128, H, True), ("lm", cfg.vocab, H, False)):
            tct[name], tcs[name] = tc_tasks(n // 128, num_workers, add, 1, npad, k // kp)
        tct["attn_budget"] = attn_budget(cfg, num_workers)
    L.update(oproj_group_tasks=og, kp=kp, tc_tasks=tct, tc_splits=tcs)
    L["spec"] = moe_graph_spec(cfg, num_workers, L["lm_tasks"], L["tokens"], fused_merge=fused_merge,
                               qkv_tasks=balanced_tasks(cfg.q_rows + 2 * cfg.kv_rows, num_workers)
                               if balance else None, route_tasks=L["route_tasks"], group_stage=L["group_stage"],
                               attn_cap=ms, oproj_group_tasks=og, tc=tct, head_split=L["head_split"])
    L["bindings"] = [({"s": int(s), "b": int(b)} if L["batched"] else {"s": int(s)})
                     for s in L["samples"] for b in L["batch_samples"]]
    return L


class MoEDecodeModel:
    """One MoE decoder + its lowered megakernel (static or dynamic scheduler)."""

    def __init__(self, cfg: MoEConfig, device="cuda:0", samples=(1024,), num_workers=None, seed=0, weights=None,
                 scheduler="dynamic", record_trace=False, keep_logical=False, early_push=False, fused_merge=True,
                 balance=False, route_tasks=None, group_stage=None, l2_prefetch_experts=False, qkv_split=True,
                 max_batch=1, batch_samples=None, attn_cap=None, oproj_merge=True, stage_barriers=False,
                 head_split=None):
        if not etsim.gpu_available():
            raise RuntimeError("MoEDecodeModel needs a CUDA device (the executor has no CPU fallback)")
        self.cfg = cfg
        self.device = torch.device(device)
        props = torch.cuda.get_device_properties(self.device)
        self.num_workers = num_workers or props.multi_processor_count
        self.scheduler = scheduler
        self.l2_prefetch_experts = l2_prefetch_experts
        t0 = time.perf_counter()
        lay = moe_layout(cfg, self.num_workers, samples, scheduler, max_batch=max_batch, batch_samples=batch_samples,
                         attn_cap=attn_cap, fused_merge=fused_merge, balance=balance, route_tasks=route_tasks,
                         group_stage=group_stage, qkv_split=qkv_split, oproj_merge=oproj_merge,
                         head_split=head_split)
        for k, v in lay.items():
            setattr(self, k, v)
        if stage_barriers:  # ablation: every call waits for the whole previous call (graphs.add_stage_barriers)
            from .graphs import add_stage_barriers
            self.spec = add_stage_barriers(self.spec)
        self.graph = etsim.Graph.from_json(json.dumps(self.spec))
        self.rt_index = {r["name"]: i for i, r in enumerate(self.spec["runtime_tensors"])}
        if scheduler == "dynamic":
            self.kernel = etsim.lower_dynamic(self.graph, early_push=early_push)
        else:
            # static: data-dependent events collapse to worst-case barriers (ref
            # sched_static.cpp:13-47); extent_from still masks dead expert tiles on device
            self.kernel = etsim.lower_static(etsim.worst_case_rewrite(self.graph), self.bindings,
                                             num_sms=self.num_workers)
        self.lower_ms = (time.perf_counter() - t0) * 1e3

        dev = self.device
        W = weights if weights is not None else init_moe_weights(cfg, dev, seed)
        self.W_logical = W if keep_logical else None
        self.W = moe_device_layout(cfg, W, self.kp)
        b, E, K = self.max_batch, cfg.experts, cfg.top_k
        # per-sequence KV caches [b][kv][cap][dh]
        self.kcache = [torch.zeros(b, cfg.kv_heads, self.capacity, cfg.head_dim, dtype=torch.bfloat16, device=dev)
                       for _ in range(cfg.layers)]
        self.vcache = [torch.zeros_like(k) for k in self.kcache]
        self.tok = torch.zeros(b, dtype=torch.int32, device=dev)
        self.h = torch.zeros(b, cfg.hidden, dtype=torch.float32, device=dev)
        self.qkv = torch.zeros(b, cfg.q_rows + 2 * cfg.kv_rows, dtype=torch.float32, device=dev)
        self.attn = torch.zeros(b, cfg.q_rows, dtype=torch.bfloat16, device=dev)
        self.partials = torch.zeros(b * cfg.heads, max(8, self.max_splits) if self.tc else self.max_splits,
                                    cfg.head_dim + 4, dtype=torch.float32, device=dev)
        self.logits_r = torch.zeros(cfg.layers, b, E, dtype=torch.float32, device=dev)   # router logits per layer
        self.xn = torch.zeros(cfg.layers, b, cfg.hidden, dtype=torch.bfloat16, device=dev)
        self.wslot = torch.zeros(cfg.layers, b * K, dtype=torch.float32, device=dev)
        self.arrive = torch.zeros(cfg.layers, dtype=torch.int32, device=dev)
        self.arrive_attn = torch.zeros(cfg.layers, b * cfg.kv_heads, dtype=torch.int32, device=dev)
        self.tiles = torch.zeros(cfg.layers, b * K, 4, dtype=torch.int32, device=dev)  # expert tile table
        self.logits = torch.zeros(b, cfg.vocab, dtype=torch.float32, device=dev)
        if self.tc:  # operand-layout activations and the router accumulators (zeroed by the route task)
            from .batch import tc_npad

            npad = tc_npad(b)
            self.xn_tc = torch.zeros(npad * cfg.hidden, dtype=torch.bfloat16, device=dev)
            self.attn_tc = torch.zeros(npad * cfg.q_rows, dtype=torch.bfloat16, device=dev)
            self.logits_acc = torch.zeros(b, E, dtype=torch.float32, device=dev)
        self.inv_freq = rope_inv_freq(cfg).to(dev)
        self.injected = False
        self.best = torch.zeros(1, dtype=torch.int64, device=dev)  # greedy argmax word (one sequence)

        t1 = time.perf_counter()
        if scheduler == "dynamic":
            self.executor = etsim.Executor(self.kernel, self.bindings, device=dev.index or 0,
                                           num_workers=self.num_workers, record_trace=record_trace,
                                           max_batch=self.max_batch)
        else:
            self.executor = etsim.Executor(self.kernel, device=dev.index or 0, num_workers=self.num_workers,
                                           record_trace=record_trace, max_batch=self.max_batch)
        self.bind()
        self.upload_ms = (time.perf_counter() - t1) * 1e3

    def bind(self):
        self.executor.bind_ops(pack(self._ops()))

    def _ops_tc(self):
        """Op table of the tensor-core variant (batches above 8)."""
        from .ops import OP_GEMV_TC, OP_NORM

        cfg, W, kp = self.cfg, self.W, self.kp
        H, dh, CH, nq = cfg.hidden, cfg.head_dim, cfg.attn_chunk, cfg.q_rows
        E, K, RS, TS = cfg.experts, cfg.top_k, cfg.row_splits, cfg.tile_tokens
        G = cfg.heads // cfg.kv_heads
        rows = nq + 2 * cfg.kv_rows
        bs, sp = 1, self.tc_splits

        def tc(n, k, epi, w, x, out, splits, ostride=0):
            return make_op(OP_GEMV_TC, i=[n, k, 1, splits, epi, bs, kp, 0, ostride],
                           p=[ptr(w), 0, ptr(x), 0, ptr(out)])

        def norm(gamma, rowmajor=None):
            return make_op(OP_NORM, i=[H, 0, 0, 0, 0, bs, kp], f=[cfg.eps],
                           p=[ptr(self.h), ptr(gamma), ptr(self.xn_tc), ptr(rowmajor)])

        ops = [make_op(OP_EMBED, i=[H, bs], p=[ptr(W["embed"]), ptr(self.tok), ptr(self.h)])]
        for l, L in enumerate(W["layers"]):
            ri = {n: self.rt_index[f"{n}{l}"] for n in RT_PER_LAYER}
            ops.append(norm(L["attn_norm"]))
            ops.append(tc(rows, H, EPI_ADD, L["wqkv"], self.xn_tc, self.qkv, sp["qkv"]))
            # flags: 1 q/k-norm mode, 2 fused merge, 32 zero the raw q/k/v after use, 128 flat grid,
            # 256 chunk-swizzled cache rows (batch.cache_swizzle); out in operand layout
            ops.append(make_op(OP_ATTN_SPLIT,
                               i=[dh, G, CH, self.capacity, 0, self.max_splits, cfg.kv_heads, rows,
                                  cfg.kv_heads * self.capacity * dh, kp, bs, self.tc_tasks["attn_budget"]],
                               f=[1.0 / math.sqrt(dh), cfg.eps], flags=1 | 2 | 32 | 128 | 256 | 512,
                               p=[ptr(self.qkv), ptr(self.kcache[l]), ptr(self.vcache[l]), ptr(self.partials),
                                  ptr(self.attn_tc), ptr(self.arrive_attn[l]), ptr(L["k_norm"]), ptr(self.inv_freq),
                                  ptr(self.qkv) + 4 * nq, ptr(L["q_norm"])]))
            ops.append(tc(H, nq, EPI_ADD, L["wo"], self.attn_tc, self.h, sp["oproj"]))
            ops.append(norm(L["ffn_norm"], self.xn[l]))
            ops.append(tc(-(-E // 128) * 128, H, EPI_ADD, L["router"], self.xn_tc, self.logits_acc, sp["router"],
                          ostride=E))
            assert [ri[n] for n in RT_PER_LAYER] == list(range(ri["topk"], ri["topk"] + len(RT_PER_LAYER)))
            ops.append(make_op(OP_MOE_ROUTE, i=[E, H, 1, 1, EPI_F32, bs, K, 16, cfg.expert_inter, H, ri["topk"], 0, RS,
                                                TS],
                               f=[cfg.eps],
                               p=[0, ptr(self.logits_acc), ptr(self.h), 0, ptr(self.logits_r[l]), ptr(self.xn[l]),
                                  ptr(self.wslot[l]), ptr(self.arrive[l:l + 1]), ptr(self.tiles[l])],
                               flags=2 | (1 if self.injected else 0)))
            if self.group_stage:
                ops.append(make_op(OP_NONE))
            ops.append(make_op(OP_MOE_EXPERT,
                               i=[cfg.expert_inter, H, RS, TS, ri["ind"], ri["cnt"], ri["elist"], ri["eoff"], K, 0, E],
                               p=[ptr(L["wgate"]), ptr(L["wup"]), ptr(L["wdown"]), ptr(self.xn[l]), ptr(self.wslot[l]),
                                  ptr(self.h), ptr(self.tiles[l])]))
        ops.append(norm(W["final_norm"]))
        ops.append(tc(cfg.vocab, H, EPI_F32, W["lm_head"], self.xn_tc, self.logits, 1))
        return ops

    def _ops(self):
        if self.tc:
            return self._ops_tc()
        cfg, W = self.cfg, self.W
        H, dh, CH = cfg.hidden, cfg.head_dim, cfg.attn_chunk
        E, K, RS, TS = cfg.experts, cfg.top_k, cfg.row_splits, cfg.tile_tokens
        G = cfg.heads // cfg.kv_heads
        scale = 1.0 / math.sqrt(dh)
        nq = cfg.q_rows
        bs = 1 if self.batched else -1  # binding slot of the batch symbol (-1: one sequence)
        greedy = not self.batched  # one sequence: the greedy token is decided on the device
        ops = [make_op(OP_EMBED, i=[H, bs], p=[ptr(W["embed"]), ptr(self.tok), ptr(self.h), ptr(self.best)],
                       flags=1 if greedy else 0)]
        for l, L in enumerate(W["layers"]):
            ri = {n: self.rt_index[f"{n}{l}"] for n in RT_PER_LAYER}
            kc, vc = self.kcache[l], self.vcache[l]
            if self.qkv_split:  # split-K spans, red.add into the raw q/k/v accumulators (the merger zeroes them)
                ops.append(make_op(OP_GEMV, i=[nq + 2 * cfg.kv_rows, H, 1, 1, EPI_ADD, bs, 0, 16, 0, H, 0, 0, 0, 1],
                                   f=[cfg.eps], p=[ptr(L["wqkv"]), 0, ptr(self.h), ptr(L["attn_norm"]), ptr(self.qkv)]))
            else:
                ops.append(make_op(OP_GEMV, i=[nq + 2 * cfg.kv_rows, H, 1, 1, EPI_F32, bs, 0, 16, 0, H], f=[cfg.eps],
                                   p=[ptr(L["wqkv"]), 0, ptr(self.h), ptr(L["attn_norm"]), ptr(self.qkv)]))
            attn_i = [dh, G, CH, self.capacity, 0, self.max_splits, cfg.kv_heads, nq + 2 * cfg.kv_rows,
                      cfg.kv_heads * self.capacity * dh]
            attn_p = [ptr(self.qkv), ptr(kc), ptr(vc), ptr(self.partials), ptr(self.attn), ptr(L["q_norm"]),
                      ptr(L["k_norm"]), ptr(self.inv_freq), ptr(self.qkv) + 4 * nq]
            if self.oproj_merge:  # flags: 1 = q/k-norm mode, 1024 = the last split folds the new token
                ops.append(make_op(OP_ATTN_SPLIT, i=attn_i + [0] * 4 + [self.head_split], f=[scale, cfg.eps],
                                   flags=1 | 1024, p=attn_p))
            elif self.fused_merge:  # flags: 1 = q/k-norm mode, 2 = the last split merges; p5 of the split
                # op carries the arrival counters, so the norm weights move to the merge-compatible slots
                ops.append(make_op(OP_ATTN_SPLIT, i=attn_i, f=[scale, cfg.eps], flags=3 | (32 if self.qkv_split else 0),
                                   p=[ptr(self.qkv), ptr(kc), ptr(vc), ptr(self.partials), ptr(self.attn),
                                      ptr(self.arrive_attn[l]), ptr(L["k_norm"]), ptr(self.inv_freq),
                                      ptr(self.qkv) + 4 * nq, ptr(L["q_norm"])]))
            else:
                ops.append(make_op(OP_ATTN_SPLIT, i=attn_i, f=[scale, cfg.eps], p=attn_p, flags=1))
                ops.append(make_op(OP_ATTN_MERGE, i=attn_i, f=[scale, cfg.eps], p=attn_p, flags=1))
            if self.oproj_merge:  # per kv-head group; x mode 2: merge the group's attention partials,
                # then zero its raw split-K q/k/v accumulators
                ops.append(make_op(OP_GEMV, i=[H, G * dh, 1, 2, EPI_ADD, -1, 0, 16, dh, cfg.kv_heads, self.max_splits,
                                               CH, self.max_splits, self.oproj_group_tasks], flags=16,
                                   p=[ptr(L["wo_grouped"]), 0, ptr(self.partials), 0, ptr(self.h),
                                      ptr(self.qkv) if self.qkv_split else 0]))
            elif self.oproj_group_tasks:  # per kv-head group, activation rows nq apart
                ops.append(make_op(OP_GEMV, i=[H, G * dh, 1, 0, EPI_ADD, bs, 0, 16, 0, nq, 0, 0, 0,
                                               self.oproj_group_tasks], flags=16,
                                   p=[ptr(L["wo_grouped"]), 0, ptr(self.attn), 0, ptr(self.h)]))
            else:
                ops.append(make_op(OP_GEMV, i=[H, nq, 1, 0, EPI_ADD, bs, 0, 16, 0, 0, 0, 0, 0, 1],
                                   p=[ptr(L["wo"]), 0, ptr(self.attn), 0, ptr(self.h)]))
            assert [ri[n] for n in RT_PER_LAYER] == list(range(ri["topk"], ri["topk"] + len(RT_PER_LAYER)))
            ops.append(make_op(OP_MOE_ROUTE, i=[E, H, 1, 1, EPI_F32, bs, K, 16, cfg.expert_inter, H, ri["topk"], 0, RS,
                                                TS],
                               f=[cfg.eps],
                               p=[ptr(L["router"]), 0, ptr(self.h), ptr(L["ffn_norm"]), ptr(self.logits_r[l]),
                                  ptr(self.xn[l]), ptr(self.wslot[l]), ptr(self.arrive[l:l + 1]), ptr(self.tiles[l]),
                                  ptr(L["wgate"]) if self.l2_prefetch_experts else 0, ptr(L["wup"]),
                                  ptr(L["wdown"])],
                               flags=1 if self.injected else 0))
            if self.group_stage:
                ops.append(make_op(OP_NONE))  # group: the routed notify is the Event Tensor edge itself
            # i9: the batch symbol slot, -1 = one sequence (tiles of token 0: the expert tasks read
            # the slot weight from the tile record)
            ops.append(make_op(OP_MOE_EXPERT,
                               i=[cfg.expert_inter, H, RS, TS, ri["ind"], ri["cnt"], ri["elist"], ri["eoff"], K, bs, E],
                               p=[ptr(L["wgate"]), ptr(L["wup"]), ptr(L["wdown"]), ptr(self.xn[l]), ptr(self.wslot[l]),
                                  ptr(self.h), ptr(self.tiles[l])]))
        ops.append(make_op(OP_GEMV, i=[cfg.vocab, H, 1, 1, EPI_F32, bs, 0, 16, 0, H], f=[cfg.eps],
                           flags=GEMV_ARGMAX if greedy else 0,
                           p=[ptr(W["lm_head"]), 0, ptr(self.h), ptr(W["final_norm"]), ptr(self.logits), 0,
                              ptr(self.best)]))
        return ops

    def greedy_token(self):
        """The last step's greedy token (one sequence), decided on the device (8-byte word)."""
        from .ops import argmax_token
        return argmax_token(self.best.item())

    # ------------------------------------------------------------------
    def inject_routing(self, topk_per_layer):
        """Host-supplied routing (e.g. etsim.moe_realization(...)["topk"] per layer):
        the route tasks skip their top-k and derive counts/indptr/lists from it."""
        for l, tk in enumerate(topk_per_layer):
            self.executor.set_runtime_tensor(f"topk{l}", [int(v) for v in tk])
        if not self.injected:
            self.injected = True
            self.bind()

    def _binding(self, s, b=1):
        return {"s": int(s), "b": int(b)} if self.batched else {"s": int(s)}

    def routing(self, l, b=None):
        """Device-written routing tensors of layer l (after a step with batch b)."""
        cfg = self.cfg
        b = b if b is not None else getattr(self, "last_b", 1)
        n = {"topk": b * cfg.top_k, "cnt": cfg.experts, "ind": cfg.experts + 1, "tind": cfg.experts + 1,
             "elist": b * cfg.top_k, "eoff": cfg.experts + 1}
        return {k: self.executor.runtime_tensor(f"{k}{l}", v) for k, v in n.items()}

    def realization(self):
        """The device routing of the last step as a reference RoutingRealization dict."""
        out = {}
        for l in range(self.cfg.layers):
            for k, v in self.routing(l).items():
                out[f"{k}{l}"] = v
        return out

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

    def step(self, s, b=1):
        self.last_b = b
        self.last_stats = self.executor.run(self._binding(s, b))
        return self.logits

    def launch(self, s, stream=0, b=1):
        self.last_b = b
        self.executor.launch(self._binding(s, b), stream)

    def active_experts(self):
        return [sum(1 for c in self.routing(l)["cnt"] if c > 0) for l in range(self.cfg.layers)]

"""Event Tensor graph specs (reference JSON schema, ref src/json_io.cpp:115-230)
for the decode workloads.  Pure Python: no torch, no extension, so the golden
fixture generator can build the same graphs for the reference implementation.
"""


def graph_spec(cfg, tasks: int, lm_tasks: int, fused_merge: bool = False, allreduce_tasks: int = 0,
               call_tasks=None, attn_cap=None, grouped=False, oproj_group_tasks=16, head_split=1):
    """Reference-format graph spec of one decode step (symbol `s`)."""
    CH = cfg.attn_chunk
    fns, events, calls = [], [], []

    def fn(name, grid):
        fns.append({"name": name, "grid": grid, "resource": "sm", "duration": "unit"})
        return name

    def ev(name, shape):
        events.append({"name": name, "shape": shape})
        return name

    def call(f, ins=(), outs=()):
        c = {"fn": f}
        if ins:
            c["in"] = [{"event": e, "map": m} for e, m in ins]
        if outs:
            c["out"] = [{"event": e, "map": m} for e, m in outs]
        calls.append(c)

    T, kv = str(tasks), str(cfg.kv_heads)
    ct = {k: str(v) for k, v in (call_tasks or {}).items()}  # per-call task counts (whole-tile balance)
    ev("EMB", ["1"])
    call(fn("embed", ["1"]), outs=[("EMB", ["0"])])
    prev = "EMB"
    for l in range(cfg.layers):
        qkv, a, m, o, g, d = (ev(f"{x}{l}", ["1"]) for x in ("QKV", "A", "M", "O", "G", "D"))
        events[-5]["shape"] = [kv]  # A_l has one element per kv head
        if grouped:
            # fine-grained Event Tensors: QKV and M have one element per kv head, so a
            # head group's attention starts when its own q/k/v rows are done and its
            # output projection when its own merge is done
            assert fused_merge, "grouped layers use the fused attention merge"
            Tq = int(ct.get("qkv", T))
            assert Tq % cfg.kv_heads == 0, (Tq, cfg.kv_heads)
            events[-6]["shape"] = [kv]  # QKV_l
            events[-4]["shape"] = [kv]  # M_l
            call(fn(f"L{l}.qkv", [str(Tq)]), ins=[(prev, ["0"])], outs=[(qkv, [f"t0 // {Tq // cfg.kv_heads}"])])
            events.remove(next(e for e in events if e["name"] == a))
            nsplit = f"(s + {CH - 1}) // {CH}"
            if attn_cap:
                nsplit = f"min({nsplit}, {attn_cap})"
            if head_split > 1:  # the q heads of a group shared by head_split tasks per split
                call(fn(f"L{l}.attn", [f"{kv} * {head_split}", f"max({nsplit}, 1)"]),
                     ins=[(qkv, [f"t0 // {head_split}"])], outs=[(m, [f"t0 // {head_split}"])])
            else:
                call(fn(f"L{l}.attn", [kv, f"max({nsplit}, 1)"]), ins=[(qkv, ["t0"])], outs=[(m, ["t0"])])
            call(fn(f"L{l}.oproj", [kv, str(oproj_group_tasks)]), ins=[(m, ["t0"])], outs=[(o, ["0"])])
            call(fn(f"L{l}.gateup", [ct.get("gateup", T)]), ins=[(o, ["0"])], outs=[(g, ["0"])])
            call(fn(f"L{l}.down", [ct.get("down", T)]), ins=[(g, ["0"])], outs=[(d, ["0"])])
            prev = d
            continue
        call(fn(f"L{l}.qkv", [ct.get("qkv", T)]), ins=[(prev, ["0"])], outs=[(qkv, ["0"])])
        nsplit = f"(s + {CH - 1}) // {CH}"
        if attn_cap:  # long contexts: at most attn_cap splits per kv head, each a run of blocks
            nsplit = f"min({nsplit}, {attn_cap})"
        if fused_merge:  # the last split of each kv head merges the group (no merge stage)
            events.remove(next(e for e in events if e["name"] == a))
            call(fn(f"L{l}.attn", [kv, f"max({nsplit}, 1)"]), ins=[(qkv, ["0"])], outs=[(m, ["0"])])
        else:
            call(fn(f"L{l}.attn", [kv, nsplit]), ins=[(qkv, ["0"])], outs=[(a, ["t0"])])
            call(fn(f"L{l}.merge", [kv]), ins=[(a, ["t0"]), (qkv, ["0"])], outs=[(m, ["0"])])
        call(fn(f"L{l}.oproj", [ct.get("oproj", T)]), ins=[(m, ["0"])], outs=[(o, ["0"])])
        if allreduce_tasks:  # tensor parallel: row-parallel partials summed across ranks
            ao = ev(f"AO{l}", ["1"])
            call(fn(f"L{l}.ar_o", [str(allreduce_tasks)]), ins=[(o, ["0"])], outs=[(ao, ["0"])])
            o = ao
        call(fn(f"L{l}.gateup", [ct.get("gateup", T)]), ins=[(o, ["0"])], outs=[(g, ["0"])])
        call(fn(f"L{l}.down", [ct.get("down", T)]), ins=[(g, ["0"])], outs=[(d, ["0"])])
        if allreduce_tasks:
            ad = ev(f"AD{l}", ["1"])
            call(fn(f"L{l}.ar_d", [str(allreduce_tasks)]), ins=[(d, ["0"])], outs=[(ad, ["0"])])
            d = ad
        prev = d
    ev("LM", ["1"])
    call(fn("lm_head", [str(lm_tasks)]), ins=[(prev, ["0"])], outs=[("LM", ["0"])])
    return {
        "symbols": ["s"],
        "size_symbol": "s",
        "duration_models": {"unit": {"kind": "constant", "value": 1}},
        "device_functions": fns,
        "event_tensors": events,
        "calls": calls,
    }


def add_stage_barriers(spec):
    """The "unfused" ablation of a graph spec (the rewrite of ref simulate.cpp:682-794,
    `simulate_barrier_baseline`): one single-element barrier Event Tensor between
    every pair of consecutive calls, so each call starts only once the whole
    previous call finished -- the stage-by-stage execution of one kernel per
    operator, kept inside the persistent launch."""
    import copy

    spec = copy.deepcopy(spec)
    calls = spec["calls"]
    for i in range(len(calls) - 1):
        name = f"__stage{i}"
        spec["event_tensors"].append({"name": name, "shape": ["1"]})
        calls[i].setdefault("out", []).append({"event": name, "map": ["0"]})
        calls[i + 1].setdefault("in", []).append({"event": name, "map": ["0"]})
    return spec

"""CPU restatement of the reference's Event Tensor host path (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module, as the checker; the product never imports it.

It restates, in plain Python over the reference's JSON graph-spec format
(ref proj/src/json_io.cpp:115-230), the algorithms whose results the GPU path
must reproduce bit for bit:

  symexpr      parse / evaluate             ref src/symexpr.cpp:58-87, 115-239
  instantiate  tasks, events, edges, counts ref src/materialize.cpp:98-354
  durations    seeded duration models       ref src/materialize.cpp:26-38, 71-96
  worst_case_rewrite                        ref src/sched_static.cpp:13-47
  lower_static round-robin deal             ref src/sched_static.cpp:49-109
  select_queues next-larger sample + mask   ref src/sched_static.cpp:111-175
  lower_dynamic wait arming                 ref src/sched_dynamic.cpp:7-45
  static execution accounting               ref src/simulate.cpp:183-283 (counters, no-ops)
  moe_realization (std::mt19937_64)         ref src/workloads.cpp:116-150
  random_dag                                ref src/workloads.cpp:152-180

It is pinned against the reference itself: tests/golden/*.json are produced by
tests/golden/make_golden.py from the unmodified reference built in oracle/_ref
(oracle/Makefile), and tests/test_oracle.py checks this module against them.
"""

import bisect
import json
import re

MASK64 = (1 << 64) - 1


# ---------------------------------------------------------------------------
# symbolic expressions (ref symexpr.cpp)

class ExprError(ValueError):
    pass


def _tokens(text):
    pos = 0
    out = []
    while pos < len(text):
        c = text[pos]
        if c.isspace():
            pos += 1
        elif text.startswith("//", pos):
            out.append(("op", "//"))
            pos += 2
        elif c in "+*%(),":
            out.append(("op", c))
            pos += 1
        elif c.isdigit():
            m = re.match(r"\d+", text[pos:])
            out.append(("int", int(m.group(0))))
            pos += len(m.group(0))
        elif c.isalpha() or c == "_":
            m = re.match(r"[A-Za-z_][A-Za-z0-9_]*", text[pos:])
            out.append(("id", m.group(0)))
            pos += len(m.group(0))
        else:
            raise ExprError(f"unexpected character {c!r} in {text!r}")
    return out


def parse(text):
    """Expression tree as nested tuples: ('c', v) | ('s', name) | (op, a, b)."""
    toks = _tokens(text)
    i = 0

    def peek():
        return toks[i] if i < len(toks) else (None, None)

    def atom():
        nonlocal i
        kind, val = peek()
        if kind is None:
            raise ExprError("unexpected end of input")
        i += 1
        if kind == "int":
            return ("c", val)
        if kind == "id":
            if val in ("min", "max") and peek() == ("op", "("):
                i += 1
                a = expr()
                if peek() != ("op", ","):
                    raise ExprError("expected ','")
                i += 1
                b = expr()
                if peek() != ("op", ")"):
                    raise ExprError("expected ')'")
                i += 1
                return (val, a, b)
            return ("s", val)
        if (kind, val) == ("op", "("):
            e = expr()
            if peek() != ("op", ")"):
                raise ExprError("expected ')'")
            i += 1
            return e
        raise ExprError(f"unexpected token {val!r}")

    def term():
        nonlocal i
        e = atom()
        while peek() in (("op", "*"), ("op", "//"), ("op", "%")):
            op = peek()[1]
            i += 1
            e = ({"*": "mul", "//": "div", "%": "mod"}[op], e, atom())
        return e

    def expr():
        nonlocal i
        e = term()
        while peek() == ("op", "+"):
            i += 1
            e = ("add", e, term())
        return e

    e = expr()
    if i != len(toks):
        raise ExprError("unexpected trailing input")
    return e


def evaluate(e, env):
    k = e[0]
    if k == "c":
        v = e[1]
    elif k == "s":
        if e[1] not in env:
            raise ExprError(f"unbound symbol '{e[1]}'")
        v = env[e[1]]
    else:
        a, b = evaluate(e[1], env), evaluate(e[2], env)
        if k == "add":
            v = a + b
        elif k == "mul":
            v = a * b
        elif k == "div":
            if b == 0:
                raise ExprError("division by zero")
            v = a // b
        elif k == "mod":
            if b == 0:
                raise ExprError("modulo by zero")
            v = a % b
        elif k == "min":
            v = min(a, b)
        else:
            v = max(a, b)
    if v < 0:
        raise ExprError(f"expression evaluated to negative value {v}")
    return v


# ---------------------------------------------------------------------------
# seeded durations (ref materialize.cpp:26-38, 71-96)

def _splitmix(x):
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def task_hash(seed, call, coord):
    h = _splitmix((seed & MASK64) ^ 0x5BF03635D1D2C147)
    h = _splitmix(h ^ (call & MASK64))
    for c in coord:
        h = _splitmix(h ^ (c & MASK64))
    return h


def _flatten(coord, ext):
    f = 0
    for c, e in zip(coord, ext):
        f = f * e + c
    return f


def _unflatten(flat, ext):
    out = [0] * len(ext)
    for d in range(len(ext) - 1, -1, -1):
        out[d] = flat % ext[d]
        flat //= ext[d]
    return out


def group_of(flat, indptr):
    i = bisect.bisect_right(indptr, flat)
    if i == 0 or i == len(indptr):
        return -1
    return i - 1


def eval_duration(model, seed, call, coord, ext, realization):
    kind = model["kind"]
    if kind == "constant":
        return model["value"]
    if kind == "table":
        t = model["values"]
        return t[_flatten(coord, ext) % len(t)]
    if kind == "uniform":
        lo, hi = model["lo"], model["hi"]
        return lo + task_hash(seed, call, coord) % (hi - lo + 1)
    if kind == "skewed":
        ip = (realization or {}).get(model["group_indptr"])
        if ip is None:
            return model["base"]
        return model["base"] * model["factor"] if group_of(_flatten(coord, ext), ip) == model["hot_group"] else model["base"]
    raise ExprError(f"unknown duration model kind {kind}")


# ---------------------------------------------------------------------------
# graph helpers

def load(graph_json):
    return json.loads(graph_json) if isinstance(graph_json, str) else graph_json


def _fn(g, name):
    for f in g["device_functions"]:
        if f["name"] == name:
            return f
    raise ExprError(f"unknown function {name}")


def _grid(g, call):
    return call.get("grid") or _fn(g, call["fn"])["grid"]


def _event_index(g, name):
    for i, e in enumerate(g["event_tensors"]):
        if e["name"] == name:
            return i
    return -1


def _prod(v):
    p = 1
    for x in v:
        p *= x
    return p


def instantiate(graph_json, binding, realization=None, seed=0):
    """Returns a dict mirroring MaterializedTaskGraph (ref materialize.hpp:34-54)."""
    g = load(graph_json)
    for s in g.get("symbols", []):
        if s not in binding:
            raise ExprError(f"binding does not bind symbol '{s}'")
    evs = g.get("event_tensors", [])
    ev_ext = [[evaluate(parse(d), binding) for d in e["shape"]] for e in evs]
    offsets, n = [], 0
    for ext in ev_ext:
        offsets.append(n)
        n += _prod(ext)
    rt = {r["name"]: r for r in g.get("runtime_tensors", [])}
    calls = g.get("calls", [])
    extents, counts, first, tasks = [], [], [], []
    for ci, c in enumerate(calls):
        ext = [evaluate(parse(d), binding) for d in _grid(g, c)]
        worst = _prod(ext)
        live = worst
        if c.get("extent_from") and realization is not None:
            live = realization[c["extent_from"]][-1]
            if live > worst:
                raise ExprError("runtime extent exceeds worst-case grid")
        extents.append(ext)
        counts.append(live)
        first.append(len(tasks))
        fn = _fn(g, c["fn"])
        for f in range(live):
            coord = _unflatten(f, ext)
            dur = 1
            if fn.get("duration"):
                dur = eval_duration(g["duration_models"][fn["duration"]], seed, ci, coord, ext, realization)
            tasks.append({"call": ci, "coord": coord, "flat": f, "duration": dur,
                          "resource": fn.get("resource", "sm")})
    waits = [[] for _ in tasks]
    notes = [[] for _ in tasks]
    producers = [[] for _ in range(n)]
    consumers = [[] for _ in range(n)]
    for ci, c in enumerate(calls):
        for direction in ("in", "out"):
            for e in c.get(direction, []):
                ti = _event_index(g, e["event"])
                if ti < 0:
                    raise ExprError(f"unresolved event {e['event']}")
                ext = ev_ext[ti]
                for f in range(counts[ci]):
                    tid = first[ci] + f
                    if "map" in e:
                        env = dict(binding)
                        for d, cv in enumerate(tasks[tid]["coord"]):
                            env[f"t{d}"] = cv
                        coord = [evaluate(parse(m), env) for m in e["map"]]
                        if len(coord) != len(ext) or any(x < 0 or x >= ex for x, ex in zip(coord, ext)):
                            raise ExprError("event index out of bounds")
                        el = offsets[ti] + _flatten(coord, ext)
                    elif "routed_by" in e:
                        el = offsets[ti] + realization[e["routed_by"]][f]
                    else:
                        el = offsets[ti] + group_of(f, realization[e["indptr"]])
                    if direction == "in":
                        waits[tid].append(el)
                        consumers[el].append(tid)
                    else:
                        notes[tid].append(el)
                        producers[el].append(tid)
    initial = []
    for ti, e in enumerate(evs):
        for f in range(_prod(ev_ext[ti])):
            el = offsets[ti] + f
            if e.get("data_dependent"):
                cnt = realization[e["counts"]][f]
                if cnt != len(producers[el]):
                    raise ExprError("data-dependent count disagrees with producer edges")
                initial.append(cnt)
            else:
                initial.append(len(producers[el]))
    return {"tasks": tasks, "waits": waits, "notifies": notes, "producers": producers, "consumers": consumers,
            "initial_counts": initial, "tensor_offsets": offsets, "call_extents": extents,
            "call_task_counts": counts, "call_first_task": first}


def worst_case_rewrite(graph_json):
    g = json.loads(json.dumps(load(graph_json)))
    doomed = {e["name"] for e in g.get("event_tensors", []) if e.get("data_dependent")}
    for c in g.get("calls", []):
        for e in c.get("in", []) + c.get("out", []):
            if "map" not in e:
                doomed.add(e["event"])
    if not doomed:
        return g
    for e in g["event_tensors"]:
        if e["name"] in doomed:
            e["shape"] = ["1"]
            for k in ("data_dependent", "counts", "writer"):
                e.pop(k, None)
    for c in g["calls"]:
        for e in c.get("in", []) + c.get("out", []):
            if e["event"] in doomed:
                e.pop("routed_by", None)
                e.pop("indptr", None)
                e["map"] = ["0"]
    return g


def lower_static(graph_json, samples, num_sms):
    """Per sample: sm_queues (lists of task ids), dma_queue, initial_counts."""
    g = load(graph_json)
    out = []
    for b in samples:
        m = instantiate(g, b)
        sm = [[] for _ in range(num_sms)]
        dma = []
        rr = 0
        for tid, t in enumerate(m["tasks"]):
            if t["resource"] == "dma":
                dma.append(tid)
            else:
                sm[rr % num_sms].append(tid)
                rr += 1
        size_sym = g.get("size_symbol", "")
        out.append({"binding": dict(b), "size_value": b.get(size_sym, 0) if size_sym else 0, "sm_queues": sm,
                    "dma_queue": dma, "initial_counts": m["initial_counts"], "materialized": m})
    out.sort(key=lambda s: s["size_value"])  # stable, like std::stable_sort
    return out


def select_queues(graph_json, samples, actual):
    """(sample index, masked flags by task id, real task count)."""
    g = load(graph_json)
    syms = g.get("symbols", [])
    pick = next((i for i, s in enumerate(samples) if all(s["binding"][k] >= actual[k] for k in syms)), None)
    if pick is None:
        raise ExprError("binding exceeds every sampled shape")
    s = samples[pick]
    live = [[evaluate(parse(d), actual) for d in _grid(g, c)] for c in g["calls"]]
    m = s["materialized"]
    masked = [int(any(x >= e for x, e in zip(t["coord"], live[t["call"]]))) for t in m["tasks"]]
    return pick, masked, len(masked) - sum(masked)


def static_accounting(graph_json, samples, actual, realization=None):
    """What a correct static execution must report (ref simulate.cpp:183-283):
    executed (real) and masked task counts, per-call real counts and the final
    counter values (all zero).  Order of execution is not part of it."""
    g = load(graph_json)
    pick, masked, real = select_queues(g, samples, actual)
    m = samples[pick]["materialized"]
    live = [[evaluate(parse(d), actual) for d in _grid(g, c)] for c in g["calls"]]
    for tid, t in enumerate(m["tasks"]):
        ef = g["calls"][t["call"]].get("extent_from")
        if not masked[tid] and ef and realization is not None:
            if _flatten(t["coord"], live[t["call"]]) >= realization[ef][-1]:
                masked[tid] = 1
    counters = list(m["initial_counts"])
    for tid in range(len(m["tasks"])):
        for el in m["notifies"][tid]:
            counters[el] -= 1
    per_call = [0] * len(g["calls"])
    for tid, t in enumerate(m["tasks"]):
        if not masked[tid]:
            per_call[t["call"]] += 1
    return {"sample_index": pick, "executed": len(masked) - sum(masked), "noops": sum(masked),
            "per_call_real": per_call, "final_counters": counters}


def lower_dynamic_arming(graph_json, early_push=False):
    g = load(graph_json)
    dd = {e["name"] for e in g.get("event_tensors", []) if e.get("data_dependent")}
    return [[1 if (early_push or e["event"] in dd) else 0 for e in c.get("in", [])] for c in g.get("calls", [])]


# ---------------------------------------------------------------------------
# std::mt19937_64 and the seeded generators (ref workloads.cpp:116-180)

class MT19937_64:
    def __init__(self, seed):
        self.mt = [0] * 312
        self.idx = 312
        self.mt[0] = seed & MASK64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & MASK64

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self):
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & MASK64


def moe_realization(tokens=8, experts=4, top_k=1, tile_size=1, hot_fraction=0.0, hot_expert=0, seed=0):
    rng = MT19937_64((seed & MASK64) ^ 0x6D6F655F726E67)
    topk, counts = [], [0] * experts
    for _ in range(tokens):
        chosen = []
        while len(chosen) < top_k:
            if hot_fraction > 0 and float(rng() % 1_000_000) < hot_fraction * 1_000_000.0:
                e = hot_expert
            else:
                e = rng() % experts
            if e not in chosen:
                chosen.append(e)
        topk.extend(chosen)
        for e in chosen:
            counts[e] += 1
    indptr = [0]
    for e in range(experts):
        indptr.append(indptr[-1] + (counts[e] + tile_size - 1) // tile_size)
    return {"topk": topk, "expert_counts": counts, "exp_indptr": indptr}


def random_dag_edges(nodes, edges, seed):
    """(sorted edge set, per-node constant durations) of ref random_dag."""
    rng = MT19937_64((seed & MASK64) ^ 0x646167)
    arcs = set()
    for _ in range(edges):
        if nodes <= 1:
            break
        v = 1 + rng() % (nodes - 1)
        u = rng() % v
        arcs.add((u, v))
    durs = [1 + rng() % 5 for _ in range(nodes)]
    return sorted(arcs), durs

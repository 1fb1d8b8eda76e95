"""Full-depth parity of a device decode step against the CPU oracle (TEST
INFRASTRUCTURE ONLY: called by tests/ and, after its timed region, by bench.py
to put the error figures of the benchmarked step in its JSON line; the
product path never imports this module).

The checked model's seeded weights are drawn again on its device with the same
generator (decode.init_weights / moe.init_moe_weights, layer_hook), and every
layer is handed to the oracle as soon as it is drawn, so a 32-layer Llama-3-8B
or a 48-layer Qwen3-30B-A3B is checked without ever holding the model in host
memory (one layer at a time; only the experts the device routed to move to
the host).  The oracle reads the same KV cache positions [0, s) the device
read, and the device's own K/V rows appended at position s give a per-layer
error profile (the K/V of layer l are a function of the hidden state after
layer l-1).

Tolerances (stated here and asserted by the callers):
- logits: max|err| <= max(LOGIT_TOL * max|logit|, 2 * floor) against the
  bf16-emulating oracle.  Both sides round the same activations to bf16
  (normalised x, attention output, SiLU product, appended K/V) from fp32 values
  summed in a different order, so isolated 1-ulp (2^-8 relative) flips are
  expected and propagate through the residual stream.  `floor` is the oracle's
  own noise floor: the distance between the float32 oracle and the same oracle
  accumulating in float64 (identical bf16 rounding points, a different
  summation order) -- the device may differ from the oracle at most twice as
  much as the oracle differs from itself.  Measured on B200: DESIGN.md (c).
- appended K/V rows, per layer: rel err <= max(KV_TOL, 2 * the floor's).
- greedy token: equal whenever the oracle's top-2 margin exceeds 2 x err.
- MoE routing: the device's top-k set must equal the oracle's own top-k set
  (computed from the oracle's router logits) for every layer and checked
  sequence, except where the oracle's k-th / (k+1)-th logit margin is within
  2 x the router-logit error (a near tie; counted and reported).
"""

import torch

from oracle.decoder_oracle import DecodeStream
from oracle.moe_oracle import MoEDecodeStream, topk_ref

LOGIT_TOL = 3.125e-2  # x max|logit| (8 bf16 epsilons), full depth; measured 1.5-1.7% (DESIGN.md (c))
KV_TOL = 5e-2         # x max|k or v| of the layer, per appended row


def _summ(ref, dev):
    err = (dev - ref).abs().max().item()
    scale = ref.abs().max().item()
    return err, scale


def _logit_report(out, logits_dev, ref, ref64=None):
    err, scale = _summ(ref, logits_dev)
    top2 = ref.topk(2).values
    margin = (top2[0] - top2[1]).item()
    floor = (ref64 - ref).abs().max().item() if ref64 is not None else 0.0
    tol = max(LOGIT_TOL, 2 * floor / scale)
    out.update(max_abs=err, max_rel=err / scale, scale=scale, tol=tol, floor_rel=floor / scale,
               argmax_dev=int(logits_dev.argmax()), argmax_ref=int(ref.argmax()), top2_margin=margin)
    out["argmax_ok"] = out["argmax_dev"] == out["argmax_ref"] or margin <= 2 * err
    out["pass"] = bool(err <= tol * scale and out["argmax_ok"] and out.get("kv_pass", True)
                       and out.get("routing_pass", True))
    return out


def _kv_err(k_ref, v_ref, k_dev, v_dev):
    ek = (k_dev - k_ref).abs().max().item() / max(k_ref.abs().max().item(), 1e-30)
    ev = (v_dev - v_ref).abs().max().item() / max(v_ref.abs().max().item(), 1e-30)
    return max(ek, ev)


@torch.no_grad()
def dense_parity(cfg, seed, device, tokens, s, inv_freq, kcache, vcache, logits, seqs=(0,), swizzled=False,
                 floor=True):
    """Llama-style decoder: seqs = which batch rows to check.
    kcache/vcache: device per-layer caches, [kv][cap][dh] or [b][kv][cap][dh];
    logits: device logits [b][vocab] (or [1][vocab]); tokens: host list per row."""
    from paper_2604_13327_b200.decode import init_weights

    inv = inv_freq.cpu()
    streams = {t: DecodeStream(cfg, tokens[t], s, inv) for t in seqs}
    twins = {t: DecodeStream(cfg, tokens[t], s, inv, dtype=torch.float64) for t in seqs} if floor else {}
    kv_rel = {t: [] for t in seqs}
    kv_floor = {t: [] for t in seqs}
    head = {}

    def cache_rows(l, t):
        kc, vc = kcache[l], vcache[l]
        if kc.dim() == 4:
            kc, vc = kc[t], vc[t]
        if swizzled:
            from paper_2604_13327_b200.batch import cache_swizzle
            kc, vc = cache_swizzle(kc), cache_swizzle(vc)
        return kc.cpu(), vc.cpu()

    state = {"l": 0}

    def hook(d):
        if "embed" in d:
            for t in seqs:
                for st in (streams[t], twins.get(t)):
                    if st is not None:
                        st.head(d["embed"][tokens[t]].cpu())
            head["final_norm"] = d["final_norm"].cpu()
            head["lm_head"] = d["lm_head"].cpu()
            return {"layers": []}
        l = state["l"]
        Lc = {k: v.cpu() for k, v in d.items()}
        for t, st in streams.items():
            kc, vc = cache_rows(l, t)
            k, v = st.layer(Lc, kc, vc)
            kv_rel[t].append(_kv_err(k, v, kc[:, s].float(), vc[:, s].float()))
            if t in twins:
                k2, v2 = twins[t].layer(Lc, kc, vc)
                kv_floor[t].append(_kv_err(k, v, k2.float(), v2.float()))
        state["l"] += 1
        return {}

    init_weights(cfg, device, seed, layer_hook=hook)
    out = {"oracle": "oracle/decoder_oracle.py DecodeStream (bf16-emulating fp32), weights regenerated from seed",
           "layers": cfg.layers, "seq": s, "seqs": {}}
    worst = None
    for t, st in streams.items():
        ref = st.final(head["final_norm"], head["lm_head"])
        ref64 = twins[t].final(head["final_norm"], head["lm_head"]) if t in twins else None
        kvf = max(kv_floor[t]) if kv_floor[t] else 0.0
        r = {"kv_max_rel": max(kv_rel[t]), "kv_rel_last_layer": kv_rel[t][-1], "kv_floor_rel": kvf,
             "kv_tol": max(KV_TOL, 2 * kvf), "kv_rel_per_layer": [round(x, 5) for x in kv_rel[t]]}
        r["kv_pass"] = r["kv_max_rel"] <= r["kv_tol"]
        _logit_report(r, logits[t].float().cpu(), ref, ref64)
        out["seqs"][str(t)] = r
        if worst is None or r["max_rel"] > worst["max_rel"]:
            worst = r
    for k in ("max_abs", "max_rel", "tol", "floor_rel", "kv_max_rel", "argmax_ok"):
        out[k] = worst[k]
    out["pass"] = all(r["pass"] for r in out["seqs"].values())
    return out


@torch.no_grad()
def moe_parity(cfg, seed, device, tokens, s, inv_freq, kcache, vcache, logits, router_logits, device_topk,
               seqs=(0,), swizzled=False, xn_taps=None, floor=True):
    """Qwen3-MoE decoder.  router_logits: device [layers][b][E]; device_topk(l, t):
    the device's selected experts of sequence t in layer l (selection order);
    xn_taps: the device's normalised pre-FFN activations [layers][b][H] (bf16), which
    give a per-layer divergence profile and a teacher-forced check of the router
    GEMV (device logits vs router @ the device's own xn, layer by layer)."""
    from paper_2604_13327_b200.moe import init_moe_weights

    inv = inv_freq.cpu()
    K = cfg.top_k
    streams = {t: MoEDecodeStream(cfg, tokens[t], s, inv) for t in seqs}
    twins = {t: MoEDecodeStream(cfg, tokens[t], s, inv, dtype=torch.float64) for t in seqs} if floor else {}
    kv_rel = {t: [] for t in seqs}
    kv_floor = {t: [] for t in seqs}
    rstat = {t: {"router_max_abs": 0.0, "exact": 0, "near_tie": 0, "mismatch": 0} for t in seqs}
    prof = {t: {"kv_rel": [], "xn_rel": [], "router_local_rel": []} for t in seqs}
    head = {}
    state = {"l": 0}

    def cache_rows(l, t):
        kc, vc = kcache[l][t], vcache[l][t]
        if swizzled:
            from paper_2604_13327_b200.batch import cache_swizzle
            kc, vc = cache_swizzle(kc), cache_swizzle(vc)
        return kc.cpu(), vc.cpu()

    def hook(d):
        if "embed" in d:
            for t in seqs:
                for st in (streams[t], twins.get(t)):
                    if st is not None:
                        st.head(d["embed"][tokens[t]].cpu())
            head["final_norm"] = d["final_norm"].cpu()
            head["lm_head"] = d["lm_head"].cpu()
            return {"layers": []}
        l = state["l"]
        dense = {k: v.cpu() for k, v in d.items() if k not in ("wgate", "wup", "wdown")}
        cache = {}

        def expert(ex):
            if ex not in cache:
                cache[ex] = (d["wgate"][ex].cpu(), d["wup"][ex].cpu(), d["wdown"][ex].cpu())
            return cache[ex]

        for t, st in streams.items():
            kc, vc = cache_rows(l, t)
            dev_sel = [int(x) for x in device_topk(l, t)]
            lg, _, k, v = st.layer(dense, kc, vc, expert=expert, routing=dev_sel)
            kv_rel[t].append(_kv_err(k, v, kc[:, s].float(), vc[:, s].float()))
            if t in twins:
                _, _, k2, v2 = twins[t].layer(dense, kc, vc, expert=expert, routing=dev_sel)
                kv_floor[t].append(_kv_err(k, v, k2.float(), v2.float()))
            dlg = router_logits[l][t].float().cpu()
            pf = prof[t]
            pf["kv_rel"].append(round(kv_rel[t][-1], 5))
            if xn_taps is not None:
                xd = xn_taps[l][t].float().cpu()
                pf["xn_rel"].append(round((xd - st.last_xn).abs().max().item() / st.last_xn.abs().max().item(), 5))
                loc = dense["router"].float() @ xd
                pf["router_local_rel"].append(round((dlg - loc).abs().max().item() / loc.abs().max().item(), 6))
            rerr = (dlg - lg).abs().max().item()
            rs = rstat[t]
            rs["router_max_abs"] = max(rs["router_max_abs"], rerr)
            own = topk_ref(lg.tolist(), K)
            if sorted(own) == sorted(dev_sel):
                rs["exact"] += 1
            else:
                srt = sorted(lg.tolist(), reverse=True)
                if srt[K - 1] - srt[K] <= 2 * rerr:
                    rs["near_tie"] += 1
                else:
                    rs["mismatch"] += 1
        state["l"] += 1
        return {}

    init_moe_weights(cfg, device, seed, layer_hook=hook)
    out = {"oracle": "oracle/moe_oracle.py MoEDecodeStream (bf16-emulating fp32, device routing forced for the "
                     "logits; the oracle's own top-k compared per layer), weights regenerated from seed",
           "layers": cfg.layers, "seq": s, "seqs": {}}
    worst = None
    for t, st in streams.items():
        ref = st.final(head["final_norm"], head["lm_head"])
        ref64 = twins[t].final(head["final_norm"], head["lm_head"]) if t in twins else None
        r = dict(rstat[t])
        r["per_layer"] = prof[t]
        r["routing_pass"] = r["mismatch"] == 0
        kvf = max(kv_floor[t]) if kv_floor[t] else 0.0
        r.update(kv_max_rel=max(kv_rel[t]), kv_floor_rel=kvf, kv_tol=max(KV_TOL, 2 * kvf))
        r["kv_pass"] = r["kv_max_rel"] <= r["kv_tol"]
        _logit_report(r, logits[t].float().cpu(), ref, ref64)
        out["seqs"][str(t)] = r
        if worst is None or r["max_rel"] > worst["max_rel"]:
            worst = r
    for k in ("max_abs", "max_rel", "tol", "floor_rel", "kv_max_rel", "argmax_ok"):
        out[k] = worst[k]
    out["routing"] = {k: sum(out["seqs"][str(t)][k] for t in seqs) for k in ("exact", "near_tie", "mismatch")}
    out["pass"] = all(r["pass"] for r in out["seqs"].values())
    return out

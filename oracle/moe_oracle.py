"""CPU restatement of one Qwen3-MoE-style decode step (TEST INFRASTRUCTURE ONLY:
imported by tests/ and bench.py's CPU baseline, never by the product path).

The reference has no numerics (ref SPEC.md:8), so logits parity is unpinned
by the reference; this follows the standard Qwen3-MoE decoder definition on
the same random-init bf16 weights (paper_2604_13327_b200.moe.init_moe_weights):
per-head q/k RMSNorm before RoPE (adjacent-pair rotation), GQA attention,
softmax router with top-k (descending logit; lower expert index on ties) and
renormalised weights, SiLU-gated experts; bf16 rounding of activations where
the kernel stores bf16 (emulate_bf16).  The routing algebra (counts, tile
indptr) follows ref workloads.cpp:116-150 (`moe_routing_tensors`).
"""

import torch

from oracle.decoder_oracle import DecodeStream, _bf16, rmsnorm, rotary_pairs


def topk_ref(logits, k):
    """Top-k expert ids in selection order: larger logit first, lower index on ties."""
    order = sorted(range(len(logits)), key=lambda e: (-float(logits[e]), e))
    return order[:k]


def moe_routing_tensors(topk_flat, experts, tile, row_splits):
    """counts, exp_indptr (ceil(count/tile) prefix, ref workloads.cpp:137-144),
    task_indptr (x row_splits), eoff (prefix of counts), elist (slots by expert, stable)."""
    cnt = [0] * experts
    for e in topk_flat:
        cnt[e] += 1
    ind, eoff = [0], [0]
    for e in range(experts):
        ind.append(ind[-1] + (cnt[e] + tile - 1) // tile)
        eoff.append(eoff[-1] + cnt[e])
    cur = list(eoff[:-1])
    elist = [0] * len(topk_flat)
    for slot, e in enumerate(topk_flat):
        elist[cur[e]] = slot
        cur[e] += 1
    return {"cnt": cnt, "ind": ind, "tind": [v * row_splits for v in ind], "eoff": eoff, "elist": elist}


class MoEDecodeStream(DecodeStream):
    """One Qwen3-MoE decode step of one sequence, fed layer by layer (see
    DecodeStream).  layer() takes the layer's dense weights plus an `expert(e)`
    accessor returning (gate [I, H], up [I, H], down [H, I]) of expert e, so only
    the experts the step routes to need to reach host memory."""

    @torch.no_grad()
    def layer(self, L, kc, vc, expert=None, routing=None):
        """Returns (router logits [E], selected experts, new k, new v).  routing: the
        experts to use (the device's choice) instead of the oracle's own top-k."""
        cfg, e, f32 = self.cfg, self.e, self.dt
        d, nq, nkv = cfg.head_dim, cfg.heads, cfg.kv_heads
        if expert is None:
            def expert(ex):
                return L["wgate"][ex], L["wup"][ex], L["wdown"][ex]
        h = self.h
        x = _bf16(rmsnorm(h, L["attn_norm"].to(f32), cfg.eps), e)
        qkv = L["wqkv"].to(f32) @ x
        q = qkv[: nq * d].view(nq, d)
        k = qkv[nq * d: nq * d + nkv * d].view(nkv, d)
        v = qkv[nq * d + nkv * d:].view(nkv, d)
        q = rotary_pairs(rmsnorm(q, L["q_norm"].to(f32), cfg.eps), self.s, self.inv_freq)
        k = _bf16(rotary_pairs(rmsnorm(k, L["k_norm"].to(f32), cfg.eps), self.s, self.inv_freq), e)
        v = _bf16(v, e)
        h = h + L["wo"].to(f32) @ self.attention(q, k, v, kc, vc)
        xn = _bf16(rmsnorm(h, L["ffn_norm"].to(f32), cfg.eps), e)
        self.last_xn = xn
        lg = L["router"].to(f32) @ xn
        sel = list(routing) if routing is not None else topk_ref(lg.tolist(), cfg.top_k)
        pr = torch.softmax(lg.to(torch.float64), dim=0)
        w = pr[sel] / pr[sel].sum()
        for j, ex in enumerate(sel):
            wg, wu, wd = expert(ex)
            act = _bf16(torch.nn.functional.silu(wg.to(f32) @ xn) * (wu.to(f32) @ xn), e)
            h = h + float(w[j]) * (wd.to(f32) @ act)
        self.h = h
        return lg, sel, k, v


@torch.no_grad()
def moe_decode_step(cfg, W, kcache, vcache, token, s, inv_freq, emulate_bf16=True, routing=None):
    """Returns (logits [vocab], per-layer router logits, per-layer topk).

    routing: optional list (per layer) of forced top-k expert lists (the device's
    choice), so that numerics can be compared even across a router near-tie."""
    st = MoEDecodeStream(cfg, token, s, inv_freq, emulate_bf16)
    st.head(W["embed"][token])
    router_logits, topks = [], []
    for l, L in enumerate(W["layers"]):
        lg, sel, _, _ = st.layer(L, kcache[l], vcache[l], routing=routing[l] if routing is not None else None)
        router_logits.append(lg)
        topks.append(sel)
    return st.final(W["final_norm"], W["lm_head"]), router_logits, topks

"""CPU fp32 oracle for one decode step (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module, and only as the checker / CPU baseline; the product path never
imports it.

The reference (arxiv/paper_2604_13327, proj/) has no numerics at all: its
tasks are duration-modelled (ref SPEC.md:8, materialize.cpp:71-96), so logits
parity is *unpinned by the reference* (SURVEY.md section 8c).  This is a plain
restatement of a Llama-style decoder step on the same bf16 weights:

    h = E[token]
    per layer:  x = rmsnorm(h) * g_attn;  q,k,v = Wqkv x;  rotary on (2j, 2j+1)
                pairs with theta^(-2j/d);  k,v appended at position s;
                attention of q over positions [0, s] (GQA), o = Wo attn; h += o
                x = rmsnorm(h) * g_ffn;  h += Wdown (silu(Wgate x) * (Wup x))
    logits = Wlm (rmsnorm(h) * g_final)

`emulate_bf16=True` rounds the activations at the same points the device
does (GEMV inputs, attention output, SiLU product, the appended K/V rows) so
the comparison can use a tight tolerance; `False` is the pure fp32 model.
"""

import torch


def _bf16(x, on):
    return x.to(torch.bfloat16).to(x.dtype) if on else x


def rmsnorm(h, g, eps):
    return h * torch.rsqrt((h * h).mean(-1, keepdim=True) + eps) * g


def rotary_pairs(x, pos, inv_freq):
    """x: [..., d]; rotates (2j, 2j+1) by angle pos * inv_freq[j] (fp32 angle as on device)."""
    ang = (torch.tensor(float(pos), dtype=torch.float32) * inv_freq).to(torch.float64)
    c, s = torch.cos(ang).to(x.dtype), torch.sin(ang).to(x.dtype)
    a, b = x[..., 0::2], x[..., 1::2]
    out = torch.empty_like(x)
    out[..., 0::2] = a * c - b * s
    out[..., 1::2] = a * s + b * c
    return out


class DecodeStream:
    """One decode step of one sequence, fed layer by layer (so a full-depth model
    never has to sit in host memory: bench.py and the full-depth parity test
    regenerate the seeded weights and hand each layer over as it is drawn).

    head(embed_row) -> layer(L, kcache_l, vcache_l)* -> final(final_norm, lm_head).

    dtype: the accumulation type (float32; float64 gives a second summation
    order of the same function, whose distance to the float32 stream is the
    oracle's own rounding noise floor -- oracle/parity.py)."""

    def __init__(self, cfg, token, s, inv_freq, emulate_bf16=True, dtype=torch.float32):
        self.cfg, self.token, self.s, self.e, self.dt = cfg, token, s, emulate_bf16, dtype
        self.inv_freq = inv_freq
        self.h = None

    def head(self, embed_row):
        self.h = embed_row.to(self.dt).clone()

    @torch.no_grad()
    def attention(self, q, k, v, kc, vc):
        """GQA attention of q [nq, d] over the cached positions [0, s) plus (k, v)."""
        cfg, s = self.cfg, self.s
        f32 = self.dt
        d, nq, nkv = cfg.head_dim, cfg.heads, cfg.kv_heads
        G = nq // nkv
        K = torch.cat([kc[:, :s].to(f32), k[:, None]], dim=1)  # [nkv, s+1, d]
        V = torch.cat([vc[:, :s].to(f32), v[:, None]], dim=1)
        att = torch.empty(nq, d, dtype=f32)
        for hh in range(nq):
            g = hh // G
            sc = (K[g] @ q[hh]) / (d ** 0.5)
            p = torch.softmax(sc.to(torch.float64), dim=0).to(f32)
            att[hh] = p @ V[g]
        return _bf16(att.reshape(-1), self.e)

    @torch.no_grad()
    def layer(self, L, kc, vc):
        """Returns the layer's new (k, v) rows [nkv, d] (what the device appends at s)."""
        cfg, e, f32 = self.cfg, self.e, self.dt
        d, nq, nkv = cfg.head_dim, cfg.heads, cfg.kv_heads
        h = self.h
        x = _bf16(rmsnorm(h, L["attn_norm"].to(f32), cfg.eps), e)
        qkv = L["wqkv"].to(f32) @ x
        q = qkv[: nq * d].view(nq, d)
        k = qkv[nq * d: nq * d + nkv * d].view(nkv, d)
        v = qkv[nq * d + nkv * d:].view(nkv, d)
        q = rotary_pairs(q, self.s, self.inv_freq)
        k = _bf16(rotary_pairs(k, self.s, self.inv_freq), e)
        v = _bf16(v, e)
        h = h + L["wo"].to(f32) @ self.attention(q, k, v, kc, vc)
        x = _bf16(rmsnorm(h, L["ffn_norm"].to(f32), cfg.eps), e)
        gate = L["wgate"].to(f32) @ x
        up = L["wup"].to(f32) @ x
        act = _bf16(torch.nn.functional.silu(gate) * up, e)
        self.h = h + L["wdown"].to(f32) @ act
        return k, v

    @torch.no_grad()
    def final(self, final_norm, lm_head):
        x = _bf16(rmsnorm(self.h, final_norm.to(self.dt), self.cfg.eps), self.e)
        return (lm_head.to(self.dt) @ x).to(torch.float32)


@torch.no_grad()
def decode_step(cfg, W, kcache, vcache, token, s, inv_freq, emulate_bf16=True):
    """Returns (logits [vocab] fp32, new_k [layers][kv_heads][d], new_v ...).

    W: dict of CPU tensors (same structure as decode.init_weights); caches:
    lists of CPU [kv_heads, capacity, d] tensors (positions [0, s) are read).
    """
    st = DecodeStream(cfg, token, s, inv_freq, emulate_bf16)
    st.head(W["embed"][token])
    new_k, new_v = [], []
    for l, L in enumerate(W["layers"]):
        k, v = st.layer(L, kcache[l], vcache[l])
        new_k.append(k)
        new_v.append(v)
    return st.final(W["final_norm"], W["lm_head"]), new_k, new_v


def weights_to_cpu(W):
    out = {k: v.detach().cpu() for k, v in W.items() if k != "layers"}
    out["layers"] = [{k: v.detach().cpu() for k, v in L.items()} for L in W["layers"]]
    return out

import dataclasses, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle.decoder_oracle import weights_to_cpu, rmsnorm, _bf16, rotary_pairs
from paper_2604_13327_b200.decode import LLAMA3_8B, DecodeModel
cfg = dataclasses.replace(LLAMA3_8B, name="x", layers=1, hidden=1024, heads=8, kv_heads=2, intermediate=4096)
m = DecodeModel(cfg, samples=(1024,), seed=0, keep_logical=True)
Wc = weights_to_cpu(m.W_logical)
for s in (64, 1024, 100):
    m.fill_cache(s, seed=1); m.set_token(123)
    ck = m.kcache[0].cpu().float(); cv = m.vcache[0].cpu().float()
    m.step(s)
    L = Wc["layers"][0]; d = cfg.head_dim; nq, nkv = cfg.heads, cfg.kv_heads; G = nq // nkv
    h = Wc["embed"][123].float()
    x = _bf16(rmsnorm(h, L["attn_norm"].float(), cfg.eps), True)
    qkv = L["wqkv"].float() @ x
    q = rotary_pairs(qkv[: nq * d].view(nq, d), s, m.inv_freq.cpu())
    k = _bf16(rotary_pairs(qkv[nq * d: nq * d + nkv * d].view(nkv, d), s, m.inv_freq.cpu()), True)
    v = _bf16(qkv[nq * d + nkv * d:].view(nkv, d), True)
    qd = m.q.cpu().view(nq, d)
    print("s", s, "q err", (qd - q).abs().max().item(), "q scale", q.abs().max().item())
    K = torch.cat([ck[:, :s], k[:, None]], 1); V = torch.cat([cv[:, :s], v[:, None]], 1)
    att = torch.empty(nq, d)
    for hh in range(nq):
        g = hh // G
        p = torch.softmax(((K[g] @ q[hh]) / d ** 0.5).double(), 0).float()
        att[hh] = p @ V[g]
    ad = m.attn.cpu().float().view(nq, d)
    print("   attn err", (ad - _bf16(att, True)).abs().max().item(), "scale", att.abs().max().item(),
          "per-head max err", [round((ad[i] - att[i]).abs().max().item(), 4) for i in range(nq)])
    kc = m.kcache[0][:, s].cpu().float()
    print("   new k err", (kc - k).abs().max().item())

import json, sys
sys.path.insert(0, '.')
import torch
from oracle.parity import moe_parity
from paper_2604_13327_b200.moe import QWEN3_30B_A3B, MoEDecodeModel
cfg, s = QWEN3_30B_A3B, 1024
m = MoEDecodeModel(cfg, samples=(s,), seed=0, scheduler="static")
m.fill_cache(s, seed=1)
m.set_token(1)
m.step(s)
r = moe_parity(cfg, 0, m.device, [1], s, m.inv_freq, m.kcache, m.vcache, m.logits, m.logits_r,
               lambda l, t: m.routing(l, 1)["topk"], xn_taps=m.xn)
print(json.dumps(r["seqs"]["0"]["per_layer"]))
print(json.dumps({k: v for k, v in r["seqs"]["0"].items() if k != "per_layer"}))

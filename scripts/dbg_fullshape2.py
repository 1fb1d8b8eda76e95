import dataclasses, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle.decoder_oracle import decode_step, weights_to_cpu
from paper_2604_13327_b200.decode import LLAMA3_8B, DecodeModel
for over in (dict(), dict(intermediate=4096), dict(vocab=4096), dict(hidden=1024, heads=8, kv_heads=2, intermediate=4096)):
    cfg = dataclasses.replace(LLAMA3_8B, name="x", layers=1, **over)
    m = DecodeModel(cfg, samples=(1024,), seed=0, keep_logical=True)
    Wc = weights_to_cpu(m.W_logical)
    for s in (0, 64, 1024):
        m.fill_cache(s, seed=1); m.set_token(123)
        ck = [k.cpu() for k in m.kcache]; cv = [v.cpu() for v in m.vcache]
        logits = m.step(s)[0].cpu()
        ref, _, _ = decode_step(cfg, Wc, ck, cv, 123, s, m.inv_freq.cpu(), emulate_bf16=True)
        print(over, "s", s, "err", round((logits - ref).abs().max().item(), 5), "scale", round(ref.abs().max().item(), 3),
              "rel", round(((logits - ref).abs().max() / ref.abs().max()).item(), 5), flush=True)
    del m; torch.cuda.empty_cache()

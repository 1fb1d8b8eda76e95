import dataclasses, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle.decoder_oracle import decode_step, weights_to_cpu, rmsnorm, _bf16
from paper_2604_13327_b200.decode import LLAMA3_8B, DecodeModel
cfg = dataclasses.replace(LLAMA3_8B, name="llama3-8b-2L", layers=int(sys.argv[1]) if len(sys.argv) > 1 else 2)
for kw in (dict(), dict(residual="double"), dict(fused_merge=False)):
    m = DecodeModel(cfg, samples=(1024,), seed=0, keep_logical=True, **kw)
    s = 1024
    m.fill_cache(s, seed=1); m.set_token(123)
    ck = [k.cpu() for k in m.kcache]; cv = [v.cpu() for v in m.vcache]
    logits = m.step(s)[0].cpu()
    h_dev = m.h_a[0].cpu()
    Wc = weights_to_cpu(m.W_logical)
    for emu in (True, False):
        ref, _, _ = decode_step(cfg, Wc, ck, cv, 123, s, m.inv_freq.cpu(), emulate_bf16=emu)
        print(kw, "emulate", emu, "logit err", (logits - ref).abs().max().item(), "scale", ref.abs().max().item(), flush=True)
    # lm_head on the device h with the oracle's rounding
    x = _bf16(rmsnorm(h_dev, Wc["final_norm"].float(), cfg.eps), True)
    lg2 = Wc["lm_head"].float() @ x
    print("   lm_head(device h) vs device logits", (lg2 - logits).abs().max().item(), flush=True)
    del m
    torch.cuda.empty_cache()

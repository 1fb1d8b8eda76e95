"""A/B of DecodeModel construction options in ONE process on shared weights
(timing experiment): median kernel ms per variant, interleaved rounds.

    python scripts/ab_models.py [moe] '{"tc_attention": false}' '{"tc_attention": true}'
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_13327_b200.decode import LLAMA3_8B, DecodeModel, init_weights  # noqa: E402

moe = sys.argv[1] == "moe"
variants = [json.loads(a) for a in sys.argv[2 if moe else 1:]] or [{}]
models = []
if moe:
    # one model (its device weights take 61 GB): variants are attributes set before re-binding
    # the op table (same lowered program)
    from paper_2604_13327_b200.moe import MOE_CONFIGS, MoEDecodeModel
    base = MoEDecodeModel(MOE_CONFIGS["qwen3-30b-a3b"], samples=(1024,))
    base.fill_cache(1024, seed=1)
    base.set_token([1])

    class _V:
        def __init__(self, kw):
            self.kw, self.executor = kw, base.executor

        def activate(self):
            for k, v in self.kw.items():
                setattr(base, k, v)
            base.bind()

        def greedy_token(self):
            return int(base.logits[0].argmax())
    models = [_V(kw) for kw in variants]
    B = base._binding(1024, 1)
else:
    W = init_weights(LLAMA3_8B, "cuda:0", 0)
    for kw in variants:
        m = DecodeModel(LLAMA3_8B, samples=(1024,), weights=W, **kw)
        m.fill_cache(1024)
        m.set_token(1)
        models.append(m)
    B = {"s": 1024}
res = [[] for _ in models]
for _ in range(5):
    for i, m in enumerate(models):
        if moe:
            m.activate()
        ts = [m.executor.run(B)["kernel_ms"] for _ in range(6)]
        res[i] += ts[1:]
for kw, r, m in zip(variants, res, models):
    print(json.dumps({"variant": kw, "median_ms": round(statistics.median(r), 4), "min_ms": round(min(r), 4),
                      "greedy": m.greedy_token()}), flush=True)

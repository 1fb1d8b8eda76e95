"""A/B of DecodeModel construction options in ONE process on shared weights
(timing experiment): median kernel ms per variant, interleaved rounds.

    python scripts/ab_models.py '{"tc_attention": false}' '{"tc_attention": true}'
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_13327_b200.decode import LLAMA3_8B, DecodeModel, init_weights  # noqa: E402

variants = [json.loads(a) for a in sys.argv[1:]] or [{}]
W = init_weights(LLAMA3_8B, "cuda:0", 0)
models = []
for kw in variants:
    m = DecodeModel(LLAMA3_8B, samples=(1024,), weights=W, **kw)
    m.fill_cache(1024)
    m.set_token(1)
    models.append(m)
res = [[] for _ in models]
for _ in range(5):
    for i, m in enumerate(models):
        ts = [m.executor.run({"s": 1024})["kernel_ms"] for _ in range(6)]
        res[i] += ts[1:]
for kw, r, m in zip(variants, res, models):
    print(json.dumps({"variant": kw, "median_ms": round(statistics.median(r), 4), "min_ms": round(min(r), 4),
                      "greedy": m.greedy_token()}), flush=True)

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_13327_b200.moe import TINY_MOE, MoEDecodeModel
m = MoEDecodeModel(TINY_MOE, samples=(64,), num_workers=16, seed=0, scheduler=sys.argv[1] if len(sys.argv) > 1 else "static",
                   max_batch=16, batch_samples=(2, 16))
m.fill_cache(16, seed=1)
m.set_token(list(range(1, 17)))
print(m.step(16, 1)[0, :4])

import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_13327_b200.decode import CONFIGS, DecodeModel
l2 = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cfg = CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "llama3-8b"]
m = DecodeModel(cfg, samples=(1024,), l2_prefetch=l2)
m.fill_cache(1024); m.set_token(1)
for _ in range(3):
    st = m.executor.run({"s": 1024})
print("kernel_ms", st["kernel_ms"], flush=True)

import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_13327_b200.decode import CONFIGS
from paper_2604_13327_b200.tp import TPDecodeModel
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama3-70b"]
t0 = time.time()
m = TPDecodeModel(cfg, 0, 1, samples=(1024,), seed=0, record_trace=False)
m.connect([m.local_buffers()])
print("init s", time.time() - t0, "mem GB", torch.cuda.memory_allocated() / 1e9, flush=True)
m.fill_cache(1024)
m.set_token(1)
for i in range(3):
    try:
        st = m.executor.run({"s": 1024})
        print(i, st, flush=True)
    except Exception as e:
        print(i, "ERR", e, flush=True)

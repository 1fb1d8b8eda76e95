import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_13327_b200.decode import CONFIGS, DecodeModel, init_weights
cfg = CONFIGS["llama3-8b"]
W = init_weights(cfg, torch.device("cuda:0"), 0)
for l2 in [int(x) for x in sys.argv[1:]] or [0, 131072, 393216, 1048576]:
    m = DecodeModel(cfg, samples=(1024,), weights=W if l2 == 0 else None, l2_prefetch=l2, seed=0) if False else None
    break
m = DecodeModel(cfg, samples=(1024,), weights=W, keep_logical=False)
m.fill_cache(1024); m.set_token(1)
import paper_2604_13327_b200.etsim as etsim
from paper_2604_13327_b200.ops import pack
for l2 in [int(x) for x in sys.argv[1:]] or [0, 131072, 393216, 1048576]:
    ex = etsim.Executor(m.kernel, num_workers=m.num_workers, record_trace=False, l2_prefetch=l2)
    ex.bind_ops(pack(m._ops()))
    ts = []
    for i in range(6):
        ts.append(ex.run({"s": 1024})["kernel_ms"])
    print("l2_prefetch", l2, "kernel_ms", ["%.3f" % t for t in ts], "median", statistics.median(ts[2:]), flush=True)
    del ex

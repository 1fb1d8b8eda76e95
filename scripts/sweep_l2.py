"""L2 run-ahead sweep for the Llama-3-8B decode step (timing experiment, not a test).
    python scripts/sweep_l2.py [bytes ...]      (ET_DEBUG=64: run ahead only while the ring is full)"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2604_13327_b200.etsim as etsim  # noqa: E402
from paper_2604_13327_b200.decode import CONFIGS, DecodeModel  # noqa: E402
from paper_2604_13327_b200.ops import pack  # noqa: E402

cfg = CONFIGS["llama3-8b"]
m = DecodeModel(cfg, samples=(1024,))
m.fill_cache(1024)
m.set_token(1)
ops = pack(m._ops())
for dbg in ("0", "64"):
    os.environ["ET_DEBUG"] = dbg
    for l2 in [int(x) for x in sys.argv[1:]] or [0, 65536, 131072, 262144, 524288, 1048576]:
        ex = etsim.Executor(m.kernel, num_workers=m.num_workers, record_trace=False, l2_prefetch=l2)
        ex.bind_ops(ops)
        ts = [ex.run({"s": 1024})["kernel_ms"] for _ in range(6)]
        print("debug", dbg, "l2_prefetch", l2, "median ms", round(statistics.median(ts[2:]), 4), flush=True)
        del ex

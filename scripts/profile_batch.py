"""A few batched decode steps (tensor-core path) for ncu captures (not a benchmark).

    python scripts/profile_batch.py [b] [s]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_13327_b200.batch import BatchDecodeModel  # noqa: E402
from paper_2604_13327_b200.decode import LLAMA3_8B  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 64
s = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
m = BatchDecodeModel(LLAMA3_8B, samples=(s,), max_batch=64)
m.fill_cache(s)
m.set_token([1 + 7 * i for i in range(b)])
for _ in range(4):
    st = m.executor.run({"s": s, "b": b})
print("kernel_ms", st["kernel_ms"], flush=True)

"""One batched decode step of the Llama-3-8B shape on the tensor-core path (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_13327_b200.batch import BatchDecodeModel  # noqa: E402
from paper_2604_13327_b200.decode import CONFIGS  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 1
m = BatchDecodeModel(CONFIGS["llama3-8b"], samples=(1024,), max_batch=64)
m.fill_cache(1024)
m.set_token(1)
for _ in range(3):
    m.step(1024, b)
torch.cuda.synchronize()

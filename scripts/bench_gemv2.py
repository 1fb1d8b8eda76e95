import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts.bench_gemv import run
for N, K, T in [(1024, 256, 8), (8192, 4096, 8), (8192, 4096, 148), (128256, 4096, 148)]:
    try:
        run(N, K, T, reps=3)
    except Exception as e:
        print("FAIL", N, K, T, e, flush=True)

import sys; sys.path.insert(0, '.')
from paper_2604_13327_b200.moe import TINY_MOE, MoEDecodeModel
for early in (False,):
    m = MoEDecodeModel(TINY_MOE, samples=(16, 64), num_workers=16, seed=0, scheduler="dynamic", record_trace=True)
    m.fill_cache(16, seed=2); m.set_token(3)
    try:
        m.step(16); print("ok")
    except Exception as e:
        print("ERR", e)
    for l in range(2):
        print(l, m.routing(l))
    print(m.executor.final_counters())

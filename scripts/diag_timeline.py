"""Per-stage critical path of one decode step (timing experiment, not a test).

    python scripts/diag_timeline.py [llama|moe] [layers...]

For each call of the chosen layers (trace of a normal step, %globaltimer per
slot): when its tasks' waits ended (first / median / last), how long their
bodies ran (median / max), when the last one notified; and the hop from the
previous stage's last notify to this stage's median wait end.
"""
import collections
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "llama"
    layers = [int(x) for x in sys.argv[2:]] or [1, 16]
    if which == "llama":
        from paper_2604_13327_b200.decode import LLAMA3_8B, DecodeModel
        m = DecodeModel(LLAMA3_8B, samples=(1024,), record_trace=True)
        m.fill_cache(1024)
        m.set_token(1)
        binding = {"s": 1024}
    else:
        from paper_2604_13327_b200.moe import MOE_CONFIGS, MoEDecodeModel
        sched = sys.argv[1].split("-")[1] if "-" in which else "static"
        mb = int(os.environ.get("MB", "1"))  # batch (MB > 8: the tensor-core instantiation)
        m = MoEDecodeModel(MOE_CONFIGS["qwen3-30b-a3b"], samples=(1024,), scheduler=sched.replace("early", "dynamic"),
                           early_push=sched == "early", record_trace=True, max_batch=mb)
        m.fill_cache(1024, seed=1)
        m.set_token([1 + 7 * i for i in range(mb)])
        binding = m._binding(1024, mb)
    ex = m.executor
    if os.environ.get("DIAG_DEBUG"):
        ex.set_debug(int(os.environ["DIAG_DEBUG"], 0))
    ts = [ex.run(binding)["kernel_ms"] for _ in range(6)]
    print("step ms", [round(t, 3) for t in ts])
    calls = m.graph.call_functions
    t = ex.trace()
    by = collections.defaultdict(list)
    for r in t.records:
        if not r["noop"]:
            by[r["call"]].append(r)
    t0 = min(r["exec"][0] for rs in by.values() for r in rs)
    t1 = max(r["exec"][1] for rs in by.values() for r in rs)
    print(f"trace span {(t1 - t0) / 1e3:.1f} us over {len(t.records)} records")
    for L in layers:
        cs = [c for c in range(len(calls)) if calls[c].startswith(f"L{L}.")]
        base = min(r["exec"][0] for c in cs for r in by[c])
        prev_end = None
        print(f"--- layer {L} (us from its first task start)")
        for c in cs + [c for c in range(len(calls)) if calls[c].startswith(f"L{L + 1}.")][:1]:
            rs = by[c]
            if not rs:
                continue
            st = sorted((r["exec"][0] - base) / 1e3 for r in rs)
            en = sorted((r["exec"][1] - base) / 1e3 for r in rs)
            du = sorted((r["exec"][1] - r["exec"][0]) / 1e3 for r in rs)
            pr = sorted(r["prologue"] / 1e3 for r in rs if r["prologue"] is not None)
            prs = f"pro {pr[len(pr) // 2]:5.2f}" if pr else "          "
            hop = f"hop(prev last end -> med start) {st[len(st) // 2] - prev_end:6.2f}" if prev_end is not None else ""
            print(f"{calls[c]:12s} n={len(rs):4d} start {st[0]:7.2f} / {st[len(st) // 2]:7.2f} / {st[-1]:7.2f}  "
                  f"dur med {du[len(du) // 2]:6.2f} max {du[-1]:6.2f} {prs} end med {en[len(en) // 2]:7.2f} "
                  f"max {en[-1]:7.2f}  {hop}")
            prev_end = en[-1]
    # per layer duration (first start of L.qkv to first start of L+1.qkv)
    firsts = []
    for L in range(200):
        cs = [c for c in range(len(calls)) if calls[c].startswith(f"L{L}.")]
        if not cs:
            break
        firsts.append(min(r["exec"][0] for c in cs for r in by[c]))
    d = [(b - a) / 1e3 for a, b in zip(firsts, firsts[1:])]
    print("layer us: med", round(statistics.median(d), 2), "min", round(min(d), 2), "max", round(max(d), 2))
    print("per-call median task dur over all layers (us):")
    agg = collections.defaultdict(list)
    for c, rs in by.items():
        key = calls[c].split(".")[-1] if "." in calls[c] else calls[c]
        agg[key] += [(r["exec"][1] - r["exec"][0]) / 1e3 for r in rs]
    for k, v in agg.items():
        v.sort()
        print(f"  {k:10s} n={len(v):6d} med {v[len(v) // 2]:7.2f} p90 {v[int(len(v) * .9)]:7.2f} max {v[-1]:7.2f}")


if __name__ == "__main__":
    main()

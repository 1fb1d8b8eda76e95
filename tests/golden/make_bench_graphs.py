"""Writes tests/golden/bench_graphs.json.gz: for every bench.py workload, the
graph this framework lowers (reference JSON spec), its bindings and scheduler.

bench.py --impl reference feeds these to the UNMODIFIED reference (oracle/_ref)
so the reference arm times the reference's own executor on exactly the graph
the GPU arm runs, without loading anything of this framework; the fixture is
pinned against the live layout functions by tests/test_bench_graphs.py.

    python tests/golden/make_bench_graphs.py
"""

import argparse
import gzip
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

WORKLOADS = (
    [("llama3-8b", 1, sch, 1024, 0) for sch in ("static", "dynamic")]
    + [("llama3-8b", 1, "static", s, 0) for s in (128, 4096, 8192)]
    + [("llama3-8b", b, "static", s, 0) for b in (8, 16, 32, 64) for s in (128, 1024, 8192)]
    + [("qwen3-30b-a3b", b, sch, 1024, 0) for b in (1, 8, 16, 32) for sch in ("static", "dynamic")]
    + [("llama3-70b", 1, "static", 1024, tp) for tp in (1, 2, 4, 8)]
)


def entry(config, batch, scheduler, seq, tp):
    args = argparse.Namespace(config=config, batch=batch, scheduler=scheduler, seq=seq, tp=tp)
    spec, bindings, binding, sched, rewrite, moe = bench.graph_for(args, world=max(1, tp))
    return {"spec": spec, "bindings": bindings, "binding": binding, "scheduler": sched, "rewrite": rewrite,
            "moe": moe, "num_sms": bench.NUM_SMS}


def build():
    return {bench.workload_key(*w): entry(*w) for w in WORKLOADS}


if __name__ == "__main__":
    out = build()
    with gzip.open(bench.FIXTURE, "wt") as f:
        json.dump(out, f, sort_keys=True)
    print("wrote", bench.FIXTURE, os.path.getsize(bench.FIXTURE), "bytes,", len(out), "workloads")

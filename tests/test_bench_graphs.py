"""The reference arm of bench.py times the reference's executor on the committed
graph fixtures (tests/golden/bench_graphs.json.gz).  These tests pin the fixture
to the graphs this framework lowers today, and run the reference arm once."""
import argparse
import gzip
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import bench  # noqa: E402
import make_bench_graphs  # noqa: E402


def _fixture():
    with gzip.open(bench.FIXTURE, "rt") as f:
        return json.load(f)


def test_fixture_is_the_lowered_graph():
    fx = _fixture()
    assert set(fx) == {bench.workload_key(*w) for w in make_bench_graphs.WORKLOADS}
    for w in make_bench_graphs.WORKLOADS:
        live = json.loads(json.dumps(make_bench_graphs.entry(*w)))
        assert fx[bench.workload_key(*w)] == live, w


def test_headline_fixture_matches_decode_model_spec():
    """The headline graph is DecodeModel's balanced / grouped / fused-merge spec."""
    from paper_2604_13327_b200.decode import LLAMA3_8B, decode_graph_spec

    spec, lay = decode_graph_spec(LLAMA3_8B, 148, 1024)
    assert lay["grouped"] and lay["call_tasks"] == {"qkv": 128, "gateup": 128}
    assert _fixture()["llama3-8b|b1|static|s1024|tp0"]["spec"] == json.loads(json.dumps(spec))


@pytest.mark.skipif(not os.path.isdir(os.path.join(ROOT, "oracle", "_ref", "etsim")), reason="oracle/_ref not built")
@pytest.mark.parametrize("argv", [[], ["--config", "qwen3-30b-a3b", "--scheduler", "dynamic", "--batch", "8"]])
def test_reference_arm_runs_the_reference_only(argv):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1"] + argv, capture_output=True, text=True, timeout=300,
                         env={k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE")})
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    d = line["cpu_baseline"]["detail"]
    assert d["reference_module"].startswith("oracle/_ref/") and d["final_counters_zero"]
    args = argparse.Namespace(config="llama3-8b", batch=1, scheduler="static", seq=1024, tp=0)
    for k, v in vars(args).items():
        if "--" + k in argv:
            setattr(args, k, type(v)(argv[argv.index("--" + k) + 1]))
    assert line["config"] == bench.config_dict(args, 1)

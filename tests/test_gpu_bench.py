"""The bench contract end to end on the GPU: the default run (extras included,
cpu_baseline skipped to stay short) prints one JSON line with every key the
driver and the judge read."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_default_line():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "2", "--warmup", "3", "--no-cpu-baseline"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks",
              "per_stage_roofline", "other_configs_and_next_rows"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["dtype"] == "f64"
    assert d["value"] > 0 and d["gpu_launches"] >= 2 * 12
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    ex = d["other_configs_and_next_rows"]
    for k in ("c1", "c2", "c3", "c3x16", "c5", "morton_256cubed", "product_c4xc4", "bie_product_2M"):
        assert k in ex, k


def test_bench_two_ranks_default_is_sharded():
    """`--gpus 2` on a single-RHS config defaults to one apply sharded by the top
    index bit: scaling "strong", sharded parallelism, the
    communicator's size in the line.  Two ranks share this box's one GPU over a
    gloo group (QTT_BENCH_DEVICE / QTT_DIST_BACKEND test hooks): a functional
    check of the path, not a scaling number."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, QTT_DIST_BACKEND="gloo", QTT_BENCH_DEVICE="0")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
                        "--steps", "2", "--warmup", "3", "--config", "c2", "--no-extra", "--no-cpu-baseline"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["parallelism"].startswith("top-bit shards x2")
    assert d["comm"]["world_size"] == 2
    assert d["value"] > 0 and d["gpu_launches"] > 0

"""bench.py host logic (-m "not gpu"): the per-stage roofline arithmetic and the
peak / traffic lookups the JSON line is assembled from."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_stage_table_single_and_merged():
    r = [1, 2, 4, 4, 1]                       # d = 4
    N, P, BW = 16, 1e12, 1e12
    stages = [{"k_first": 1, "k_last": 2, "variant": "merged"}, {"k_first": 3, "k_last": 3, "variant": "dmma"},
              {"k_first": 4, "k_last": 4, "variant": "dmma"}]
    rows, sT, st = bench.stage_table(stages, r, N, 1, [2.0, 1.0, 1.0], 2, P, BW)
    # stage 1-2: Alg. 2 flops 4 (1*2 + 2*4) N; executed 2^(L+1) r_in r_out N = 8 * 1 * 4 * N
    assert rows[0]["flops_alg2"] == 4 * (2 + 8) * N
    assert rows[0]["flops_executed"] == 8 * 4 * N
    assert rows[0]["ms"] == pytest.approx(1.0)          # 2.0 ms over 2 timed applies
    # single level: executed == Alg. 2; bytes 8 N (r_in + r_out) + 32 r_in r_out
    assert rows[1]["flops_executed"] == rows[1]["flops_alg2"] == 4 * 4 * 4 * N
    B = 8 * N * (4 + 4) + 32 * 16
    assert rows[1]["gbs"] == pytest.approx(B / 0.5e-3 / 1e9)
    T = max(4 * 16 * N / P, B / BW)
    assert rows[1]["roofline_frac"] == pytest.approx(T / 0.5e-3)
    assert st == pytest.approx(2e-3)


def test_peaks_from_measured_files():
    hbm, hbm_src, fp64, fp64_src = bench.load_peaks()
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")):
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            assert hbm == pytest.approx(float(json.load(f)["hbm_gbs"]))
        assert "measured" in hbm_src
    assert 30.0 < fp64 < 45.0                              # DMMA probe (37.08) or the nominal 37.2


def test_traffic_lookup_picks_latest_c4_summary():
    """The dominant kernel's traffic comes from the latest capture of THAT
    kernel shape (an r = 48 level, 4*48*48*N flops), not from another c4 stage
    captured in the same round."""
    level_flops = 4 * 48 * 48 * (1 << 24)
    tr = bench.load_traffic("c4", level_flops)
    assert tr is not None
    nbytes, name = tr
    assert 1.2e10 < nbytes < 1.4e10                        # one r = 48 level: ~12.9 GB
    import glob
    import re
    def key(n):
        m = re.match(r"r(\d+)([a-z]*)", n)
        return (int(m.group(1)), len(m.group(2)), m.group(2))
    c4 = [os.path.basename(p) for p in glob.glob(os.path.join(ROOT, "profiles", "*ncu_full*summary.json"))
          if json.load(open(p)).get("config") == "c4"
          and json.load(open(p)).get("algorithmic_flops_per_launch") == level_flops]
    assert name == max(c4, key=key)                       # the latest capture by round, then suffix


def test_reference_arm_line():
    """bench.py --impl reference (the oracle timed on host cores) prints the
    contract line: impl, metric/unit of our arm, cpu_baseline, e2e."""
    import subprocess
    import sys
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1",
                        "--config", "c3"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == bench.UNIT and d["metric"] == bench.METRIC
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    # every timed step is one whole apply (no extrapolation): ms_per_step is the
    # median measured step, and the timed steps fit in the measured wall time
    assert len(d["step_seconds"]) == 2
    assert d["ms_per_step"] * 1e-3 <= d["timed_wall_s"]
    assert "whole c3 apply" in d["cpu_baseline"]["sample"]
    # the same config dict our arm prints for the same arguments
    from qtt_workload.configs import make_config
    assert d["config"] == bench.config_desc(make_config("c3"), 1, "single GPU")
    assert d["scaling"] == "strong"      # single-RHS config: the multi-GPU mode is top-bit sharding


def test_multi_gpu_mode_defaults():
    import argparse
    a = argparse.Namespace(mode=None, exchange="nccl")
    assert bench.resolve_mode(a, 1) == "sharded"
    assert bench.resolve_mode(a, 16) == "replicas"
    a.mode = "replicas"
    assert bench.resolve_mode(a, 1) == "replicas"
    assert bench.parallelism_desc("sharded", 2) == "top-bit shards x2 + NCCL reduce-scatter"
    assert bench.parallelism_desc("sharded", 1) == "single GPU"
    assert bench.parallelism_desc("replicas", 4).startswith("replicas x4")


def test_reference_arm_under_torchrun_uses_all_cores():
    """Under torchrun (OMP_NUM_THREADS=1 per worker) rank 0 alone runs the oracle
    and prints the line, on all host cores; rank 1 exits without work."""
    import socket
    import subprocess
    import sys
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "3", "--config", "c2"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"
    assert d["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))

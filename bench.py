#!/usr/bin/env python
"""Benchmark: QTT apply y = A x in fp64 on B200 (Alg. 2).

Workload (BASELINE.json metric): config c4, N = 2^24 (256^3 volume grid), tapered
rank profile r_k = min(2^k, 2^(24-k), 48), one RHS x ~ U[-1,1), seed 0.
A "step" is one full apply (all d = 24 levels) over one input vector that is
resident in HBM.  Every buffer exceeds L2 (x 128 MiB; intermediates up to
6.4 GB), so no L2 flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl reference]

Multi-GPU (--gpus N, launched by torchrun): for a single-RHS config (c4) one
apply is sharded over the N GPUs by the top index bits with one NCCL
reduce-scatter (strong scaling); multi-RHS configs
(or --mode replicas) run N independent replicas (weak scaling, no data-path
collective).  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "QTT apply fp64 GFLOP/s, ms/apply and % of per-stage roofline at N=2^24 on 1 B200"
UNIT = "GFLOP/s"
HBM_FALLBACK_GBS = 6650.0        # B200_PROFILING.md fallback (used only if MEASURED_PEAKS.json is absent)
FP64_NOMINAL_TFLOPS = 37.2       # 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz


# --------------------------------------------------------------------------- peaks
def load_peaks():
    hbm, hbm_src = HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            hbm = float(json.load(f)["hbm_gbs"])
        hbm_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    fp64, fp64_src = FP64_NOMINAL_TFLOPS, "nominal"
    q = os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")
    if os.path.exists(q):
        with open(q) as f:
            d = json.load(f)
        vals = [v for k, v in d.items() if k.startswith("dmma_")]
        if vals:
            fp64, fp64_src = max(vals), "measured (profiles/r01_fp64_peaks.json, DMMA burst)"
    return hbm, hbm_src, fp64, fp64_src


def load_traffic(config, flops=None):
    """dram read+write bytes per launch of the dominant kernel from the committed
    ncu --set full capture summary (profiles/*_ncu_full_summary.json), or None.
    With `flops`, only a summary of a launch of that many algorithmic flops
    (the dominant kernel's shape, not another stage of the same config) counts."""
    import glob
    best = None
    # tags r<round><suffix>, suffixes a .. z, aa, ab, ...: latest round, then latest suffix wins
    def tag_key(path):
        import re
        m = re.match(r"r(\d+)([a-z]*)", os.path.basename(path))
        return (int(m.group(1)), len(m.group(2)), m.group(2)) if m else (-1, 0, "")
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu_full*summary.json")), key=tag_key):
        try:
            with open(p) as f:
                d = json.load(f)
            if flops is not None and d.get("algorithmic_flops_per_launch") != flops:
                continue
            if d.get("config") == config and d.get("dram_bytes_per_launch"):
                best = (float(d["dram_bytes_per_launch"]), os.path.basename(p))
        except Exception:
            pass
    return best


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.05)
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 8:
                self.rows.append(parts)

    def summary(self):
        rows = getattr(self, "rows", [])
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        pw = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        # "under load": samples within 25% of the busiest clock seen
        load = [s for s in sm if s >= 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None,
                "samples": len(rows), "reasons": reasons}


# --------------------------------------------------------------------------- distributed plumbing
def dist_setup(n_gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: several ranks on one GPU (gloo barriers only; no kernel waits on another rank)
    if os.environ.get("QTT_BENCH_DEVICE") is not None:
        local = int(os.environ["QTT_BENCH_DEVICE"])
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("QTT_DIST_BACKEND", "nccl")
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world, rank, local


def dist_max(value: float, world: int, device=None) -> float:
    """Max over ranks (device-timed numbers are reduced, never wall clock)."""
    if world <= 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# --------------------------------------------------------------------------- helpers
def resolve_mode(args, nrhs: int) -> str:
    """Multi-GPU mode: one apply sharded by the top index bits (SURVEY 8(e),
    strong scaling) for single-RHS configs, independent replicas otherwise;
    --mode overrides."""
    if args.mode is not None:
        return args.mode
    return "sharded" if nrhs == 1 else "replicas"


def parallelism_desc(mode: str, world: int, exchange: str = "nccl") -> str:
    if world <= 1:
        return "single GPU"
    if mode == "sharded":
        return (f"top-bit shards x{world} + "
                + ("fused peer-store exchange" if exchange == "fused" else "NCCL reduce-scatter"))
    return f"replicas x{world} (independent problems, no data-path collective)"


def config_desc(cfg, nrhs, parallelism="single GPU"):
    """The workload description; both arms (ours and --impl reference) print
    exactly this dict for the same arguments."""
    prof = "tapered r_k=min(2^k,2^(d-k),48)" if cfg.name == "c4" else f"r={max(cfg.ranks)}"
    return {"workload": f"{cfg.name}: QTT apply d={cfg.d} N=2^{cfg.d} {prof}, nrhs={nrhs}, seed {cfg.seed}",
            "d": cfg.d, "N": cfg.N, "nrhs": nrhs, "max_rank": max(cfg.ranks),
            "x_dist": cfg.x_dist, "stands_for": cfg.stands_for,
            "l2": "no flush: inputs larger than L2 (x %d MiB, intermediates up to %.1f GB)"
                  % (cfg.N * nrhs * 8 >> 20, max(cfg.ranks[1:-1] or [1]) * cfg.N * nrhs * 8 / 1e9),
            "parallelism": parallelism}


# host buffers of the oracle's sweep above this size switch it to the chunked
# variant (top-bit blocks; same result, SURVEY 8(c) oracle 4): c5 only
ORACLE_BUFFER_LIMIT = 8 << 30


def oracle_whole_apply(cores, x, cfg):
    """One whole apply by the CPU oracle, as it stands: Alg. 2 with BLAS calls
    (oracle.apply_blas_sweep, SURVEY 8(c) oracle 3), or its chunked form when
    one intermediate buffer would exceed ORACLE_BUFFER_LIMIT.  Returns
    (seconds, description)."""
    import oracle
    rmax = max(cfg.ranks)
    s = 0
    while (cfg.N >> s) * rmax * 8 > ORACLE_BUFFER_LIMIT:
        s += 1
    t0 = time.perf_counter()
    if s == 0:
        oracle.apply_blas_sweep(cores, x)
        what = "oracle.apply_blas_sweep (Alg. 2, two numpy matmul(out=half) per level)"
    else:
        oracle.apply_chunked(cores, x, s)
        what = f"oracle.apply_chunked (Alg. 2 BLAS sweep per 2^{s} top-bit blocks + projections)"
    return time.perf_counter() - t0, what


def oracle_warm_sample(cores, x, cfg, s_bits=3):
    """Untimed warm-up of the oracle: Alg. 2 levels 1..d-s on the first of 2^s
    top-bit blocks of x (these levels never mix blocks)."""
    import oracle
    n = cfg.N >> s_bits
    oracle.blas_sweep(cores[: cfg.d - s_bits], x[0, :n])


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max((i.get("num_threads", 1) for i in info), default=1), [i.get("internal_api") for i in info]
    except Exception:
        return os.cpu_count() or 1, []


def run_cpu_baseline(cfg, cores, x):
    """Time the oracle (as it stands) on ONE WHOLE APPLY of the workload (all d
    levels, every entry of x; ~10-20 s of CPU work at c4): no sampling and no
    extrapolation."""
    dt, what = oracle_whole_apply(cores, x, cfg)
    F = 4 * sum(cfg.ranks[k] * cfg.ranks[k + 1] for k in range(cfg.d)) * cfg.N * cfg.nrhs
    threads, apis = blas_threads()
    return {"value": F / dt / 1e9, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"one whole {cfg.name} apply ({F / 1e9:.0f} GFLOP, all {cfg.d} levels, {cfg.N} x "
                      f"{cfg.nrhs} entries): {what}, {dt:.2f} s",
            "seconds": dt, "ms_per_apply": dt * 1e3, "blas": apis, "host_cpus": os.cpu_count(),
            "affinity_cpus": _affinity(), "cpu_model": _cpu_model()}


def small_config_oracle_ms(threads=None):
    """cpu_baseline leg: the same oracle timed on c1, c2, c3 (whole applies);
    threads=1 limits BLAS to one thread (comparable to the
    paper's serial Xeon)."""
    import contextlib
    import oracle
    from qtt_workload import generate
    ctx = contextlib.nullcontext()
    if threads is not None:
        try:
            from threadpoolctl import threadpool_limits
            ctx = threadpool_limits(limits=threads)
        except Exception:
            return None
    out = {}
    with ctx:
        for name in ("c1", "c2", "c3"):
            _, cores, x = generate(name)
            oracle.apply_blas_sweep(cores, x)            # warm-up
            ts = []
            for _ in range(3 if name != "c3" else 1):
                t0 = time.perf_counter()
                oracle.apply_blas_sweep(cores, x)
                ts.append((time.perf_counter() - t0) * 1e3)
            out[name] = statistics.median(ts)
    return out


def _affinity():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return None


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def stage_table(stages, r, N, nrhs, stage_ms, n_timed, P, BW):
    """Per-stage roofline rows: T_s = max(F_s/P, B_s/BW) with F_s the
    Alg. 2 flops of the stage's levels and B_s its HBM bytes; also the executed-flop basis."""
    stage_rows = []
    sum_T, sum_t = 0.0, 0.0
    for s, st in enumerate(stages):
        k0, k1 = st["k_first"], st["k_last"]
        F = sum(4 * r[k - 1] * r[k] for k in range(k0, k1 + 1)) * N * nrhs
        B = 8 * N * nrhs * (r[k0 - 1] + r[k1]) + 32 * sum(r[k - 1] * r[k] for k in range(k0, k1 + 1))
        # flops the kernel actually executes (unpadded): a merged stage of L levels
        # applies the 2^L r_in x 2^L r_out super-core, 2^(L+1) r_in r_out per element
        F_exec = (2 ** (k1 - k0 + 2)) * r[k0 - 1] * r[k1] * N * nrhs if k1 > k0 else F
        if st["variant"] == "diag":        # block-diagonal digits: one batched GEMV, 2 r_in r_out per element
            F_exec = 2 * r[k0 - 1] * r[k1] * N * nrhs
        t = stage_ms[s] / max(n_timed, 1) * 1e-3
        T = max(F / P, B / BW)
        sum_T += T
        sum_t += t
        stage_rows.append({"levels": [k0, k1], "ranks": [r[k0 - 1], r[k1]], "variant": st["variant"],
                           "ms": t * 1e3, "gflops": F / t / 1e9 if t else None,
                           "gbs": B / t / 1e9 if t else None, "roofline_frac": T / t if t else None,
                           "flops_alg2": F, "flops_executed": F_exec,
                           "roofline_frac_executed": max(F_exec / P, B / BW) / t if t else None})
    return stage_rows, sum_T, sum_t


def time_applies(fn, steps, warmup, stream):
    """(ms per call over `steps` back-to-back calls, min ms of a single call), CUDA
    events on `stream`.  The batch figure keeps the device busy (host enqueue runs
    ahead); the single-call figure includes the host's launch latency."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        fn()
    b.record(stream)
    b.synchronize()
    batch = a.elapsed_time(b) / steps
    single = []
    for _ in range(min(steps, 5)):
        torch.cuda.synchronize()
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        single.append(a.elapsed_time(b))
    return batch, min(single)


def op_flops_c4(cfg):
    return 4 * sum(cfg.ranks[k] * cfg.ranks[k + 1] for k in range(cfg.d)) * cfg.N


def extra_measurements(dev, stream, P, BW, max_stage_levels=None):
    """The other BASELINE configs and the NEXT rows, timed after the headline
    (not part of `value`): per config ms/apply, Alg. 2 and executed rates and
    per-stage roofline fractions; Morton pack/unpack GB/s at 256^3; the product
    X = M Y of two c4-profile operators; the grid apply at 256^3."""
    import torch
    import paper_1511_06029_b200 as q
    from qtt_workload import generate
    out = {}
    for name in ("c1", "c2", "c3", "c3x16", "c5"):
        cfg, cores, x_np = generate(name)
        with q.QttOperator(cores, max_stage_levels=max_stage_levels) as op:
            x = torch.from_numpy(x_np).to(dev)
            y = torch.empty_like(x)
            ws = None
            reps = 5 if name == "c5" else (200 if name in ("c1", "c2") else 20)
            # the default user path: qtt_apply on the handle's cached workspace
            fn = lambda: op.apply(x, out=y, stream=stream)
            med, mn = time_applies(fn, reps, 3, stream)
            apply_plan = op.stages(cfg.nrhs)
            launches = op.launches(cfg.nrhs)
            # per-stage times: stage timing runs (and reports) the per-stage launches
            op.set_stage_timing(True)
            op.stage_times()
            timed_stages = op.stages(cfg.nrhs)
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            op.set_stage_timing(False)
            sms, nt = op.stage_times()
            rows, sT, st_ = stage_table(timed_stages, cfg.ranks, cfg.N, cfg.nrhs, sms, nt, P, BW)
            F = op.flops_per_rhs * cfg.nrhs
            Fx = sum(rr["flops_executed"] for rr in rows)
            if apply_plan and apply_plan[0]["variant"] == "fused":
                Lf = [a_["k_last"] - a_["k_first"] + 1 for a_ in apply_plan]
                Fx = sum(2 ** (L_ + 1) * cfg.ranks[a_["k_first"] - 1] * cfg.ranks[a_["k_last"]] * cfg.N * cfg.nrhs
                         for L_, a_ in zip(Lf, apply_plan))
            if name in ("c1", "c2"):
                # latency-bound sizes: the device time of an apply without host
                # launch gaps -- 100 applies captured in one CUDA graph, replayed
                g = torch.cuda.CUDAGraph()
                cap = torch.cuda.Stream(dev)           # capture needs a non-default stream
                torch.cuda.synchronize()
                with torch.cuda.graph(g, stream=cap):
                    for _ in range(100):
                        op.apply(x, out=y)
                with torch.cuda.stream(cap):
                    g.replay()
                torch.cuda.synchronize()
                ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                best = None
                for _ in range(3):
                    ga.record(cap)
                    with torch.cuda.stream(cap):
                        g.replay()
                    gb.record(cap)
                    gb.synchronize()
                    t_ = ga.elapsed_time(gb) / 100
                    best = t_ if best is None else min(best, t_)
                del g
                in_graph = {"ms_per_apply_in_graph": best,
                            "in_graph_note": "100 applies captured in one CUDA graph (device time without host launch gaps)"}
            else:
                in_graph = {}
            out[name] = {"ms_per_apply": med, "ms_single_call_min": mn, **in_graph,
                         "gflops_alg2": F / (med * 1e-3) / 1e9,
                         "tflops_executed": Fx / (med * 1e-3) / 1e12, "launches": launches,
                         "apply_plan": [[a_["k_first"], a_["k_last"], a_["variant"]] for a_ in apply_plan],
                         "per_stage_note": "per-stage rows below: the per-stage launches stage timing runs",
                         "per_stage_frac": sT / st_ if st_ else None,
                         "per_stage_frac_executed": sum(
                             max(rr["flops_executed"] / P, (8 * cfg.N * cfg.nrhs * (rr["ranks"][0] + rr["ranks"][1])) / BW)
                             for rr in rows) / st_ if st_ else None,
                         "stages": [[rr["levels"][0], rr["levels"][1], rr["variant"], round(rr["ms"], 4),
                                     round(rr["roofline_frac_executed"] or 0, 3)] for rr in rows],
                         "sum_stage_ms": sum(rr["ms"] for rr in rows)}
            del x, y, ws
        torch.cuda.empty_cache()
    # NEXT-2: Morton pack / unpack at 256^3 (16 bytes moved per element), on a
    # side stream, 50 back-to-back calls (host enqueue ~9 us < kernel ~50 us)
    N = 1 << 24
    g = torch.randn(N, dtype=torch.float64, device=dev)
    xq = torch.empty((1, N), dtype=torch.float64, device=dev)
    gb = torch.empty_like(xq)
    ms_ = torch.cuda.Stream(dev)
    with torch.cuda.stream(ms_):
        mp, _ = time_applies(lambda: q.morton_pack(g, 3, 8, out=xq, stream=ms_), 50, 5, ms_)
        mu, _ = time_applies(lambda: q.morton_unpack(xq, 3, 8, out=gb, stream=ms_), 50, 5, ms_)
    out["morton_256cubed"] = {"pack_ms": mp, "unpack_ms": mu, "pack_gbs": 16 * N / (mp * 1e-3) / 1e9,
                              "unpack_gbs": 16 * N / (mu * 1e-3) / 1e9,
                              "pack_frac_hbm": 16 * N / (mp * 1e-3) / BW, "unpack_frac_hbm": 16 * N / (mu * 1e-3) / BW}
    del g, xq, gb
    # NEXT-4a: large constant ranks (wide kernel, streamed super-cores)
    from qtt_workload import random_case
    for d_, r_ in ((20, 128), (18, 256)):
        ranks = [1] + [r_] * (d_ - 1) + [1]
        _, cores, x_np = random_case(4242, d_, r_, 1, ranks=ranks)
        with q.QttOperator(cores) as op:
            x = torch.from_numpy(x_np).to(dev)
            y = torch.empty_like(x)
            ws = torch.empty(op.workspace_size(1) // 8 + 64, dtype=torch.float64, device=dev)
            med, _ = time_applies(lambda: op.apply(x, out=y, workspace=ws, stream=stream), 5, 2, stream)
            st_ = op.stages()
            rows, _, _ = stage_table(st_, ranks, 1 << d_, 1, [1.0] * len(st_), 1, P, BW)
            Fx = sum(rr["flops_executed"] for rr in rows)
            out[f"rank{r_}_d{d_}"] = {"ms_per_apply": med, "gflops_alg2": op.flops_per_rhs / (med * 1e-3) / 1e9,
                                      "tflops_executed": Fx / (med * 1e-3) / 1e12,
                                      "frac_executed_fp64": Fx / (med * 1e-3) / P,
                                      "stages": [[a["k_first"], a["k_last"], a["variant"]] for a in st_]}
            del x, y, ws
    # NEXT-3: compressed matvec (c4 operator x rank-4 TT vector) + GPU densify; the call synchronizes
    from qtt_workload import random_tt_vector
    _, cA, _ = generate("c4", with_x=False)
    _, bv = random_tt_vector(11, 24, 4)
    with q.QttOperator(cA) as A:
        c = torch.empty(1 << 24, dtype=torch.float64, device=dev)
        A.compressed_matvec(bv, out=c, stream=stream)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            A.compressed_matvec(bv, out=c, stream=stream)
            ts.append((time.perf_counter() - t0) * 1e3)
        out["compressed_c4_x_rank4"] = {"ms_wall_median": statistics.median(ts),
                                        "note": "host wall time of the synchronous call: b cores H2D, "
                                                "product cores, GPU densify of the 2^24-entry result"}
        del c
    # SPEC acceptance #9: apply time ~ N log N -- fit the exponent of
    # time vs N at constant rank 16 over d = 18..24 (per level it is ~N^1)
    ts, ns = [], []
    for d_ in (18, 20, 22, 24):
        ranks = [1] + [16] * (d_ - 1) + [1]
        _, cores, x_np = random_case(77, d_, 16, 1, ranks=ranks)
        with q.QttOperator(cores) as op:
            x = torch.from_numpy(x_np).to(dev)
            y = torch.empty_like(x)
            ms, _ = time_applies(lambda: op.apply(x, out=y, stream=stream), 10, 3, stream)
        ts.append(ms)
        ns.append(1 << d_)
    slope = float(np.polyfit(np.log(ns), np.log(ts), 1)[0])
    out["time_vs_N_rank16"] = {"d": [18, 20, 22, 24], "ms": ts, "loglog_slope": slope,
                               "note": "Alg. 2 is O(r^2 N log N); slope ~1 (log factor + fixed launch costs)"}
    # B12: same-box library comparator -- Alg. 2 level by level on
    # the same rotating layout with two cuBLAS DGEMMs per level (one per output
    # half i_k), through torch.matmul; and cuBLAS DGEMM 8192^3 as the library's
    # FP64 ceiling on this box.  Not the product; a number to beat.
    cfg4, c4cores, x4 = generate("c4")
    N4 = cfg4.N
    rmax = max(cfg4.ranks)
    bufs = [torch.empty(N4 * rmax, dtype=torch.float64, device=dev) for _ in range(2)]
    xg = torch.from_numpy(x4).to(dev).view(-1)
    Bs = []
    for k, G in enumerate(c4cores):
        ri, ro = G.shape[0], G.shape[3]
        Gt = torch.from_numpy(np.ascontiguousarray(G)).to(dev)            # [a][i][j][b]
        # Bmat_i[j*ri + a][b] = G[a, i, j, b]
        Bs.append([Gt[:, i, :, :].permute(1, 0, 2).reshape(2 * ri, ro).contiguous() for i in range(2)])

    def cublas_apply():
        src = xg
        for k, G in enumerate(c4cores):
            ri, ro = G.shape[0], G.shape[3]
            A = src[: N4 * ri].view(N4 // 2, 2 * ri)
            dst = bufs[k & 1][: N4 * ro].view(2, N4 // 2, ro)
            for i in range(2):
                torch.matmul(A, Bs[k][i], out=dst[i])
            src = bufs[k & 1][: N4 * ro]
        return src
    cb_ms, _ = time_applies(cublas_apply, 3, 1, stream)
    yk = cublas_apply()[:N4].clone()
    a8 = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    b8 = torch.randn_like(a8)
    c8 = torch.empty_like(a8)
    gemm_ms, _ = time_applies(lambda: torch.matmul(a8, b8, out=c8), 3, 1, stream)
    with q.QttOperator(c4cores) as A4:
        yq = A4.apply(xg.view(1, -1)).view(-1)
    rel = float((yq - yk).norm() / yk.norm())
    out["cublas_comparator"] = {
        "c4_alg2_two_dgemm_per_level_ms": cb_ms,
        "c4_alg2_gflops": op_flops_c4(cfg4) / (cb_ms * 1e-3) / 1e9,
        "rel_l2_vs_library_apply": rel,
        "dgemm_8192_tflops": 2 * 8192 ** 3 / (gemm_ms * 1e-3) / 1e12,
        "note": "torch.matmul fp64 (cuBLAS DGEMM) on the same rotating layout as the library's level kernel"}
    del bufs, xg, Bs, a8, b8, c8, yk, yq
    torch.cuda.empty_cache()
    # NEXT-4 top-bit shards, emulated on this one GPU: the local kernel time of each
    # part's shard plan (levels 1..d-s on its block + projection) for c4 at P = 2, 4, 8
    from paper_1511_06029_b200 import parallel as par
    _, c4c, x4s = generate("c4")
    xs_full = torch.from_numpy(x4s).to(dev)
    shard_out = {}
    for s_ in (1, 2, 3):
        P_ = 1 << s_
        per = []
        for g_ in range(P_):
            with par.QttShard(c4c, s_, g_) as sh:
                xb = par.block_of(xs_full, g_, P_).contiguous()
                send = torch.empty((1, P_, sh.n), dtype=torch.float64, device=dev)
                ws_ = torch.empty(sh.workspace_size(1) // 8 + 64, dtype=torch.float64, device=dev)
                ms_g, _ = time_applies(lambda: sh.apply(xb, send=send, workspace=ws_, stream=stream), 3, 1, stream)
                per.append(ms_g)
                del xb, send, ws_
        xfer = (P_ - 1) / P_ * (1 << 24) * 8 / 770e9 * 1e3      # reduce-scatter bytes / measured NVLink 770 GB/s
        shard_out[f"P{P_}"] = {"local_ms_max": max(per), "local_ms_mean": sum(per) / P_,
                               "exchange_ms_est": xfer, "projected_ms": max(per) + xfer,
                               "projected_speedup_vs_1gpu": None}
    out["sharded_c4_emulated"] = shard_out
    del xs_full
    torch.cuda.empty_cache()
    # NEXT-1: product of two c4-profile operators, and the grid apply
    _, cM, xg = generate("c4")
    _, cY, _ = generate("c4", seed=1, with_x=False)
    with q.QttOperator(cM) as M, q.QttOperator(cY) as Y, q.QttProduct([M, Y]) as PR:
        x = torch.from_numpy(xg).to(dev)
        y = torch.empty_like(x)
        ws = torch.empty(PR.workspace_size(1) // 8 + 64, dtype=torch.float64, device=dev)
        pm, _ = time_applies(lambda: PR.apply(x, out=y, workspace=ws, stream=stream), 5, 2, stream)
        F = M.flops_per_rhs + Y.flops_per_rhs
        out["product_c4xc4"] = {"ms_per_apply": pm, "gflops_alg2": F / (pm * 1e-3) / 1e9}
        gm, _ = time_applies(lambda: M.apply_grid(x, 3, out=y, stream=stream), 5, 2, stream)
        out["grid_apply_c4"] = {"ms_per_apply": gm, "gflops_alg2": M.flops_per_rhs / (gm * 1e-3) / 1e9}
        del x, y, ws
    # grid apply at the latency-bound sizes (16^3, 32^3): the fused apply gathers /
    # scatters the Morton order in its first / last stage, against the plain apply
    for name in ("c1", "c2"):
        cfg_, cores_, xg_ = generate(name)
        with q.QttOperator(cores_) as op_:
            x_ = torch.from_numpy(xg_).to(dev)
            y_ = torch.empty_like(x_)
            pa, _ = time_applies(lambda: op_.apply(x_, out=y_, stream=stream), 200, 10, stream)
            ga, _ = time_applies(lambda: op_.apply_grid(x_, 3, out=y_, stream=stream), 200, 10, stream)
            out[f"grid_apply_{name}"] = {"us_per_apply": ga * 1e3, "plain_apply_us": pa * 1e3,
                                         "launches": op_.launches(1),
                                         "note": "natural-order 3-D grid in and out (Morton pack/unpack "
                                                 "inside the one fused launch)" if op_.launches(1) == 1 else
                                                 "Morton pack + stages + unpack"}
    # boundary-integral preconditioner shape (Table 3's largest case, qtt_workload.bie_case):
    # X = M Y, N = 2^21 = 4096 surfaces x 512 points, Y ranks <= 95, block-diagonal M ranks <= 50
    from qtt_workload import bie_case
    rmb, cMb, ryb, cYb, xb = bie_case(0, 21, 9, 95, 50, 1)
    with q.QttOperator(cMb) as M, q.QttOperator(cYb) as Y, q.QttProduct([M, Y]) as PR:
        x = torch.from_numpy(xb).to(dev)
        y = torch.empty_like(x)
        ws = torch.empty(PR.workspace_size(1) // 8 + 64, dtype=torch.float64, device=dev)
        pm, _ = time_applies(lambda: PR.apply(x, out=y, workspace=ws, stream=stream), 10, 3, stream)
        ym, _ = time_applies(lambda: Y.apply(x, out=y, stream=stream), 10, 3, stream)
        F = M.flops_per_rhs + Y.flops_per_rhs
        Fx = 0.0
        for op_, rr_ in ((M, rmb), (Y, ryb)):
            rows_, _, _ = stage_table(op_.stages(), rr_, 1 << 21, 1, [1.0] * op_.launches_per_apply, 1, P, BW)
            Fx += sum(r_["flops_executed"] for r_ in rows_)
        out["bie_product_2M"] = {
            "ms_per_apply": pm, "ms_Y_alone": ym, "gflops_alg2": F / (pm * 1e-3) / 1e9,
            "tflops_executed": Fx / (pm * 1e-3) / 1e12, "frac_executed_fp64": Fx / (pm * 1e-3) / P,
            "stages_M": [[a["k_first"], a["k_last"], a["variant"], a["ksplit"]] for a in M.stages()],
            "stages_Y": [[a["k_first"], a["k_last"], a["variant"], a["ksplit"]] for a in Y.stages()],
            "note": "synthetic stand-in for Table 3 (N=1,966,080 padded to 2^21; paper's M/Y ranks 50/95)"}
        del x, y, ws
    torch.cuda.empty_cache()
    return out


# --------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference arm: the CPU oracle as it stands (no reference code exists;
    the paper ships none), on the host cores of rank 0.  Every timed step is
    one WHOLE apply of the workload (oracle_whole_apply); warm-up steps run a
    1/8 top-bit sample (untimed).  Under torchrun only rank 0 runs."""
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from qtt_workload import generate
    cfg, cores, x = generate(args.config)
    nrhs = cfg.nrhs
    # torchrun sets OMP_NUM_THREADS=1 for every worker; rank 0 runs the oracle
    # alone, on all of the host's cores
    import contextlib
    try:
        from threadpoolctl import threadpool_limits
        blas_ctx = threadpool_limits(limits=_affinity() or os.cpu_count() or 1)
    except Exception:
        blas_ctx = contextlib.nullcontext()
    with blas_ctx:
        return _run_reference_timed(args, world, cfg, cores, x, nrhs)


def _run_reference_timed(args, world, cfg, cores, x, nrhs):
    for _ in range(args.warmup):
        oracle_warm_sample(cores, x, cfg)
    secs = []
    what = None
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        dt, what = oracle_whole_apply(cores, x, cfg)
        secs.append(dt)
    wall = time.perf_counter() - wall0
    total_flops = 4 * sum(cfg.ranks[k] * cfg.ranks[k + 1] for k in range(cfg.d)) * cfg.N * nrhs
    ms_step = statistics.median(secs) * 1e3
    v = total_flops / (ms_step * 1e-3) / 1e9
    threads, _ = blas_threads()
    mode = resolve_mode(args, nrhs)
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
           "higher_is_better": True, "scaling": "strong" if mode == "sharded" else "weak",
           "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded; random cores with the config's rank profile stand in for the paper's inverse cores)",
           "config": config_desc(cfg, nrhs, parallelism_desc(mode, world, args.exchange)),
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                            "sample": f"every timed step is one whole {cfg.name} apply: {what}; "
                                      f"warm-up steps: levels 1..{cfg.d - 3} on 1/8 of x (untimed)"},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "timed_wall_s": wall, "step_seconds": secs,
           "note": "the oracle runs on rank 0's host cores only; ms_per_step is the median measured whole apply"}
    print(json.dumps(out))
    return 0


# --------------------------------------------------------------------------- our arm
def comm_info(world: int):
    """The communicator the data-path collective runs on (checkable: its size
    must equal n_gpus)."""
    if world <= 1:
        return None
    import torch.distributed as dist
    info = {"backend": dist.get_backend(), "world_size": dist.get_world_size()}
    try:
        import torch
        if info["backend"] == "nccl":
            info["nccl_version"] = ".".join(str(v) for v in torch.cuda.nccl.version())
    except Exception:
        pass
    return info


def run_sharded(args, world, rank, local, dev, cfg, cores, x_np):
    """One apply of the config sharded over `world` GPUs by the top index bits:
    each rank runs its shard plan on its block, then one sum reduce-scatter
    (NCCL).  value = Alg. 2 flops of the whole apply / max-over-ranks time."""
    import torch
    from paper_1511_06029_b200 import parallel as par
    nrhs = cfg.nrhs
    op = par.ShardedQttOperator(cores, fused=(args.exchange == "fused"), max_nrhs=nrhs)
    xb = torch.from_numpy(np.ascontiguousarray(par.block_of(x_np, rank, world))).to(dev)
    send = torch.empty((nrhs, world, op.n), dtype=torch.float64, device=dev)
    yb = torch.empty((nrhs, op.n), dtype=torch.float64, device=dev)
    ws = torch.empty(op.workspace_size(nrhs) // 8 + 64, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    step = lambda: op.apply(xb, out=yb, workspace=ws, send=send, stream=stream)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        dist_barrier(world)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        dist_barrier(world)
    ms_total = dist_max(e0.elapsed_time(e1), world, dev)
    ms_step = ms_total / args.steps
    flops = op.flops_per_rhs * nrhs
    # e2e: this rank's block H2D, sharded apply, block D2H
    xh = torch.from_numpy(np.ascontiguousarray(par.block_of(x_np, rank, world))).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    dist_barrier(world)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.e2e_steps):
        xb.copy_(xh, non_blocking=True)
        step()
        yh.copy_(yb, non_blocking=True)
    t1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = dist_max(t0.elapsed_time(t1), world, dev) / args.e2e_steps
    out = {"metric": METRIC, "value": flops * args.steps / (ms_total * 1e-3) / 1e9, "unit": UNIT,
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded; random cores with the config's rank profile)",
           "config": config_desc(cfg, nrhs, parallelism_desc("sharded", world, args.exchange)),
           "comm": comm_info(world),
           "e2e": {"value": flops / (e2e_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": e2e_ms,
                   "h2d_bytes_per_step": int(xh.numel() * 8), "d2h_bytes_per_step": int(yh.numel() * 8)},
           # stages (+ split-K reduce launches), + the slot reduction of the fused exchange
           "gpu_launches": (sum(1 + (st_.get("ksplit", 1) > 1) for st_ in op._shard.stages())
                            + (1 if args.exchange == "fused" else 0)) * args.steps,
           "clocks": clk.summary()}
    if rank == 0:
        print(json.dumps(out))
    op.close()
    import torch.distributed as dist
    dist.destroy_process_group()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=20.0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-extra", action="store_true", help="skip the other configs / NEXT-row measurements")
    ap.add_argument("--max-stage-levels", type=int, default=None,
                    help="cap on levels per launch (1 = Alg. 2 level by level); default: the library's")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "fused"],
                    help="sharded mode: NCCL reduce-scatter of a send buffer, or the fused projection "
                         "storing into the other GPUs' receive buffers (CUDA IPC over NVLink)")
    ap.add_argument("--mode", default=None, choices=["replicas", "sharded"],
                    help="N>1: one apply sharded by the top index bits with one NCCL reduce-scatter "
                         "(strong scaling; DESIGN.md 9; the default for single-RHS configs) or independent "
                         "replicas (weak scaling; the default for multi-RHS configs)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    world, rank, local = dist_setup(args.gpus)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    import paper_1511_06029_b200 as q
    from qtt_workload import generate

    cfg, cores, x_np = generate(args.config)
    nrhs = cfg.nrhs
    mode = resolve_mode(args, nrhs)
    if mode == "sharded" and world > 1:
        return run_sharded(args, world, rank, local, dev, cfg, cores, x_np)
    op = q.QttOperator(cores, max_stage_levels=args.max_stage_levels)
    x = torch.from_numpy(x_np).to(dev)
    y = torch.empty_like(x)
    ws = torch.empty(max(op.workspace_size(nrhs), 8) // 8 + 64, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    flops_step = op.flops_per_rhs * nrhs

    for _ in range(args.warmup):
        op.apply(x, out=y, workspace=ws, stream=stream)
    torch.cuda.synchronize(dev)

    op.set_stage_timing(True)
    op.stage_times()                      # reset accumulators
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        dist_barrier(world)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(args.steps):
            op.apply(x, out=y, workspace=ws, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        dist_barrier(world)
    op.set_stage_timing(False)
    ms_local = e0.elapsed_time(e1)
    stage_ms, n_timed = op.stage_times()
    ms_total = dist_max(ms_local, world, dev)
    ms_step = ms_total / args.steps
    value = flops_step * world * args.steps / (ms_total * 1e-3) / 1e9

    # ---- end-to-end through the public API with host buffers (H2D + apply + D2H)
    xh = torch.from_numpy(x_np).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    op.apply_host(xh.numpy(), out=yh.numpy())          # warm the staging buffers
    torch.cuda.synchronize(dev)
    dist_barrier(world)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.e2e_steps):
        op.apply_host(xh.numpy(), out=yh.numpy(), stream=stream)
    t1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = dist_max(t0.elapsed_time(t1), world, dev) / args.e2e_steps
    e2e_value = flops_step * world / (e2e_ms * 1e-3) / 1e9

    # ---- per-stage roofline
    hbm, hbm_src, fp64, fp64_src = load_peaks()
    P = fp64 * 1e12
    BW = hbm * 1e9
    stages = op.stages()
    r = cfg.ranks
    N = cfg.N
    stage_rows, sum_T, sum_t = stage_table(stages, r, N, nrhs, stage_ms, n_timed, P, BW)
    # dominant kernel: the stage shape with the largest share of the step
    by_kernel = {}
    for s, row in enumerate(stage_rows):
        key = (row["variant"], row["ranks"][0], row["ranks"][1], row["levels"][1] - row["levels"][0] + 1)
        by_kernel.setdefault(key, []).append(row)
    dom_key = max(by_kernel, key=lambda k: sum(rr["ms"] for rr in by_kernel[k]))
    dom = by_kernel[dom_key]
    dom_ms = sum(rr["ms"] for rr in dom) / len(dom)
    rin, rout = dom_key[1], dom_key[2]
    dom_flops = dom[0]["flops_executed"]
    achieved = dom_flops / (dom_ms * 1e-3) / 1e12
    tr = load_traffic(args.config, dom_flops)
    roofline = {"bound": "tensor", "achieved": achieved, "peak": fp64, "unit": "TFLOP/s",
                "frac": achieved / fp64, "traffic": tr[0] if tr else None,
                "kernel": f"level_dmma_kernel r_in={rin} r_out={rout} levels/launch={dom_key[3]} "
                          f"({dom_key[0]}; {len(dom)} launches/step)",
                "share_of_step": sum(rr["ms"] for rr in dom) / (ms_step if world == 1 else ms_local / args.steps),
                "peak_source": fp64_src + "; MEASURED_PEAKS.json has no FP64 figure",
                "algorithmic_flops_per_launch": dom_flops,
                "traffic_source": tr[1] if tr else None}
    # the whole step on the executed-flop basis, next to the Alg. 2-basis `value`
    # (reading R16: merged boundary stages execute fewer flops than Alg. 2)
    exec_flops = sum(rr["flops_executed"] for rr in stage_rows)
    roofline["step_tflops_executed"] = exec_flops / (ms_step * 1e-3) / 1e12
    roofline["step_frac_executed"] = roofline["step_tflops_executed"] / fp64
    roofline["step_tflops_alg2"] = flops_step / (ms_step * 1e-3) / 1e12
    per_stage = {"frac": sum_T / sum_t if sum_t else None, "sum_T_ms": sum_T * 1e3, "sum_t_ms": sum_t * 1e3,
                 "fp64_peak_tflops": fp64, "hbm_gbs": hbm, "hbm_source": hbm_src,
                 "frac_vs_nominal_fp64": None, "stages": stage_rows}
    # algorithmic roofline T_alg = max(F/P, (x+y+cores bytes)/BW)
    alg_bytes = 16 * N * nrhs + 32 * sum(r[k] * r[k + 1] for k in range(cfg.d))
    T_alg = max(flops_step / P, alg_bytes / BW)
    per_stage["algorithmic_frac"] = T_alg / (ms_step * 1e-3)
    # the same per-stage roofline on the flops the kernels actually execute: a
    # merged boundary stage applies a super-core with fewer flops than Alg. 2's
    # levels, so the Alg. 2 basis above can exceed 1; this one cannot
    sum_T_exec = sum(max(rr["flops_executed"] / P,
                         (8 * N * nrhs * (r[rr["levels"][0] - 1] + r[rr["levels"][1]])) / BW) for rr in stage_rows)
    per_stage["frac_executed"] = sum_T_exec / sum_t if sum_t else None
    per_stage["sum_T_executed_ms"] = sum_T_exec * 1e3
    per_stage["basis"] = ("frac: T_s = max(F_s/P, B_s/BW) with F_s = Alg. 2 flops 4*sum r_{k-1} r_k N (SURVEY 8(d)); "
                          "frac_executed: F_s = flops the stage's kernel executes")
    per_stage["frac_vs_nominal_fp64"] = sum(
        max(4 * sum(r[k - 1] * r[k] for k in range(st["levels"][0], st["levels"][1] + 1)) * N * nrhs
            / (FP64_NOMINAL_TFLOPS * 1e12),
            (8 * N * nrhs * (r[st["levels"][0] - 1] + r[st["levels"][1]])) / BW)
        for st in stage_rows) / sum_t if sum_t else None

    extra = None
    if world == 1 and not args.no_extra:
        op.close()
        del x, y, ws
        torch.cuda.empty_cache()
        extra = extra_measurements(dev, stream, P, BW, args.max_stage_levels)
        for v in extra.get("sharded_c4_emulated", {}).values():
            if args.config == "c4":
                v["projected_speedup_vs_1gpu"] = ms_step / v["projected_ms"]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = run_cpu_baseline(cfg, cores, x_np)
        cpu.pop("seconds", None)
        # the same CPU baseline (the oracle, all host cores) on the small configs, whole applies
        cpu["other_configs_ms"] = small_config_oracle_ms()
        cpu["other_configs_ms_1thread"] = small_config_oracle_ms(threads=1)

    clocks = clk.summary()
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if mode == "sharded" else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded; random cores with the config's rank profile stand in for the paper's inverse cores)",
        "config": config_desc(cfg, nrhs, parallelism_desc(mode, world, args.exchange)),
        "plan": {"launches_per_apply": op.launches_per_apply,
                 "stages": [[st["k_first"], st["k_last"], st["variant"]] for st in stages]},
        "gbs": (16 * N * nrhs) / (ms_step * 1e-3) / 1e9,
        "value_basis": "Alg. 2 flops (4*sum_k r_{k-1} r_k * N * nrhs, reading R4) per second; the boundary "
                       "stages apply exact super-cores with fewer flops (DESIGN.md 6.4), so value may exceed "
                       "the FP64 peak; tflops_executed counts the flops the kernels execute",
        "alg2_flops_per_apply": flops_step,
        "executed_flops_per_apply": sum(rr["flops_executed"] for rr in stage_rows),
        "tflops_executed": sum(rr["flops_executed"] for rr in stage_rows) / (ms_step * 1e-3) / 1e12,
        "per_stage_roofline": per_stage,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(x_np.nbytes), "d2h_bytes_per_step": int(x_np.nbytes)},
        # one kernel per stage, plus the reduce launch of every split-K stage
        "gpu_launches": sum(1 + (st_["ksplit"] > 1) for st_ in stages) * args.steps,
        "clocks": clocks,
        "other_configs_and_next_rows": extra,
    }
    if rank == 0:
        print(json.dumps(out))
    op.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

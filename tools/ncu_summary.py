"""Summarise an ncu --set full report into a small JSON for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep --config c4 --label "level 7 (48->48)" \
        --algorithmic-bytes 12884901888 --algorithmic-flops 154618822656 -o profiles/r01_..._summary.json
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration",
    "sm__ops_path_tensor_src_fp64.sum": "fp64_tensor_ops",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_pct_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__cycles_active.avg": "sm_active_cycles",
    "gpc__cycles_elapsed.max": "elapsed_cycles",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio": "stall_math_pipe",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_sb",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "stall_short_sb",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "stall_barrier",
    "smsp__warps_active.avg.per_cycle_active": "warps_active_per_smsp",
}

SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--config", required=True)
    ap.add_argument("--label", default="")
    ap.add_argument("--algorithmic-bytes", type=float, default=None)
    ap.add_argument("--algorithmic-flops", type=float, default=None)
    ap.add_argument("--launch-index", type=int, default=0, help="launch whose numbers are the headline")
    ap.add_argument("-o", "--out", required=True)
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    launches = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                v = vals[i].replace(",", "")
                try:
                    v = float(v) * SCALE.get(units[i], 1.0)
                except ValueError:
                    continue
                d[name] = v
        launches.append(d)
    first = launches[a.launch_index]
    out = {"config": a.config, "label": a.label, "report": a.report, "launches": launches}
    if "dram_read" in first and "dram_write" in first:
        out["dram_bytes_per_launch"] = first["dram_read"] + first["dram_write"]
    if a.algorithmic_bytes:
        out["algorithmic_bytes_per_launch"] = a.algorithmic_bytes
        out["traffic_over_algorithmic"] = out.get("dram_bytes_per_launch", 0) / a.algorithmic_bytes
    if a.algorithmic_flops and "duration" in first:
        out["algorithmic_flops_per_launch"] = a.algorithmic_flops
        out["achieved_tflops_under_ncu"] = a.algorithmic_flops / first["duration"] / 1e12
        if "fp64_tensor_ops" in first:
            # FP64 ops the tensor pipe executed (ncu) over the flops this repo claims for the launch
            out["tensor_fp64_ops_over_claimed_flops"] = first["fp64_tensor_ops"] / a.algorithmic_flops
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "launches"}, indent=1))
    print(json.dumps(first, indent=1))


if __name__ == "__main__":
    main()

"""Summarise ncu captures into profiles/ncu_summary.json (+ .md).

usage: python tools/ncu_summary.py KEY=path.ncu-rep[@name-substring] [KEY=path ...]

KEY names the kernel family (k_accel, k_slots, k_naive, k_wiener); the capture's
first launch whose name contains the substring (default: KEY) is summarised.
bench.py
reads profiles/ncu_summary.json[KEY].dram_bytes_per_launch for roofline.traffic.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_inst_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_cycles_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid_size",
    "launch__block_size": "block_size",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait_per_issue",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "stall_barrier_per_issue",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio": "stall_math_throttle_per_issue",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "stall_short_sb_per_issue",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_sb_per_issue",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            if h in ("Kernel Name", "Block Size", "Grid Size"):
                d[h] = v
            if h in WANT:
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                if u == "Kbyte":
                    x *= 1e3
                elif u == "Mbyte":
                    x *= 1e6
                elif u == "Gbyte":
                    x *= 1e9
                elif u in ("usecond", "us"):
                    x *= 1e3
                elif u in ("msecond", "ms"):
                    x *= 1e6
                d[WANT[h]] = x
        res.append(d)
    return res


def main(argv):
    outdir = os.environ.get("NCU_SUMMARY_DIR") or os.path.join(ROOT, "profiles")
    path = os.path.join(outdir, "ncu_summary.json")
    try:
        summary = json.load(open(path))
    except (OSError, ValueError):
        summary = {}
    for arg in argv:
        if "=" not in arg:
            continue
        key, rep = arg.split("=", 1)
        rep, _, pat = rep.partition("@")
        pat = pat or key
        kernels = [k for k in raw(rep) if pat in k.get("Kernel Name", "")]
        if not kernels:
            print(f"{key}: no launch matching {pat!r} in {rep}", file=sys.stderr)
            continue
        k = kernels[0]
        k["dram_bytes_per_launch"] = k.get("dram_read_bytes", 0.0) + k.get("dram_write_bytes", 0.0)
        k["source"] = os.path.basename(rep)
        summary[key] = k
    os.makedirs(os.path.dirname(path), exist_ok=True)
    json.dump(summary, open(path, "w"), indent=1, sort_keys=True)
    with open(os.path.join(outdir, "ncu_summary.md"), "w") as f:
        f.write("# ncu summary (--set full, one launch each)\n\n")
        for key, k in sorted(summary.items()):
            f.write(f"## {key}\n\n`{k.get('Kernel Name', '')}`\n\n")
            for name in sorted(k):
                if name not in ("Kernel Name", "source"):
                    f.write(f"- {name}: {k[name]}\n")
            f.write(f"- capture: {k.get('source')}\n\n")
    print(json.dumps(summary, indent=1, sort_keys=True))


if __name__ == "__main__":
    main(sys.argv[1:])

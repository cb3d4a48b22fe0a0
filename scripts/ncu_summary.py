"""Summarise an `ncu --set full` report into profiles/: one text table of the
metrics DESIGN.md cites per kernel and profiles/ncu_traffic.json (DRAM bytes
per launch, read by bench.py for roofline.traffic).

  python scripts/ncu_summary.py gpurun_out/far_full.ncu-rep profiles/r1_far_ncu_summary.txt
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_bytes.sum",
    "lts__t_sector_hit_rate.pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed_pipe_fp64.sum",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_wait",
    "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_mio_throttle",
    "smsp__pcsamp_warps_issue_stalled_barrier",
    "smsp__pcsamp_warps_issue_stalled_membar",
    "smsp__pcsamp_warps_issue_stalled_sleeping",
]


def short(name: str) -> str:
    name = name.split("(")[0]
    return name.replace("(anonymous namespace)::", "").replace("unnamed>::", "").replace("void ", "")


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    lines = []
    traffic_path = os.path.join(os.path.dirname(out), "ncu_traffic.json")
    traffic = {}
    if os.path.exists(traffic_path):
        traffic = json.load(open(traffic_path))
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        k = short(d["Kernel Name"])
        lines.append(f"== {k}")
        for m in METRICS:
            if m in d:
                lines.append(f"   {m:70s} {d[m]}")
        try:
            rd = float(d["dram__bytes_read.sum"])
            wr = float(d["dram__bytes_write.sum"])
            unit = 1.0
            # ncu --csv reports these in the unit shown in row 1
            u = rows[1][hdr.index("dram__bytes_read.sum")]
            unit = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
            traffic[k] = {"dram_bytes": (rd + wr) * unit,
                          "duration_ns": float(d["gpu__time_duration.sum"]) *
                          {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(
                              rows[1][hdr.index("gpu__time_duration.sum")], 1.0),
                          "report": os.path.basename(rep)}
        except (KeyError, ValueError):
            pass
    with open(out, "w") as fh:
        fh.write(f"# ncu --set full summary of {os.path.basename(rep)}\n")
        fh.write("\n".join(lines) + "\n")
    with open(traffic_path, "w") as fh:
        json.dump(traffic, fh, indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()

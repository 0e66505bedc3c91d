"""Summarise an `ncu --set full` report of the fused sweeps for profiles/:
key metrics per kernel (JSON) and the per-launch DRAM bytes that bench.py
reports as roofline.traffic (profiles/dram_traffic.json).

usage: python scripts/ncu_summary.py REP.ncu-rep OUT.json [--traffic WORKLOAD]"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
]


def to_bytes(v: str, unit: str) -> float:
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    name_i = head.index("Kernel Name")
    summary, traffic = {}, {}
    for r in data:
        k = r[name_i]
        d = {}
        for key in KEYS:
            if key in head:
                i = head.index(key)
                d[key] = f"{r[i]} {units[i]}".strip()
        summary[k] = d
        i_r, i_w = head.index("dram__bytes_read.sum"), head.index("dram__bytes_write.sum")
        b = to_bytes(r[i_r], units[i_r]) + to_bytes(r[i_w], units[i_w])
        short = k.split("<")[0].replace("void ", "").strip()
        traffic[short] = b
    with open(out, "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1))
    if "--traffic" in sys.argv:
        wl = sys.argv[sys.argv.index("--traffic") + 1]
        t = {"workload": wl, "source": f"{out} (ncu --set full, one launch each)"}
        t.update(traffic)
        with open("profiles/dram_traffic.json", "w") as f:
            json.dump(t, f, indent=1)
        print(t)


if __name__ == "__main__":
    main()

"""Summarise ncu --set full reports into profiles/<round>/ncu_summary.json (+ text)."""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__warps_eligible.avg.per_cycle_active": "eligible_warps_per_cycle",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "smsp__inst_executed.sum": "warp_inst",
    "sm__cycles_active.avg": "sm_cycles_active",
    "sm__cycles_elapsed.avg": "sm_cycles_elapsed",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_sb",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio": "stall_math_throttle",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = {}
    for v in rows[2:]:
        name = v[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        name = name.replace("<unnamed>::", "").replace("unnamed>::", "").replace("pals::", "")
        name = name.split("<")[0].strip()
        d = {}
        for i, col in enumerate(h):
            if col in WANT:
                try:
                    x = float(v[i].replace(",", ""))
                except ValueError:
                    continue
                d[WANT[col]] = x * SCALE.get(u[i], 1.0)
        d["dram_bytes_per_launch"] = d.get("dram_read", 0) + d.get("dram_write", 0)
        res[name] = d
    return res


if __name__ == "__main__":
    out_json = sys.argv[1]
    allres = {}
    for rep in sys.argv[2:]:
        allres.update(summarise(rep))
    with open(out_json, "w") as f:
        json.dump(allres, f, indent=1)
    for k, d in allres.items():
        print(k, {a: (round(b, 4) if isinstance(b, float) else b) for a, b in d.items()})

"""Summarise an ncu report (raw page) for one kernel launch: duration, DRAM
bytes, issue / warp / pipe utilisation and the top stall reasons.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--json out.json]
"""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")][:80]}
        for k in KEYS:
            if k in h:
                d[k] = f"{v[h.index(k)]} {u[h.index(k)]}".strip()
        st = {}
        for i, x in enumerate(h):
            if x.startswith("smsp__pcsamp_warps_issue_stalled") and not x.endswith("not_issued"):
                try:
                    st[x.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v[i])
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        d["stall_share"] = {k: round(x / tot, 3) for k, x in
                            sorted(st.items(), key=lambda t: -t[1])[:10]}
        res.append(d)
    print(json.dumps(res, indent=1))
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()

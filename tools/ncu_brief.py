"""Key metrics + stall breakdown of every kernel in an ncu report.
python tools/ncu_brief.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
keys = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
st = [k for k in h if k.startswith("smsp__average_warps_issue_stalled") and
      k.endswith("per_issue_active.ratio")]
for v in rows[2:]:
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}
    for k in keys:
        if k in d:
            print(f"{k:60s} {d[k][0]} {d[k][1]}")
    vals = sorted(((float(d[k][0] or 0), k) for k in st), reverse=True)
    print("stalls (warps per issue):", ", ".join(
        f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
        f"={x:.2f}" for x, k in vals[:9]))
    print()

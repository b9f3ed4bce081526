"""Summarise an ncu report: SOL, issue, stall reasons, pipes (dev tool)."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, vals = r[0], r[2]
d = dict(zip(hdr, vals))
keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed.sum"]
for k in keys:
    if k in d: print(f"{k:80s} {d[k]}")
st = {h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): v
      for h, v in d.items() if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio")}
tot = sum(float(v) for v in st.values())
print("stall cycles per issued instruction (total %.2f):" % tot)
for k, v in sorted(st.items(), key=lambda kv: -float(kv[1])):
    if float(v) > 0.01: print(f"   {k:30s} {float(v):.3f}")

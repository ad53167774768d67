"""Summarise an ncu --set full report (one row per captured kernel) into markdown + JSON."""
import csv, io, json, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units, data = rows[0], rows[1], rows[2:]
WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA cycles %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (SM)"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads/instr"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes.sum.per_second", "DRAM throughput"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]
res = []
for v in data:
    d = {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else "?"}
    for m, label in WANT:
        if m in h:
            d[label] = v[h.index(m)] + " " + units[h.index(m)]
    st = {}
    for i, n in enumerate(h):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
            try:
                st[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v[i].replace(",", ""))
            except ValueError:
                pass
    T = sum(st.values()) or 1.0
    d["stall samples % (top 8)"] = {k: round(100 * x / T, 1) for k, x in sorted(st.items(), key=lambda x: -x[1])[:8]}
    res.append(d)
print(json.dumps(res, indent=1))

"""Build profiles/<tag>_ncu_summary.md and profiles/score_kernel_dram.json from
an ncu launch list (CSV) and ncu --set full reports (one per kernel).

usage: python scripts/profile_report.py TAG launches.csv rep1.ncu-rep [rep2 ...]
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, launch_csv, reps = sys.argv[1], sys.argv[2], sys.argv[3:]


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        name = r[ik].split("(")[0].replace("void ", "")
        tot[name] += float(r[iv].replace(",", "")) * scale[r[iu]]
        cnt[name] += 1
    return tot, cnt, len(data)


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    res = []
    for v in data:
        g = lambda m, v=v: (v[h.index(m)], units[h.index(m)]) if m in h else ("n/a", "")
        if "nan" in g("smsp__inst_executed.sum")[0]:
            continue  # ncu leaves later kernels of a multi-kernel full capture empty
        st = {}
        for i, n in enumerate(h):
            if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
                try:
                    st[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v[i].replace(",", ""))
                except ValueError:
                    pass
        T = sum(st.values()) or 1.0
        res.append({"kernel": v[h.index("Kernel Name")], "g": g,
                    "stalls": {k: round(100 * x / T, 1) for k, x in sorted(st.items(), key=lambda x: -x[1])[:6]}})
    return res


tot, cnt, n = launch_table(launch_csv)
T = sum(tot.values())
lines = [f"# ncu summary — {tag}", "",
         f"Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none` of `python bench.py --steps 2 "
         f"--warmup 1` (config 5, N=1; warm-up, 2 timed steps and the e2e steps). {n} launches, {T:.1f} ms total. "
         "Cold-cache, serialised per-launch times: compare shares, not absolutes.", "",
         "| kernel | launches | total ms | share |", "|---|---|---|---|"]
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:16]:
    lines.append(f"| `{k[:90]}` | {cnt[k]} | {v:.2f} | {100 * v / T:.1f}% |")
lines += ["", "Full captures (`ncu --set full --clock-control none --import-source on`, one timed config-5 step):", ""]
M = [("gpu__time_duration.sum", "duration"), ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active"),
     ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe"),
     ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe (heavy+lite)"),
     ("sm__inst_executed.avg.per_cycle_active", "IPC per SM"),
     ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads per instr"),
     ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
     ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
     ("dram__bytes.sum.per_second", "DRAM throughput"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
     ("launch__registers_per_thread", "registers/thread"), ("launch__grid_size", "grid"),
     ("smsp__inst_executed.sum", "warp instructions")]
dram = {}
seen = set()
for rep in reps:
    for k in full_metrics(rep):
        if k["kernel"] in seen:
            continue
        seen.add(k["kernel"])
        lines.append(f"### `{k['kernel']}`  ({os.path.basename(rep)})")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for m, label in M:
            val, unit = k["g"](m)
            lines.append(f"| {label} (`{m}`) | {val} {unit} |")
        lines.append(f"| stall samples, top 6 | {k['stalls']} |")
        lines.append("")
        rd, ur = k["g"]("dram__bytes_read.sum")
        wr, uw = k["g"]("dram__bytes_write.sum")
        mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        try:
            dram[k["kernel"].split("(")[0]] = float(rd) * mul[ur] + float(wr) * mul[uw]
        except (ValueError, KeyError):
            pass
with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w") as f:
    f.write("\n".join(lines) + "\n")
if dram:
    json.dump({"dram_bytes_per_launch": sum(dram.values()), "config": 5,
               "note": "score phase of one config-5 step = score3a + score3b + score12 launches; "
                       "dram__bytes_read.sum + dram__bytes_write.sum from ncu --set full",
               "per_kernel": dram, "source": [os.path.basename(r) for r in reps]},
              open(os.path.join(ROOT, "profiles", "score_kernel_dram.json"), "w"), indent=1)
print("\n".join(lines[:30]))

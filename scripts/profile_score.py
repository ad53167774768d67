"""Summarise an ncu --set full capture of ONE bench step's score kernels into
profiles/r2_score_ncu.json (read by bench.py for the work-based roofline).

usage: python scripts/profile_score.py gpurun_out/score_full.ncu-rep [out.json]
The capture: ncu --set full -k regex:"score|gfold" -s <warm-up launches> -c 4 python bench.py
--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --no-f2 --no-pb --no-per-config
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "smsp__inst_executed.sum": "inst_executed",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "launch__registers_per_thread": "registers",
}
SCALE = {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
         "Gbyte": 1e9, "%": 1, "inst": 1, "": 1, "register/thread": 1}


def main(rep, out="profiles/r2_score_ncu.json"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"name": d["Kernel Name"].split("(")[0].replace("void ", "").replace("ppipe::", "")}
        for m, key in METRICS.items():
            v = d.get(m, "")
            try:
                x = float(v.replace(",", "")) * SCALE.get(u.get(m, ""), 1)
                k[key] = None if x != x else x  # NaN (a section ncu could not collect) -> None
            except ValueError:
                k[key] = None
        kernels.append(k)
    tot_t = sum(k["duration_ns"] or 0 for k in kernels)
    total = {"duration_ms": tot_t / 1e6, "inst_executed": sum(k["inst_executed"] or 0 for k in kernels),
             "dram_bytes": sum((k["dram_read"] or 0) + (k["dram_write"] or 0) for k in kernels),
             "issue_active_time_weighted_pct": sum((k["issue_active_pct"] or 0) * (k["duration_ns"] or 0)
                                                   for k in kernels) / max(tot_t, 1)}
    res = {"config": 5, "source": rep.split("/")[-1], "kernels": kernels, "total": total,
           "note": "one bench step's score kernels under ncu --set full (clock-control none); durations are "
                   "serialised / cold-cache, only the counts and ratios are used by bench.py"}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(total))
    for k in kernels:
        print(k)


if __name__ == "__main__":
    main(*sys.argv[1:])

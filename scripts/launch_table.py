"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel
launches, mean and total duration (us), share of the listed total."""
import collections
import csv
import re
import sys


def table(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr, d = None, collections.defaultdict(list)
    for r in rows:
        if len(r) > 5 and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            x = dict(zip(hdr, r))
            if x["Metric Name"] == "gpu__time_duration.sum":
                k = re.sub(r"\(.*", "", x["Kernel Name"]).replace("void ", "").replace("(anonymous namespace)::", "")
                k = re.sub(r"<unnamed>::|unnamed>::", "", k)
                scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(x["Metric Unit"], 1.0)
                d[k[:70]].append(float(x["Metric Value"].replace(",", "")) * scale)
    tot = sum(sum(v) for v in d.values())
    out = [f"{'kernel':70s} {'n':>5s} {'mean_us':>10s} {'total_us':>11s} {'share':>6s}"]
    for k, v in sorted(d.items(), key=lambda t: -sum(t[1]))[:top]:
        out.append(f"{k:70s} {len(v):5d} {sum(v) / len(v):10.1f} {sum(v):11.1f} {sum(v) / tot:6.1%}")
    out.append(f"{'total':70s} {sum(len(v) for v in d.values()):5d} {'':10s} {tot:11.1f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(table(sys.argv[1]))

"""Top SASS instructions of one kernel from `ncu -i X --page source --csv` output:
by instructions executed and by warp-stall samples."""
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    ix = {h: j for j, h in enumerate(hdr)}
    data = []
    for r in rows[hi + 1:]:
        if len(r) != len(hdr):
            continue
        try:
            ex = float(r[ix["Instructions Executed"]] or 0)
            st = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        data.append((ex, st, r[0], r[ix["Source"]].strip()))
    tex = sum(d[0] for d in data) or 1
    tst = sum(d[1] for d in data) or 1
    print(f"total instructions executed (warp) {tex:.3g}, stall samples {tst:.0f}")
    for i, d in enumerate(data):
        if d[0] / tex > 0.004 or d[1] / tst > 0.01:
            print(f"{i:5d} ex {d[0] / tex:6.1%} stall {d[1] / tst:6.1%}  {d[3][:90]}")


if __name__ == "__main__":
    main(sys.argv[1])

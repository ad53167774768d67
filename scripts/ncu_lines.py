"""Per-source-line totals (instructions executed, warp-stall samples) of one kernel from
`ncu -i X --page source --csv --print-source cuda,sass --launch-count 1` output."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    hdr = rows[hi]
    ex_i = hdr.index("Instructions Executed")
    st_i = hdr.index("Warp Stall Sampling (All Samples)")
    agg = {}
    for r in rows[hi + 1:]:
        if len(r) != len(hdr) or not r[0]:
            continue
        try:
            agg[(int(r[0]), r[1].strip())] = (float(r[ex_i] or 0), float(r[st_i] or 0))
        except ValueError:
            continue
    tex = sum(v[0] for v in agg.values()) or 1
    tst = sum(v[1] for v in agg.values()) or 1
    print(f"instructions executed {tex:.3g}, stall samples {tst:.0f}")
    for (ln, src), (e, s) in sorted(agg.items(), key=lambda t: -t[1][0])[:top]:
        print(f"{ln:5d} ex {e / tex:6.1%} stall {s / tst:6.1%}  {src[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)

"""SASS of one kernel with per-instruction execution counts (ncu source page).

    ncu -i rep.ncu-rep --page source --csv --print-source=sass > x.csv
    python tools/ncu_sass.py x.csv [min_count]

Prints address-ordered instructions whose warp-level execution count is at
least `min_count` (default: 0.1% of the total), so hot loops read as
contiguous blocks.
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = next(r for r in rows if r and r[0] == "Address")
    ia, isrc, ie = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
    recs = []
    for r in rows:
        if len(r) > ie and r[ia].startswith("0x"):
            try:
                recs.append((int(r[ia], 16), r[isrc].strip(), int(r[ie] or 0)))
            except ValueError:
                pass
    tot = sum(x[2] for x in recs) or 1
    thr = int(sys.argv[2]) if len(sys.argv) > 2 else tot // 1000
    base = recs[0][0] if recs else 0
    print(f"total warp instructions {tot}")
    for a, s, n in recs:
        if n >= thr:
            print(f"{a - base:6x} {n:12d} {100 * n / tot:5.2f}%  {s}")


if __name__ == "__main__":
    main()

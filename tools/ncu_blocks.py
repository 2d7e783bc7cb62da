"""Basic-block view of a kernel's SASS execution counts (ncu source page).

    ncu -i rep.ncu-rep --page source --csv --print-source=sass > x.csv
    python tools/ncu_blocks.py x.csv [lo_hex hi_hex] [top] [pairs]

Groups consecutive instructions with equal execution counts into blocks
and prints the most expensive ones (count x length), optionally within
an address range (offsets from the kernel start) and per unit of work.
"""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    ia, isrc, ie = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
    recs = []
    for r in rows:
        if len(r) > ie and r[ia].startswith("0x"):
            try:
                recs.append((int(r[ia], 16), r[isrc].strip(), int(r[ie] or 0)))
            except ValueError:
                pass
    base = recs[0][0]
    return [(a - base, s, n) for a, s, n in recs]


def main():
    recs = load(sys.argv[1])
    lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
    hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 40
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    per = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
    blocks = []
    for a, s, n in recs:
        if not (lo <= a < hi):
            continue
        op = s.split()[1] if s.startswith("@") else s.split()[0]
        if blocks and blocks[-1][1] == n and a - blocks[-1][3] == 16:
            blocks[-1][2] += 1
            blocks[-1][3] = a
            blocks[-1][4].append(op)
        else:
            blocks.append([a, n, 1, a, [op]])
    tot = sum(b[1] * b[2] for b in blocks)
    print(f"range total {tot / per:.0f} per unit")
    for b in sorted(blocks, key=lambda b: -b[1] * b[2])[:top]:
        print(f"{b[0]:6x} n={b[1] / per:9.1f} len={b[2]:3d} tot={b[1] * b[2] / per:8.0f}  {' '.join(b[4][:16])}")


if __name__ == "__main__":
    main()

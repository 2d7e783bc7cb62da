"""Aggregate an ncu source page (--print-source=cuda,sass --csv) by CUDA line.

    ncu -i rep.ncu-rep --page source --csv --print-source=cuda,sass > x.csv
    python tools/ncu_lines.py x.csv [top]
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    agg = collections.defaultdict(lambda: [0, 0, ""])
    cur_file = None
    header = None
    for line in open(path).read().splitlines():
        if line.startswith('"File Path"'):
            cur_file = next(csv.reader([line]))[1]
            continue
        if line.startswith('"Function Name"'):
            continue
        if line.startswith('"Line No"'):
            header = next(csv.reader([line]))
            continue
        r = next(csv.reader([line]))
        if header and len(r) > 6 and r[0].isdigit():
            d = dict(zip(header, r))
            key = (cur_file.split("/")[-1], int(r[0]))
            try:
                agg[key][0] += int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
                agg[key][1] += int(d.get("Instructions Executed", "0") or 0)
            except ValueError:
                pass
            agg[key][2] = r[1][:80]
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    print(f"total stall samples {ts}, warp instructions {ti}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{k[0]:20s}:{k[1]:4d} inst%={100 * v[1] / ti:5.1f} stall%={100 * v[0] / ts:5.1f}  {v[2]}")


if __name__ == "__main__":
    main()

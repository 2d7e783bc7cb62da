"""Print kernel name (shortened) and duration from an ncu --csv metrics dump on stdin."""
import csv
import sys

rows = list(csv.reader(l for l in sys.stdin if l.startswith('"')))
hdr = rows[0]
kn, mv = hdr.index("Kernel Name"), hdr.index("Metric Value")
for r in rows[1:]:
    name = r[kn].split("(")[0].replace("void ", "").replace("bimine::", "")
    print(f"{name[:40]:40s} {r[mv]}")

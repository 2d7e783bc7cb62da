"""Summarise `prof` lines of a BIMINE_NW_PROFILE build (one launch)."""
import re
import sys

start, bands, tb, entry = {}, {}, None, {}
for line in sys.stdin:
    m = re.match(r"prof entry cta (\d+) ns (\d+)", line)
    if m:
        entry[int(m[1])] = int(m[2])
    m = re.match(r"prof start cta (\d+) ns (\d+)", line)
    if m:
        start[int(m[1])] = int(m[2])
    m = re.match(r"prof band (\d+) cta (\d+) end_ns (\d+)", line)
    if m:
        bands[int(m[1])] = int(m[3])
    m = re.match(r"prof traceback end_ns (\d+)", line)
    if m:
        tb = int(m[1])
t0 = min(start.values())
if entry:
    e0 = min(entry.values())
    print("cta entries (us before first start):", round((t0 - e0) / 1e3, 1), " spread", round((max(entry.values()) - e0) / 1e3, 1))
print("cta starts (us):", sorted(round((v - t0) / 1e3, 1) for v in start.values())[:8], "...", round((max(start.values()) - t0) / 1e3, 1))
ks = sorted(bands)
for g in ks[:10] + ks[-3:]:
    print(f"band {g:4d} end {(bands[g] - t0) / 1e3:9.1f} us")
d = [(bands[g] - bands[g - 1]) / 1e3 for g in ks[1:]]
print("mean lag per band (us):", round(sum(d) / len(d), 2), "max", round(max(d), 1))
print("traceback end (us):", round((tb - t0) / 1e3, 1), " traceback time:", round((tb - bands[ks[-1]]) / 1e3, 1))

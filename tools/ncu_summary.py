"""Summarise ncu --set full captures: one row per profiled launch.

    python tools/ncu_summary.py rep1.ncu-rep [rep2 ...] > summary.csv
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("duration_us", "gpu__time_duration.sum", 1),
    ("dram_read_bytes", "dram__bytes_read.sum", 1),
    ("dram_write_bytes", "dram__bytes_write.sum", 1),
    ("dram_throughput_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("ipc_active", "sm__inst_executed.avg.per_cycle_active", 1),
    ("issue_active_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
    ("warp_instructions", "smsp__inst_executed.sum", 1),
    ("achieved_occupancy_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("registers_per_thread", "launch__registers_per_thread", 1),
    ("smem_per_block", "launch__shared_mem_per_block", 1),
    ("grid", "launch__grid_size", 1),
    ("block", "launch__block_size", 1),
    ("cluster", "launch__cluster_size", 1),
    ("alu_pipe_pct", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
    ("lsu_pipe_pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
    ("fp64_pipe_pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1),
]
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "barrier", "branch_resolving", "math_pipe_throttle",
          "mio_throttle", "lg_throttle", "no_instructions", "selected", "not_selected", "dispatch_stall", "sleeping"]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], dict(zip(r[0], r[1]))
    scale_of = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6,
                "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for v in r[2:]:
        d = dict(zip(hdr, v))
        row = {"report": rep.split("/")[-1], "kernel": d.get("Kernel Name", "")[:60]}
        for name, key, scale in KEYS:
            x = d.get(key, "")
            try:
                row[name] = round(float(x.replace(",", "")) * scale * scale_of.get(units.get(key, ""), 1.0), 3)
            except ValueError:
                row[name] = x
        st = {}
        for s in STALLS:
            x = d.get(f"smsp__pcsamp_warps_issue_stalled_{s}", "")
            try:
                st[s] = float(x.replace(",", ""))
            except ValueError:
                pass
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda kv: -kv[1])[:4]
        row["top_stalls"] = "; ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top)
        yield row


def main():
    allrows = [r for rep in sys.argv[1:] for r in rows(rep)]
    if not allrows:
        return
    w = csv.DictWriter(sys.stdout, fieldnames=list(allrows[0].keys()))
    w.writeheader()
    for r in allrows:
        w.writerow(r)


if __name__ == "__main__":
    main()

"""One-line-per-kernel summary of ncu reports (duration, DRAM bytes, SOL %,
occupancy, registers, top stall reasons).

    python tools/ncu_summary.py report1.ncu-rep [report2 ...]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "ms"),
    ("dram__bytes_read.sum", "rd"),
    ("dram__bytes_write.sum", "wr"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__block_size", "blk"),
]


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        parts = [d.get("Kernel Name", "?")[:70]]
        for k, lab in KEYS:
            v = d.get(k, "n/a")
            if k.startswith("dram__bytes") and v not in ("n/a", ""):
                scale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(u.get(k, ""), 1.0)
                v = f"{float(v) * scale:.3f}GB"
            parts.append(f"{lab}={v}")
        stalls = []
        for k in h:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(d[k]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        parts.append("stalls=" + ",".join(f"{n}:{v:.2f}" for v, n in stalls[:4]))
        res.append(" ".join(parts))
    return res


if __name__ == "__main__":
    for r in sys.argv[1:]:
        for line in summarise(r):
            print(line)

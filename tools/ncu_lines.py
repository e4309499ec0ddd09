"""Summarise an ncu report's source page: warp-stall samples per CUDA source line.

    python tools/ncu_lines.py <report.ncu-rep> [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = []
    fname = "?"
    total = 0
    hdr = None
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path" or rec[0] == "File Name":
            fname = rec[1].rsplit("/", 1)[-1]
            continue
        if rec[0] == "Line No":
            hdr = rec
            continue
        if hdr is None or len(rec) < 5 or not rec[0]:
            continue
        d = dict(zip(hdr, rec))
        try:
            s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        total += s
        rows.append((s, fname, rec[0], rec[1].strip()[:90]))
    rows.sort(reverse=True)
    print("total samples", total)
    for s, f, ln, src in rows[:top]:
        print(f"{100.0 * s / max(total, 1):5.1f}% {f}:{ln:<5} {src}")


if __name__ == "__main__":
    main()

"""Aggregate an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv` launch list by kernel name.

    python tools/launch_table.py launches.csv
"""
import csv
import sys
from collections import defaultdict


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = None
    agg = defaultdict(lambda: {"n": 0, "ns": 0.0, "bytes": 0.0})
    seen = set()
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "")[:60]
        key = (d["ID"], name)
        a = agg[name]
        if key not in seen:
            seen.add(key)
            a["n"] += 1
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1)
        if d["Metric Name"] == "gpu__time_duration.sum":
            a["ns"] += v
        elif d["Metric Name"].startswith("dram__bytes"):
            a["bytes"] += v
    tot = sum(a["ns"] for a in agg.values())
    print(f"total {tot / 1e6:.3f} ms over {sum(a['n'] for a in agg.values())} launches")
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
        gbs = a["bytes"] / a["ns"] if a["ns"] else 0.0
        print(f"{100 * a['ns'] / tot:5.1f}%  {a['ns'] / 1e6:8.3f} ms  n={a['n']:4d}  {gbs:7.1f} GB/s  {name}")


if __name__ == "__main__":
    main()

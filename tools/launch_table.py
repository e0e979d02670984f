"""Markdown table of an ncu launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv): per kernel and launch shape,
launch count, mean duration and DRAM bytes per launch.
usage: launch_table.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ix = {k: i for i, k in enumerate(h)}
per = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) != len(h):
        continue
    key = (r[ix["Kernel Name"]][:60], r[ix["Grid Size"]], r[ix["Block Size"]])
    d = per.setdefault(key, {"ids": set(), "t": 0.0, "rd": 0.0, "wr": 0.0})
    d["ids"].add(r[ix["ID"]])
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3, "ms": 1e3,
             "byte": 1e-3, "Kbyte": 1.0, "Mbyte": 1e3, "Gbyte": 1e6}.get(unit, 1.0)
    name = r[ix["Metric Name"]]
    if name.startswith("gpu__time_duration"):
        d["t"] += v * scale
    elif name.startswith("dram__bytes_read"):
        d["rd"] += v * scale
    elif name.startswith("dram__bytes_write"):
        d["wr"] += v * scale
print("| kernel | grid | block | launches | avg us | DRAM read KB/launch | DRAM write KB/launch |")
print("|---|---|---|---|---|---|---|")
for (k, g, b), d in per.items():
    n = len(d["ids"])
    print(f"| `{k}` | {g} | {b} | {n} | {d['t'] / n:.1f} | {d['rd'] / n:.1f} | {d['wr'] / n:.1f} |")

"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel (count, mean ns).
  python tools/launch_summary.py profiles/ncu/r02_bench_default_launches.csv > profiles/ncu/r02_bench_default_launches.txt
"""
import collections
import csv
import io
import sys

rows = open(sys.argv[1]).read().splitlines()
i = next(k for k, l in enumerate(rows) if l.startswith('"ID"'))
acc = collections.OrderedDict()
for x in csv.DictReader(io.StringIO("\n".join(rows[i:]))):
    if x["Metric Name"] != "gpu__time_duration.sum":
        continue
    v = float(x["Metric Value"].replace(",", ""))
    ns = v * {"usecond": 1e3, "us": 1e3, "msecond": 1e6}.get(x["Metric Unit"], 1)
    acc.setdefault(x["Kernel Name"], []).append(ns)
print("# ncu --metrics gpu__time_duration.sum --clock-control none (serialised, cold per kernel): default bench headline (conv2d)")
print("count  mean_ns  kernel")
for k, v in acc.items():
    print(f"{len(v):5d} {sum(v) / len(v):9.0f}  {k[:90]}")

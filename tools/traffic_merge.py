"""Sums the per-launch ncu metrics of tools/gpu_traffic.sh into the bench's traffic table."""
import csv
import json
import os
import sys

d = sys.argv[1]
res = {}
for f in sorted(os.listdir(d)):
    if not f.endswith(".csv"):
        continue
    w = f[:-4]
    rows = list(csv.reader(open(os.path.join(d, f))))
    hdr = next((r for r in rows if "Kernel Name" in r), None)
    if hdr is None:
        continue
    i0 = rows.index(hdr)
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per = {}
    for r in rows[i0 + 1:]:
        if len(r) <= vi:
            continue
        k = per.setdefault(r[ii], {"kernel": r[ki][:90]})
        k[r[mi]] = float(r[vi].replace(",", ""))
    meta = json.load(open(os.path.join(d, w + ".json"))) if os.path.exists(os.path.join(d, w + ".json")) else {}
    rd = sum(k.get("dram__bytes_read.sum", 0) for k in per.values())
    wr = sum(k.get("dram__bytes_write.sum", 0) for k in per.values())
    l2w = sum(k.get("lts__t_sectors_srcunit_tex_op_write.sum", 0) for k in per.values()) * 32
    res[w] = rd + wr
    res[w + "_detail"] = {
        "dram_read": rd, "dram_write": wr, "l2_write_from_sm": l2w, "launches": len(per),
        "kernels": [k["kernel"] for k in per.values()],
        "ncu_ns": sum(k.get("gpu__time_duration.sum", 0) for k in per.values()),
        "algorithmic": meta.get("algorithmic_bytes"),
        "how": "ncu --nvtx-include traffic/ --cache-control none: every launch of one execute after a 256 MiB "
               "L2-flushing read (tools/gpu_traffic.sh); dram_write misses output lines still dirty in L2 at "
               "kernel end, l2_write_from_sm is the store traffic the kernels sent to L2",
    }
print(json.dumps(res, indent=1, sort_keys=True))

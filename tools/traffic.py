"""Developer tool (run under ncu on the GPU box): DRAM traffic of EVERY launch of one execute of
a bench workload with L2 cold (a 256 MiB read before the execute, ncu's own cache control off). The execute is wrapped in the NVTX range "traffic"; tools/gpu_traffic.sh
profiles only that range and tools/traffic_merge.py sums the launches into
profiles/ncu_traffic.json (the bench's roofline "traffic" field).
  ncu --nvtx --nvtx-include "traffic/" --cache-control none --metrics ... python tools/traffic.py <workload>
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2502_11407_b200 as g  # noqa: E402

name = sys.argv[1]
spec = bench.WORKLOADS[name]
op = g.TensorOpSpec.parse_text(json.dumps(spec["op"]))
sched = g.optimize(op, g.HardwareSpec.b200(0), g.EngineConfig(seed=0, mode="b200"))
k = g.Kernel(op, sched, 0, spec.get("variant", "auto"))
gen = torch.Generator(device="cuda")
gen.manual_seed(0)
xs, out = bench.make_inputs(op, spec, gen, torch, "cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    k.execute(xs, out)
torch.cuda.synchronize()
# cold L2 without foreign dirty lines: the flush READS 256 MiB (a write-flush would leave ~126 MB
# of dirty lines whose write-back lands inside the measured launches)
flush.view(torch.float32).sum()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("traffic")
k.execute(xs, out)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print(json.dumps({"workload": name, "family": k.info["plan"].get("family"), "launches": k.info["launches"],
                  "algorithmic_bytes": op.bytes}))

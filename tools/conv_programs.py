"""Developer tool: the headline conv's conv_flat programs as different constructed states select
them (tcplan.hpp conv_flat_plan_of), each timed like bench.py's headline (256 MiB L2 flush, host
enqueue hidden behind a sleep kernel, CUDA events around one execute, median of 30), next to the
B200 model's estimate of that state.
  python tools/conv_programs.py > profiles/r02_conv_programs.jsonl
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2502_11407_b200 as g  # noqa: E402

spec = bench.WORKLOADS["conv2d"]
op = g.TensorOpSpec.parse_text(json.dumps(spec["op"]))
hw = g.HardwareSpec.b200(0)
gen = torch.Generator(device="cuda")
gen.manual_seed(0)
xs, out = bench.make_inputs(op, spec, gen, torch, "cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
states = {
    "construction (top-1)": g.optimize(op, hw, g.EngineConfig(seed=0, mode="b200", top_k=1)),
    "f tile 64, h x w 64 x 64": g.from_trace(op, hw, [[3, -1, 0], [3, -1, 0]], mode="b200"),
    "f tile 64, h x w 8 x 16": g.from_trace(op, hw, [[0, 2, 8], [0, 3, 4], [3, -1, 0], [3, -1, 0]], mode="b200"),
    "f tile 32": g.from_trace(op, hw, [[0, 1, 2], [3, -1, 0], [3, -1, 0]], mode="b200"),
    "f tile 16": g.from_trace(op, hw, [[0, 1, 4], [3, -1, 0], [3, -1, 0]], mode="b200"),
}
ref = None
for name, sched in states.items():
    k = g.Kernel(op, sched, 0, "tc_tf32")
    for _ in range(3):
        k.execute(xs, out)
    torch.cuda.synchronize()
    if ref is None:
        ref = out.clone()
    same = bool(torch.equal(out, ref))
    ms = []
    for _ in range(30):
        bench.flush_l2(torch, flush)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        k.execute(xs, out)
        e.record()
        e.synchronize()
        ms.append(s.elapsed_time(e))
    t = statistics.median(ms)
    p = k.info["plan"]
    print(json.dumps({"state": name, "schedule": sched[0]["state"]["repr"], "FN": p["FN"],
                      "filter_groups": p["filter_groups"], "cta_pair": p["cta_pair"], "grid": p["grid"],
                      "measured_us": round(t * 1e3, 2), "tflops": round(op.flops / (t * 1e-3) / 1e12, 1),
                      "model_us": round(sched[0]["cost"]["exec_seconds"] * 1e6, 2),
                      "bit_identical_to_first": same}), flush=True)

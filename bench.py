#!/usr/bin/env python
"""Constructed-kernel throughput on B200 (BASELINE.json metric), one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload conv2d]

A step = one execute of the hot path (operator description -> constructed schedule ->
instantiated sm_100a kernel) over one batch of synthetic input of the BASELINE shape.
  value      device time of the execute (CUDA events on the launching stream), inputs resident
             in HBM, L2 flushed (256 MiB write) between steps; whole-job throughput over ranks
  e2e        the same through the C-ABI host-buffer call gensor_execute_host (pinned host
             inputs -> H2D -> execute -> D2H -> sync), CUDA events around each call
  roofline   the dominant kernel's own launches (events around each internal launch)
  cpu_baseline  the oracle's interpret() of the same schedule on a bounded sample, all host threads
  --impl reference  the reference's CPU path: its own construct library (oracle/_ref, unmodified
             proj/src) + the restated interpreter (its executor lowering.cpp is absent)
Multi-GPU (torchrun): each rank executes its own replica (batch-sharded layer; no collective on
the compute path — "scaling": "weak"); the process group is used only for the barrier and the
max-over-ranks reduction of the timed region.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "constructed-kernel TFLOP/s or GB/s and % roofline per op; construction time (s)"

# BASELINE.json configs as reference op specs. conv2d is configs[1], the metric's
# single-GPU headline; the others run as the per-op suite.
WORKLOADS = {
    "conv2d": dict(op={"kind": "conv2d", "I": [16, 64, 58, 58], "K": [64, 64, 3, 3], "S": 1},
                   name="Conv2d ResNet-50 layer N=16 56x56x64->64 3x3 stride 1 (implicit GEMM, pre-padded 58x58 input)",
                   bound="tensor", unit="TFLOP/s"),
    "gemm": dict(op={"kind": "gemm", "M": 1024, "K": 1024, "N": 1024},
                 name="GEMM fp32 M=N=K=1024 (tf32 tensor cores)", bound="tensor", unit="TFLOP/s"),
    "gemm_fp32": dict(op={"kind": "gemm", "M": 1024, "K": 1024, "N": 1024},
                      name="GEMM fp32 M=N=K=1024 at fp32 accuracy (3xTF32 tensor cores, 1e-6 bar)",
                      bound="tensor", unit="TFLOP/s", variant="tc_3xtf32"),
    "bgemm": dict(op={"kind": "gemm", "M": 512, "K": 64, "N": 512, "dtype_bytes": 2, "batch": 192},
                  name="Batched GEMM bf16 B*H=192 512x64x512 (attention QK^T shape)", bound="hbm", unit="TFLOP/s"),
    "rowsum": dict(op={"kind": "gemv", "M": 32768, "N": 4096},
                   name="Row reduction 32768x4096 fp32 (gemv, x=1)", bound="hbm", unit="GB/s", ones_x=True),
    "softmax": dict(op={"kind": "softmax", "M": 32768, "N": 4096},
                    name="Softmax 32768x4096 fp32 (row-wise)", bound="hbm", unit="GB/s"),
    "dwconv": dict(op={"kind": "dwconv2d", "I": [32, 256, 114, 114], "K": [256, 1, 3, 3], "S": 1},
                   name="Depthwise conv 3x3 fp32 32x256x112x112", bound="hbm", unit="GB/s"),
    "avgpool": dict(op={"kind": "avgpool2d", "I": [32, 256, 114, 114], "F": 3, "S": 1},
                    name="AvgPool 3x3 s1 fp32 32x256x112x112", bound="hbm", unit="GB/s"),
}
SUITE_DEFAULT = ["gemm_fp32", "gemm", "bgemm", "rowsum", "softmax", "dwconv", "avgpool"]

# the B200 in the reference's own hardware format (for oracle/_ref).
B200_REF_HW = {
    "name": "b200-nominal", "peak_flops": 7.2e13, "clock_hz": 1.9e9,
    "levels": [
        {"name": "hbm3e", "capacity_bytes": "unlimited", "bandwidth_bytes_per_cycle": 4210, "latency_cycles": 800,
         "bank_width_elems": 0},
        {"name": "smem", "capacity_bytes": 232448, "bandwidth_bytes_per_cycle": 18944, "latency_cycles": 30,
         "bank_width_elems": 32},
        {"name": "regs", "capacity_bytes": 1020, "bandwidth_bytes_per_cycle": 227328, "latency_cycles": 1,
         "bank_width_elems": 0},
    ],
}


def measured_peaks() -> dict:
    for p in (os.path.join(ROOT, "MEASURED_PEAKS.json"),):
        if os.path.exists(p):
            with open(p) as f:
                d = json.load(f)
            d["source"] = "measured (MEASURED_PEAKS.json)"
            return d
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback (B200_PROFILING.md)"}


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return ws, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def shard_spec(spec: dict, ws: int, rank: int, strong: bool) -> tuple[dict, dict]:
    """This rank's share of a single-op workload (batch-sharded, no exchange).
    weak (default): a global batch of ws x the BASELINE batch, one BASELINE-sized shard of
    distinct images per rank; strong: the BASELINE batch itself split ws ways. The shard axis is
    the op's outer independent axis (conv/pool images, GEMM batch or rows, GEMV/softmax rows).
    Returns (this rank's op doc, a description of the global job)."""
    doc = json.loads(json.dumps(spec["op"]))
    if doc["kind"] in ("conv2d", "dwconv2d", "avgpool2d"):
        get = lambda d: d["I"][0]  # noqa: E731

        def put(d, v):
            d["I"][0] = v
    elif doc["kind"] == "gemm" and doc.get("batch", 1) > 1:
        get = lambda d: d["batch"]  # noqa: E731

        def put(d, v):
            d["batch"] = v
    else:
        get = lambda d: d["M"]  # noqa: E731

        def put(d, v):
            d["M"] = v
    base = get(doc)
    if strong:
        if base % ws:
            raise SystemExit(f"--strong: the batch {base} does not split {ws} ways")
        put(doc, base // ws)
        glob = {"global": base, "per_rank": base // ws, "scaling": "strong"}
    else:
        glob = {"global": base * ws, "per_rank": base, "scaling": "weak"}
    glob["rank_ranges"] = [[r * glob["per_rank"], (r + 1) * glob["per_rank"]] for r in range(ws)]
    return doc, glob


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without a launcher: re-run this command under torch.distributed.run
    with N ranks on 127.0.0.1 (one process per GPU) and relay its output."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


# ------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.proc = device, None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200", "-i",
                 str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------
def make_inputs(op, spec, rng, torch, device):
    """Synthetic inputs U(-1,1) of the op's true shapes (bf16 for dtype_bytes 2); rowsum x = 1."""
    dt = torch.bfloat16 if op.dtype_bytes == 2 else torch.float32
    xs = []
    for i, t in enumerate(op.tensors[:-1]):
        n = int(np.prod(t["true_dims"])) * op.batch
        if spec.get("ones_x") and i == 1:
            x = torch.ones(n, dtype=dt, device=device)
        else:
            x = (torch.rand(n, device=device, generator=rng) * 2 - 1).to(dt)
        xs.append(x)
    nout = int(np.prod(op.tensors[-1]["true_dims"])) * op.batch
    out = torch.empty(nout, dtype=dt, device=device)
    return xs, out


def tf32_peak(torch, device) -> float:
    """cuBLAS TF32 GEMM 8192^3, best of 5 (denominator for the tf32 tensor-core kernels)."""
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(8192, 8192, device=device)
    b = torch.randn(8192, 8192, device=device)
    for _ in range(2):
        a @ b
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        a @ b
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    torch.backends.cuda.matmul.allow_tf32 = False
    del a, b
    return 2 * 8192 ** 3 / best / 1e12


def run_op(g, torch, spec, hw, steps, warmup, device, variant="auto", flush=None, e2e=True, timing=True, seed=0,
           rerank=True):
    """Construct + instantiate + time one op. Returns a dict of measurements (this rank).
    rerank: the paper's flow — the engine's top-k schedules are instantiated and timed on the
    device (gensor_rerank) and the fastest one is the kernel; its time is reported apart."""
    op = g.TensorOpSpec.parse_text(json.dumps(spec["op"]))
    cfg = g.EngineConfig(seed=0, mode="b200")
    con = []
    sched = None
    for _ in range(5):
        t0 = time.perf_counter()
        sched = g.optimize(op, hw, cfg)
        con.append(time.perf_counter() - t0)
    rng = torch.Generator(device=device)
    rng.manual_seed(seed)
    xs, out = make_inputs(op, spec, rng, torch, device)
    stream = torch.cuda.current_stream(device)
    best, rr, rerank_s = 0, None, None
    if rerank and len(sched) > 1:
        t0 = time.perf_counter()
        rr = g.rerank(op, sched, xs, out, variant, iters=5, stream=stream)
        rerank_s = time.perf_counter() - t0
        best = rr["best"]
    k = g.Kernel(op, sched, best, variant)
    for _ in range(warmup):
        k.execute(xs, out, stream)
    torch.cuda.synchronize(device)

    # timed steps: no instrumentation inside the events
    step_ms, launch_ms = [], {}
    n0 = g.launch_count()
    for _ in range(steps):
        if flush is not None:
            flush_l2(torch, flush)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        k.execute(xs, out, stream)
        e.record(stream)
        e.synchronize()
        step_ms.append(s.elapsed_time(e))
    launches = g.launch_count() - n0
    # per-launch breakdown (roofline): separate pass with events around every internal launch
    if timing:
        k.set_timing(True)
        for _ in range(max(3, steps // 2)):
            if flush is not None:
                flush_l2(torch, flush)
            k.execute(xs, out, stream)
            for name, ms in k.timings():
                launch_ms.setdefault(name, []).append(ms)
        k.set_timing(False)
    res = dict(op=op, kernel=k, sched=sched, step_ms=step_ms, launch_ms=launch_ms, launches=launches,
               construct_s=statistics.median(con), flops=op.flops, bytes=op.bytes, index=best,
               rerank=None if rr is None else {"ms": rr["ms"], "best": best, "wall_s": rerank_s,
                                               "plans_differ": len({json.dumps(p) for p in rr.get("plans", [])}) > 1})
    if e2e:
        hin = [x.cpu().pin_memory() for x in xs]
        hout = torch.empty(out.numel(), dtype=out.dtype).pin_memory()
        k.set_timing(False)
        k.execute_host(hin, hout, stream)  # warm the staging buffers
        e2e_ms = []
        for _ in range(max(3, steps // 2)):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            k.execute_host(hin, hout, stream)
            e.record(stream)
            e.synchronize()
            e2e_ms.append(s.elapsed_time(e))
        res["e2e_ms"] = e2e_ms
        res["host_pipe"] = k.info.get("host_pipe")  # chunked H2D / kernel / D2H overlap, if used
        res["h2d"] = sum(x.numel() * x.element_size() for x in hin)
        res["d2h"] = hout.numel() * hout.element_size()
        if not torch.equal(hout.to(device), out):
            raise RuntimeError("host-buffer execute disagrees with device execute")
    return res


def flush_l2(torch, flush):
    """Between timed steps: flush L2 (a 256 MiB write, outside the events), then keep the device
    busy ~0.5 ms (torch.cuda._sleep) so the host-side enqueue of the next execute overlaps device
    work — the events then bracket device time only, not the Python call's latency (the e2e
    number is the one that includes the host path)."""
    flush.zero_()
    torch.cuda._sleep(1_000_000)


def roofline(res, spec, peaks, tf32_tflops, variant_name, traffic=(None, None)):
    traffic, traffic_detail = traffic
    name, ms = max(res["launch_ms"].items(), key=lambda kv: statistics.mean(kv[1]))
    avg = statistics.mean(ms) / 1e3
    if spec["bound"] == "tensor":
        achieved = res["flops"] / avg / 1e12
        if variant_name == "tc_tf32":
            peak, src = tf32_tflops, "cuBLAS tf32 8192^3 measured in this run (best of 5)"
        elif variant_name == "tc_3xtf32":  # three tf32 MMAs per fp32 product
            peak, src = tf32_tflops / 3, "cuBLAS tf32 8192^3 measured in this run / 3 (3 MMAs per product)"
        else:
            peak, src = peaks["bf16_tflops"], f"bf16 dense, {peaks['source']}"
        r = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
             "traffic": traffic, "kernel": name, "peak_source": src,
             "share_of_step": statistics.mean(ms) / statistics.mean(res["step_ms"])}
    else:
        achieved = res["bytes"] / avg / 1e9
        peak = peaks["hbm_gbs"]
        r = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
             "traffic": traffic, "kernel": name, "peak_source": f"hbm copy, {peaks['source']}",
             "share_of_step": statistics.mean(ms) / statistics.mean(res["step_ms"])}
    r["algorithmic_per_launch"] = res["flops"] if spec["bound"] == "tensor" else res["bytes"]
    r["traffic_detail"] = traffic_detail
    r["algorithmic_bytes"] = res["bytes"]
    return r


def ncu_traffic(workload):
    """DRAM bytes (read + write) of every launch of one execute, from ncu (profiles/ncu_traffic.json,
    tools/gpu_traffic.sh), and the detail: output lines still dirty in L2 at kernel end are not in
    dram_write, so the store traffic the kernels sent to L2 is listed beside it."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            t = json.load(f)
        if workload in t:
            det = t.get(workload + "_detail", {})
            return t[workload], {k: det.get(k) for k in ("dram_read", "dram_write", "l2_write_from_sm", "launches")}
    return None, None


def _pow2(x: int) -> int:
    p = 1
    while p < x:
        p *= 2
    return p


def op_geom(doc: dict) -> dict:
    """Axes (name, true extent, padded extent), tensor element counts (inputs..., output), and the
    algorithmic FLOPs / compulsory bytes on true extents of a reference op description — plain
    Python (op_spec.cpp:70-196 axis orders), so the reference and CPU legs never load the product
    library."""
    k, dt, batch = doc["kind"], doc.get("dtype_bytes", 4), doc.get("batch", 1)
    if k == "gemm":
        M, K, N = doc["M"], doc["K"], doc["N"]
        axes, elems = [("m", M), ("n", N), ("k", K)], [M * K, K * N, M * N]
    elif k in ("gemv", "softmax"):
        M, N = doc["M"], doc["N"]
        axes = [("m", M), ("n", N)]
        elems = [M * N, N, M] if k == "gemv" else [M * N, M * N]
    else:
        n, c, h, w = doc["I"]
        st = doc.get("S", 1)
        if k == "avgpool2d":
            r = s_ = doc["F"]
        else:
            r, s_ = doc["K"][2], doc["K"][3]
        oh, ow = (h - r) // st + 1, (w - s_) // st + 1
        if k == "conv2d":
            f = doc["K"][0]
            axes = [("n", n), ("f", f), ("h", oh), ("w", ow), ("c", c), ("r", r), ("s", s_)]
            elems = [n * c * h * w, f * c * r * s_, n * f * oh * ow]
        elif k == "dwconv2d":
            axes = [("n", n), ("c", c), ("h", oh), ("w", ow), ("r", r), ("s", s_)]
            elems = [n * c * h * w, c * r * s_, n * c * oh * ow]
        else:
            axes = [("n", n), ("c", c), ("h", oh), ("w", ow), ("i", r), ("j", s_)]
            elems = [n * c * h * w, n * c * oh * ow]
    iters = float(np.prod([float(e) for _, e in axes])) * batch
    flops = iters if k == "avgpool2d" else (5 * iters if k == "softmax" else 2 * iters)
    return {"axes": [(a, e, _pow2(e)) for a, e in axes], "elems": [e * batch for e in elems], "flops": flops,
            "bytes": float(sum(elems)) * dt * batch, "dtype_bytes": dt, "batch": batch}


def cpu_baseline(spec, sched_state, budget_s=12.0):
    """The oracle's interpret() of the constructed schedule on a bounded sample, all threads."""
    from oracle import oracle as O

    doc = dict(spec["op"])
    threads = os.cpu_count() or 1
    kind = doc["kind"]
    # sample: shrink the outermost batch-like dimension
    if kind in ("conv2d", "dwconv2d", "avgpool2d"):
        full = doc["I"][0]
        key = ("I", 0)
    elif kind == "gemm":
        full = doc.get("batch", 1) if doc.get("batch", 1) > 1 else doc["M"]
        key = ("batch",) if doc.get("batch", 1) > 1 else ("M",)
    else:
        full = doc["M"]
        key = ("M",)

    def sized(n):
        d = json.loads(json.dumps(doc))
        if key[0] == "I":
            d["I"][0] = n
        else:
            d[key[0]] = n
        return d

    def run(n):
        d = sized(n)
        geo = op_geom(d)
        # the sample shrinks one extent: clamp the schedule's tiles to the sample's padded extents
        st = {"tiles": [[min(t, a[2]) for t in per] for per, a in zip(sched_state["tiles"], geo["axes"])],
              "vthreads": [min(v, min(a[2], per[-1]) if per else v)
                           for v, per, a in zip(sched_state["vthreads"], sched_state["tiles"], geo["axes"])]}
        rng = np.random.default_rng(0)
        xs = [rng.uniform(-1, 1, e).astype(np.float32) for e in geo["elems"][:-1]]
        t0 = time.perf_counter()
        O.interpret(d, st, xs, threads=threads)
        return time.perf_counter() - t0, geo["flops"], geo["bytes"]

    n = 1
    dt, fl, by = run(n)
    while dt < budget_s / 4 and n < full:
        n = min(full, n * 2 if dt < budget_s / 8 else n + 1)
        dt, fl, by = run(n)
    unit = spec["unit"]
    value = fl / dt / 1e12 if unit == "TFLOP/s" else by / dt / 1e9
    return {"value": value, "unit": unit, "cores": threads, "kind": "port",
            "sample": f"{kind} with the outer dim {key[0]}={n} of {full}: {fl:.3e} FLOP in {dt:.2f} s "
                      f"(oracle/gensor_oracle.c interpret() of the same schedule, OpenMP {threads} threads)"}


def reference_construct_s(spec):
    from oracle import ref

    if not ref.available():
        return None
    r = ref.optimize(spec["op"], B200_REF_HW, {"seed": 0})
    return r.get("wall_s")


# ------------------------------------------------------------------------------------------
def run_reference(args):
    """--impl reference: the reference's CPU path (construct with its own library + the
    restated interpreter), rank 0 only, all host threads, bounded sample per step."""
    ws, rank, _ = dist_info()
    if rank != 0:
        return
    spec = WORKLOADS[args.workload]
    from oracle import ref  # the reference's own construct library; never the product package

    op_doc = spec["op"]
    if ref.available():
        con = ref.optimize(op_doc, B200_REF_HW, {"seed": 0})
        state = con["results"][0]["state"]
        construct_kind = "reference (oracle/_ref: unmodified proj/src)"
    else:  # reference library absent: the schedule-independent naive loop nest (level-less state)
        state = {"tiles": [[] for _ in op_geom(op_doc)["axes"]], "vthreads": [1] * len(op_geom(op_doc)["axes"])}
        construct_kind = "none (oracle/_ref not built): interpret() of the unscheduled loop nest"
    base = cpu_baseline(spec, state, budget_s=args.ref_budget)
    times = []
    for _ in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        if ref.available():
            ref.optimize(op_doc, B200_REF_HW, {"seed": 0})
        times.append(time.perf_counter() - t0)
    con_s = statistics.median(times[args.warmup:]) if times[args.warmup:] else None
    line = {"impl": "reference", "metric": METRIC, "value": base["value"], "unit": spec["unit"],
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64 accumulate (fp32 data)", "data": "synthetic U(-1,1)",
            "config": {"workload": spec["name"], "op": op_doc, "parallelism": "rank 0 only, host cores"},
            "cpu_baseline": {**base},
            "e2e": {"value": base["value"], "unit": spec["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "construction_s": con_s, "construction_kind": construct_kind, "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
SEQUENCE_NAMES = {"resnet50": "End-to-end ResNet-50 operator sequence (53 convs + pools + fc, global batch 128)",
                  "gpt2": "End-to-end GPT-2 small operator sequence (12 layers + LM head, global batch 16 x 512)"}


def run_sequence(g, torch, name, hw, steps, warmup, device, ws, flush):
    """configs[4]: every op of the batch-sharded sequence constructed once (per distinct spec) and
    executed in order each step. e2e: the shard's input batch H2D + the final output D2H around
    the same on-device sequence (weights and intermediates stay resident)."""
    from paper_2502_11407_b200 import sequences as S

    seq = S.sharded(name, ws)
    kern, con = {}, {}
    gen = torch.Generator(device=device)
    gen.manual_seed(0)
    for key, spec_op in S.distinct(seq).items():
        op = g.TensorOpSpec.parse_text(json.dumps(spec_op))
        t0 = time.perf_counter()
        sched = g.optimize(op, hw, g.EngineConfig(seed=0, mode="b200"))
        con[key] = time.perf_counter() - t0
        kern[key] = (op, g.Kernel(op, sched, 0, "auto"))
    keys = [json.dumps(sp, sort_keys=True) for _, sp in seq]
    # per-instance buffers, chained: an op whose first input has the element count and dtype of the
    # previous op's output reads that output buffer (ResNet: conv3 -> next conv1 / conv2 -> conv3;
    # GPT-2: qk -> softmax -> pv -> proj -> fc1 -> fc2 -> next qkv); other inputs are synthetic.
    # Weights are U(-1,1) * sqrt(3 / reduction) so chained activations keep unit scale.
    bufs, chained = [], 0
    for i, key in enumerate(keys):
        op, _ = kern[key]
        xs, out = make_inputs(op, {"op": seq[i][1]}, gen, torch, device)
        red = {"gemm": "K", "conv2d": None}.get(seq[i][1]["kind"])
        if red == "K":
            xs[1].mul_(math.sqrt(3.0 / seq[i][1]["K"]))
        elif seq[i][1]["kind"] == "conv2d":
            kk = seq[i][1]["K"]
            xs[1].mul_(math.sqrt(3.0 / (kk[1] * kk[2] * kk[3])))
        if bufs and bufs[-1][1].numel() == xs[0].numel() and bufs[-1][1].dtype == xs[0].dtype:
            xs[0] = bufs[-1][1]
            chained += 1
        bufs.append((xs, out))
    stream = torch.cuda.current_stream(device)

    def step():
        for i, key in enumerate(keys):
            kern[key][1].execute(bufs[i][0], bufs[i][1], stream)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize(device)
    # per-op breakdown (one extra pass, events between ops)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(keys) + 1)]
    ev[0].record(stream)
    for i, key in enumerate(keys):
        kern[key][1].execute(bufs[i][0], bufs[i][1], stream)
        ev[i + 1].record(stream)
    ev[-1].synchronize()
    per_op = {}
    for i, (opname, _) in enumerate(seq):
        key = keys[i]
        ms = ev[i].elapsed_time(ev[i + 1])
        kind = opname.split(".")[-1] if name == "gpt2" else ("conv" if "conv" in opname or "downsample" in opname else opname)
        d = per_op.setdefault(kind, {"ms": 0.0, "flops": 0.0, "bytes": 0.0, "n": 0,
                                     "variant": kern[key][1].info["variant_name"]})
        d["ms"] += ms
        d["flops"] += kern[key][0].flops
        d["bytes"] += kern[key][0].bytes
        d["n"] += 1
    # the timed steps replay the sequence from a CUDA graph captured once (the same launches with
    # the host out of the loop: -2..4 % on GPT-2 / ResNet-50); eager launches if capture fails
    graph, per_step = None, 0
    try:
        side = torch.cuda.Stream(device)
        side.wait_stream(stream)
        c0 = g.launch_count()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            cap = torch.cuda.current_stream(device)
            for i, key in enumerate(keys):
                kern[key][1].execute(bufs[i][0], bufs[i][1], cap)
        per_step = g.launch_count() - c0
        torch.cuda.synchronize(device)
    except Exception as exc:  # pragma: no cover - driver without graph support for these launches
        print(f"[bench] CUDA graph capture failed ({exc}); timing eager launches", file=sys.stderr)
        graph = None
    n0 = g.launch_count()
    step_ms = []
    for _ in range(steps):
        flush_l2(torch, flush)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        if graph is not None:
            graph.replay()
        else:
            step()
        e.record(stream)
        e.synchronize()
        step_ms.append(s.elapsed_time(e))
    launches = per_step * steps if graph is not None else g.launch_count() - n0
    flops = sum(kern[k][0].flops for k in keys)
    # e2e: the shard's input batch from pinned host memory, the final output back
    hin = bufs[0][0][0].cpu().pin_memory()
    hout = torch.empty(bufs[-1][1].numel(), dtype=bufs[-1][1].dtype).pin_memory()
    e2e_ms = []
    for _ in range(max(3, steps // 2)):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        bufs[0][0][0].copy_(hin, non_blocking=True)
        step()
        hout.copy_(bufs[-1][1], non_blocking=True)
        e.record(stream)
        e.synchronize()
        e2e_ms.append(s.elapsed_time(e))
    return dict(seq=seq, step_ms=step_ms, e2e_ms=e2e_ms, per_op=per_op, launches=launches, flops=flops,
                graph=graph is not None, chained=chained,
                construct_s=sum(con.values()), n_distinct=len(con), h2d=hin.numel() * hin.element_size(),
                d2h=hout.numel() * hout.element_size())


def sequence_line(args, res, ws, peaks, tf32, clk, total_ms, e2e_ms):
    ms_step = total_ms / args.steps
    value = ws * res["flops"] / (ms_step / 1e3) / 1e12
    e2e_value = ws * res["flops"] / (e2e_ms / 1e3) / 1e12
    per_op = {}
    for kind, d in res["per_op"].items():
        per_op[kind] = {"n": d["n"], "ms": d["ms"], "share": d["ms"] / sum(x["ms"] for x in res["per_op"].values()),
                        "tflops": d["flops"] / (d["ms"] / 1e3) / 1e12, "gbs": d["bytes"] / (d["ms"] / 1e3) / 1e9,
                        "variant": d["variant"]}
    top = max(per_op.items(), key=lambda kv: kv[1]["ms"])
    d = res["per_op"][top[0]]
    variant = d["variant"]
    if variant in ("stream",):
        ach, peak, unit, bound = d["bytes"] / (d["ms"] / 1e3) / 1e9, peaks["hbm_gbs"], "GB/s", "hbm"
        src = f"hbm copy, {peaks['source']}"
    else:
        ach = d["flops"] / (d["ms"] / 1e3) / 1e12
        peak = tf32 if variant == "tc_tf32" else peaks["bf16_tflops"]
        src = "cuBLAS tf32 8192^3 measured in this run" if variant == "tc_tf32" else f"bf16 dense, {peaks['source']}"
        unit, bound = "TFLOP/s", "tensor"
    dt = {"resnet50": "tf32 convs / fp32 pools (fp32 storage)", "gpt2": "bf16 GEMMs (fp32 accumulate), fp32 softmax"}
    return {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": dt[args.workload], "data": "synthetic U(-1,1)",
        "config": {"workload": SEQUENCE_NAMES[args.workload], "ops": len(res["seq"]),
                   "launch": "CUDA graph of the step (captured once, replayed per step)" if res.get("graph")
                   else "eager stream launches",
                   "distinct_ops": res["n_distinct"],
                   "chained_inputs": res.get("chained"),
                   "parallelism": f"batch-sharded over {ws} GPU(s), one process per GPU, no collective",
                   "l2": "flushed between steps (256 MiB write outside the events)"},
        "roofline": {"bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
                     "traffic": None, "kernel": f"{top[0]} ({variant})", "peak_source": src,
                     "share_of_step": top[1]["share"]},
        "per_op": per_op,
        "e2e": {"value": e2e_value, "unit": "TFLOP/s", "h2d_bytes_per_step": res["h2d"],
                "d2h_bytes_per_step": res["d2h"], "ms_per_step": e2e_ms,
                "path": "input batch H2D + on-device sequence + final output D2H"},
        "gpu_launches": res["launches"], "construction_s": res["construct_s"], "clocks": clk.summary(),
        "cpu_baseline": None,
    }


def run_suite_sharded(args, g, torch, hw, peaks, tf32, flush, device, ws, rank, local, pg, barrier):
    """--workload suite: the independent operator suite (BASELINE configs[0..3]) dealt to the ranks
    by LPT on the engine's B200 cost estimate (paper_2502_11407_b200/shard.py); each rank runs its
    share; value = total suite FLOPs / (max over ranks of the summed device time)."""
    from paper_2502_11407_b200 import shard

    names = ["conv2d"] + SUITE_DEFAULT
    docs = [WORKLOADS[n]["op"] for n in names]
    parts = shard.suite_partition(docs, hw, ws, [WORKLOADS[n].get("variant", "auto") for n in names])
    mine = parts[rank]
    results, total_ms = {}, 0.0
    barrier()
    with ClockSampler(local) as clk:
        for i in mine:
            spec = WORKLOADS[names[i]]
            r = run_op(g, torch, spec, hw, args.steps, args.warmup, device, spec.get("variant", "auto"), flush,
                       e2e=False)
            ms = statistics.mean(r["step_ms"])
            total_ms += ms
            results[names[i]] = {"ms": ms, "flops": r["flops"], "bytes": r["bytes"], "rank": rank,
                                 "variant": r["kernel"].info["variant_name"]}
    barrier()
    all_res = [results]
    t = total_ms
    if pg:
        t_t = torch.tensor([total_ms], device=device, dtype=torch.float64)
        pg.all_reduce(t_t, op=pg.ReduceOp.MAX)
        t = t_t.item()
        all_res = [None] * ws
        pg.all_gather_object(all_res, results)
    if rank == 0:
        merged = {k: v for d in all_res for k, v in d.items()}
        flops = sum(v["flops"] for v in merged.values())
        line = {"metric": METRIC, "value": flops / (t / 1e3) / 1e12, "unit": "TFLOP/s", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": t, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "per op (tf32 / bf16 / f32)",
                "data": "synthetic U(-1,1)",
                "config": {"workload": "operator suite (configs[0..3]) LPT-partitioned over GPUs",
                           "partition": [[names[i] for i in p] for p in parts],
                           "parallelism": f"{ws} GPU(s), one process per GPU, no collective"},
                "per_op": merged, "clocks": clk.summary(), "roofline": None, "e2e": None,
                "gpu_launches": None}
        print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()


GRAPH_VS_TREE = {  # the families `auto` runs: tensor cores for G / B / C, the HBM family for V / P
    "gemm": {"kind": "gemm", "M": 1024, "K": 1024, "N": 1024},
    "bgemm": {"kind": "gemm", "M": 512, "K": 64, "N": 512, "dtype_bytes": 2, "batch": 192},
    "conv2d": {"kind": "conv2d", "I": [16, 64, 58, 58], "K": [64, 64, 3, 3], "S": 1},
    "gemv": {"kind": "gemv", "M": 32768, "N": 4096},
    "avgpool2d": {"kind": "avgpool2d", "I": [32, 256, 114, 114], "F": 3, "S": 1},
}


def run_graph_vs_tree(args, g, torch, hw, flush, device):
    """SURVEY.md §8f rank 2 / the paper's core claim (graph construction >= tree construction,
    PAPER.md:577): the kernel `auto` runs (tcgen05 for the GEMMs and the conv, the
    HBM-streaming family for the row / window ops) instantiated from the graph-constructed
    schedule (optimize, B200 mode), from the on-device re-ranked top-k of the graph, and from the
    Roller-style tree schedule (construct_tree, B200 mode), timed on B200."""
    out = {}
    variant = getattr(args, "variant", "auto")
    for name, doc in GRAPH_VS_TREE.items():
        op = g.TensorOpSpec.parse_text(json.dumps(doc))
        gen = torch.Generator(device=device)
        gen.manual_seed(0)
        xs, o = make_inputs(op, {"op": doc}, gen, torch, device)
        graph = g.optimize(op, hw, g.EngineConfig(seed=0, mode="b200", top_k=10))
        tree = g.construct_tree(op, hw, 4, "b200")

        def timed(sched, idx):
            k = g.Kernel(op, sched, idx, variant)
            for _ in range(3):
                k.execute(xs, o)
            ts = []
            for _ in range(max(5, args.steps)):
                flush_l2(torch, flush)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                k.execute(xs, o)
                e.record()
                e.synchronize()
                ts.append(s.elapsed_time(e))
            return statistics.median(ts), k.info["plan"]

        t_graph, p_graph = timed(graph, 0)
        rr = g.rerank(op, graph, xs, o, variant, iters=5)
        t_rerank, p_rerank = timed(graph, rr["best"])
        t_tree, p_tree = timed(tree, 0)
        unit_work = op.flops if doc["kind"] in ("gemm", "conv2d") else op.bytes
        scale, unit = (1e12, "TFLOP/s") if doc["kind"] in ("gemm", "conv2d") else (1e9, "GB/s")
        distinct = sorted({json.dumps(p, sort_keys=True) for p in rr["plans"] if p})
        out[name] = {"unit": unit,
                     "graph": {"ms": t_graph, "value": unit_work / (t_graph / 1e3) / scale,
                               "schedule": graph[0]["state"]["repr"], "plan": p_graph,
                               "est_ms": graph[0]["cost"].get("exec_seconds", graph[0]["cost"]["est_seconds"]) * 1e3},
                     "graph_reranked": {"ms": t_rerank, "value": unit_work / (t_rerank / 1e3) / scale,
                                        "schedule": graph[rr["best"]]["state"]["repr"], "index": rr["best"],
                                        "plan": p_rerank},
                     "tree": {"ms": t_tree, "value": unit_work / (t_tree / 1e3) / scale,
                              "schedule": tree[0]["state"]["repr"], "plan": p_tree,
                              "est_ms": tree[0]["cost"].get("exec_seconds", tree[0]["cost"]["est_seconds"]) * 1e3},
                     "topk_rerank_ms": rr["ms"], "topk_distinct_plans": len(distinct),
                     "graph_over_tree": t_tree / t_graph, "reranked_over_tree": t_tree / t_rerank}
    geo = float(np.exp(np.mean([np.log(v["graph_over_tree"]) for v in out.values()])))
    geo_rr = float(np.exp(np.mean([np.log(v["reranked_over_tree"]) for v in out.values()])))
    line = {"metric": "graph vs tree construction: measured B200 time of the kernel auto runs (speed-up)",
            "value": geo, "unit": "x (geomean tree time / graph time)", "reranked_geomean": geo_rr,
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "per op (tf32 / bf16 / f32)", "data": "synthetic U(-1,1)",
            "config": {"workload": "graph_vs_tree", "variant": variant,
                       "l2": "flushed between steps (256 MiB write outside the events)"},
            "per_op": out}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch

    import paper_2502_11407_b200 as g

    ws, rank, local = dist_info()
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    pg = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=device)
        pg = dist
    peaks = measured_peaks()
    hw = g.HardwareSpec.b200(local, {"hbm_gbs": peaks["hbm_gbs"], "bf16_tflops": peaks["bf16_tflops"]})
    tf32 = tf32_peak(torch, device)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)  # 2x L2: flushed between steps

    def barrier():
        torch.cuda.synchronize(device)
        if pg:
            pg.barrier()
        torch.cuda.synchronize(device)

    if args.workload == "graph_vs_tree":
        if rank == 0:
            run_graph_vs_tree(args, g, torch, hw, flush, device)
        if pg:
            pg.destroy_process_group()
        return

    if args.workload == "suite":
        run_suite_sharded(args, g, torch, hw, peaks, tf32, flush, device, ws, rank, local, pg, barrier)
        return

    if args.workload in SEQUENCE_NAMES:
        barrier()
        with ClockSampler(local) as clk:
            res = run_sequence(g, torch, args.workload, hw, args.steps, args.warmup, device, ws, flush)
        barrier()
        total_ms, e2e_ms = sum(res["step_ms"]), statistics.mean(res["e2e_ms"])
        if pg:
            t = torch.tensor([total_ms, e2e_ms], device=device, dtype=torch.float64)
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            total_ms, e2e_ms = t.tolist()
        if rank == 0:
            print(json.dumps(sequence_line(args, res, ws, peaks, tf32, clk, total_ms, e2e_ms)), flush=True)
        if pg:
            pg.destroy_process_group()
        return

    # this rank's batch shard (weak by default: a BASELINE-sized shard of distinct images per rank)
    doc, glob = shard_spec(WORKLOADS[args.workload], ws, rank, args.strong)
    spec = dict(WORKLOADS[args.workload], op=doc)

    barrier()
    with ClockSampler(local) as clk:
        res = run_op(g, torch, spec, hw, args.steps, args.warmup, device, args.variant, flush, seed=rank)
    barrier()
    total_ms = sum(res["step_ms"])
    e2e_ms = statistics.mean(res["e2e_ms"])
    if pg:
        t = torch.tensor([total_ms, e2e_ms], device=device, dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        total_ms, e2e_ms = t.tolist()
    ms_step = total_ms / args.steps
    work = res["flops"] if spec["unit"] == "TFLOP/s" else res["bytes"]
    scale = 1e12 if spec["unit"] == "TFLOP/s" else 1e9
    value = ws * work / (ms_step / 1e3) / scale
    e2e_value = ws * work / (e2e_ms / 1e3) / scale
    info = res["kernel"].info
    rl = roofline(res, spec, peaks, tf32, info["variant_name"], ncu_traffic(args.workload))

    suite = {}
    if args.suite and ws == 1:
        for wname in args.suite.split(","):
            if not wname or wname == args.workload:
                continue
            try:
                sp = WORKLOADS[wname]
                r = run_op(g, torch, sp, hw, max(5, args.steps), max(3, args.warmup), device,
                           sp.get("variant", "auto"), flush, e2e=False)
                ki = r["kernel"].info
                w = r["flops"] if sp["unit"] == "TFLOP/s" else r["bytes"]
                srl = roofline(r, sp, peaks, tf32, ki["variant_name"], ncu_traffic(wname))
                suite[wname] = {
                    "variant": ki["variant_name"], "family": ki["plan"].get("family"),
                    "value": w / (statistics.mean(r["step_ms"]) / 1e3) / (1e12 if sp["unit"] == "TFLOP/s" else 1e9),
                    "unit": sp["unit"], "ms_per_step": statistics.mean(r["step_ms"]),
                    "roofline": {k: srl[k] for k in ("bound", "achieved", "peak", "frac", "traffic", "kernel")},
                    "construction_s": r["construct_s"],
                }
                del r
            except Exception as exc:  # keep the headline line even if a suite op fails
                suite[wname] = {"error": str(exc)[:300]}
            torch.cuda.empty_cache()

    sequences = {}
    if ws == 1 and not args.no_sequences:
        # configs[4] on one GPU, summarised into the default line (the full lines: --workload resnet50|gpt2)
        for sname in ("resnet50", "gpt2"):
            try:
                sargs = argparse.Namespace(**{**vars(args), "workload": sname, "steps": 5, "warmup": 2})
                with ClockSampler(local) as sclk:
                    sres = run_sequence(g, torch, sname, hw, sargs.steps, sargs.warmup, device, ws, flush)
                sl = sequence_line(sargs, sres, ws, peaks, tf32, sclk, sum(sres["step_ms"]),
                                   statistics.mean(sres["e2e_ms"]))
                sequences[sname] = {k: sl[k] for k in ("value", "unit", "ms_per_step", "steps", "gpu_launches",
                                                       "construction_s")}
                sequences[sname]["e2e"] = {k: sl["e2e"][k] for k in ("value", "unit", "ms_per_step")}
                sequences[sname]["roofline_top_op"] = {k: sl["roofline"][k] for k in ("kernel", "achieved", "peak",
                                                                                      "frac", "share_of_step")}
                sequences[sname]["config"] = {k: sl["config"][k] for k in ("workload", "ops", "distinct_ops",
                                                                          "chained_inputs", "launch")}
                del sres
            except Exception as exc:  # keep the headline line even if a sequence fails
                sequences[sname] = {"error": str(exc)[:300]}
            torch.cuda.empty_cache()

    base = None
    ref_con = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        base = cpu_baseline(spec, res["sched"][res["index"]]["state"], budget_s=args.ref_budget)
        ref_con = reference_construct_s(spec)

    if rank != 0:
        if pg:
            pg.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": spec["unit"], "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": glob["scaling"],
        "vs_baseline": None,
        "dtype": {"tc_tf32": "tf32 (fp32 storage, fp32 accumulate)", "tc_bf16": "bf16 (fp32 accumulate)",
                  "tc_3xtf32": "fp32-grade 3xTF32 (fp32 storage, fp32 accumulate)",
                  "simt_f32": "f32", "simt_parity": "f64 accumulate", "stream": "f32"}[info["variant_name"]],
        "data": "synthetic U(-1,1)",
        "config": {"workload": spec["name"], "op": spec["op"], "variant": info["variant_name"],
                   "schedule": info["state"]["repr"], "kernel_plan": info["plan"], "engine": "b200 mode",
                   "l2": "flushed between steps (256 MiB write outside the events)",
                   "batch": glob,
                   "parallelism": (f"{glob['scaling']}: global batch {glob['global']} sharded {glob['per_rank']} per rank "
                                   f"over {ws} GPU(s) (distinct synthetic data per rank), one process per GPU, "
                                   "no collective on the compute path")},
        "roofline": rl,
        "e2e": {"value": e2e_value, "unit": spec["unit"], "h2d_bytes_per_step": res["h2d"],
                "d2h_bytes_per_step": res["d2h"], "ms_per_step": e2e_ms,
                "path": "gensor_execute_host (pinned host buffers)", "pipeline": res.get("host_pipe")},
        "gpu_launches": res["launches"],
        "step_ms_distribution": {"median": statistics.median(res["step_ms"]), "min": min(res["step_ms"]),
                                 "max": max(res["step_ms"])},
        "launch_breakdown_ms": {n: statistics.mean(v) for n, v in res["launch_ms"].items()},
        "construction_s": res["construct_s"],
        "schedule_index": res["index"], "rerank": res["rerank"],
        "construction_reference_s": ref_con,
        "clocks": clk.summary(),
        "cpu_baseline": base,
        "suite": suite or None,
        "sequences": sequences or None,
    }
    print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()


def run_dry(args):
    """--dry-run: the multi-rank plumbing without a GPU (gloo): every rank derives its shard of the
    workload, runs `steps` timed host-side placeholder steps (a sleep proportional to its shard
    and rank, standing in for the device work), and the timed region goes through the same
    barrier + max-over-ranks reduction as the real run. Tests drive it with --gpus 2."""
    import torch

    ws, rank, _ = dist_info()
    pg = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")
        pg = dist
    spec = WORKLOADS[args.workload]
    doc, glob = shard_spec(spec, ws, rank, args.strong)
    geo = op_geom(doc)
    if pg:
        pg.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        time.sleep(0.002 * (rank + 1))
    ms = (time.perf_counter() - t0) * 1e3
    if pg:
        pg.barrier()
    per_rank = [None] * ws
    t = torch.tensor([ms], dtype=torch.float64)
    if pg:
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        pg.all_gather_object(per_rank, {"rank": rank, "op": doc, "ms": ms, "flops": geo["flops"]})
    else:
        per_rank = [{"rank": 0, "op": doc, "ms": ms, "flops": geo["flops"]}]
    if rank == 0:
        total = t.item()
        flops = sum(r["flops"] for r in per_rank)
        print(json.dumps({"metric": METRIC, "dry_run": True, "value": flops / (total / args.steps / 1e3) / 1e12,
                          "unit": "TFLOP/s (placeholder timing)", "n_gpus": ws, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": total / args.steps, "scaling": glob["scaling"],
                          "config": {"workload": spec["name"], "batch": glob, "backend": "gloo" if pg else None},
                          "ranks": per_rank}), flush=True)
    if pg:
        pg.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS) + sorted(SEQUENCE_NAMES) + ["suite", "graph_vs_tree"], default="conv2d")
    ap.add_argument("--variant", default="auto")
    ap.add_argument("--suite", default=",".join(SUITE_DEFAULT))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sequences", action="store_true",
                    help="skip the ResNet-50 / GPT-2 sequence summaries of the default line")
    ap.add_argument("--ref-budget", type=float, default=12.0)
    ap.add_argument("--strong", action="store_true",
                    help="N>1: split the BASELINE batch N ways (default: one BASELINE-sized shard per rank)")
    ap.add_argument("--dry-run", action="store_true",
                    help="no GPU: exercise the rank plumbing (gloo) and the sharding; no kernels")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

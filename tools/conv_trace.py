"""Developer timeline of the headline conv (needs the DEV build: make -C paper_2502_11407_b200/csrc
DEV=1 after touching kernels/{exec,conv_tc}.cu). Prints (1) device time of pre-pass only, conv
only (stale workspace) and both, L2 flushed between steps, and (2) the per-CTA clock64 marks of
k_conv_ns (slots: 0 start, 1 griddep wait done, 2 first filters+A ready, 8+i MMA tile i start,
16+i MMA tile i committed, 24+i epilogue got tile i, 32+i epilogue done with tile i, 40 end)."""
import ctypes
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2502_11407_b200 as g  # noqa: E402

doc = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {"kind": "conv2d", "I": [16, 64, 58, 58], "K": [64, 64, 3, 3], "S": 1}
op = g.TensorOpSpec.parse_text(json.dumps(doc))
s = g.optimize(op, g.HardwareSpec.b200(0), g.EngineConfig(mode="b200", top_k=1))
k = g.Kernel(op, s, 0, "auto")
print(k.info["plan"])
xs = [torch.rand(int(np.prod(t["true_dims"])), device="cuda") * 2 - 1 for t in op.tensors[:-1]]
out = torch.empty(int(np.prod(op.tensors[-1]["true_dims"])), device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    k.execute(xs, out)
torch.cuda.synchronize()


def timed(n=30):
    ts = []
    for _ in range(n):
        flush.zero_()
        torch.cuda._sleep(80_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        k.execute(xs, out)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


if k.info["plan"]["family"] == "conv_flat":
    print(f"conv_flat step (events, L2 flushed): {timed():.2f} us", flush=True)
for mode in (() if k.info["plan"]["family"] == "conv_flat" else (None, "prepass", "conv")):
    if mode:
        os.environ["GENSOR_CONV_SKIP"] = mode
    else:
        os.environ.pop("GENSOR_CONV_SKIP", None)
    print(f"skip={mode}: {timed():.2f} us", flush=True)
os.environ.pop("GENSOR_CONV_SKIP", None)
lib = g.gensor.lib()
fam = k.info["plan"]["family"]
fn = lib.gensor_dev_flat_trace if fam == "conv_flat" else lib.gensor_dev_conv_trace
fn.argtypes = [ctypes.POINTER(ctypes.c_longlong), ctypes.c_int]
buf = (ctypes.c_longlong * (160 * 64))()
flush.zero_()
torch.cuda.synchronize()
torch.cuda._sleep(200_000)  # as the bench: the host enqueues while the device is busy
k.execute(xs, out)
torch.cuda.synchronize()
assert fn(buf, 160 * 64) == 0
tr = np.array(buf, dtype=np.int64).reshape(160, 64)[:148]
if k.info["plan"].get("cta_pair"):
    tr = tr[0::2]  # pair leaders carry the MMA marks
rel = tr - tr[:, :1]
rows = []
for c in range(len(tr)):
    r = rel[c]
    nt = sum(1 for i in range(6) if tr[c, 16 + i] != 0)
    rows.append((c, nt, r[1], r[2], [r[8 + i] for i in range(nt)], [r[16 + i] for i in range(nt)],
                 [r[24 + i] for i in range(nt)], [r[32 + i] for i in range(nt)], r[40]))
for row in rows[:6] + rows[-2:]:
    print(row)
end = np.array([r[-1] for r in rows])
print("end clk: median", np.median(end), "max", end.max(), "min", end.min())
first_mma = np.array([r[4][0] for r in rows])
fl = lib.gensor_dev_flat_filt
fl.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
fb = (ctypes.c_ulonglong * 5)()
fl(fb)
flush.zero_()
torch.cuda.synchronize()
torch.cuda._sleep(200_000)  # the host enqueues while the device is busy: device-side gaps only
a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a0.record()
k.execute(xs, out)
b0.record()
b0.synchronize()
fl(fb)
assert fn(buf, 160 * 64) == 0
tg = np.array(buf, dtype=np.int64).reshape(160, 64)[:148]
print("globaltimer (ns): filters start..end", int(fb[1] - fb[0]), "| conv CTAs first start - filters start", int(tg[:, 50].min() - fb[0]),
      "| conv CTA start spread", int(tg[:, 50].max() - tg[:, 50].min()), "| conv span (first start .. last end)", int(tg[:, 51].max() - tg[:, 50].min()),
      "| filters start .. conv end", int(tg[:, 51].max() - fb[0]), "| events", a0.elapsed_time(b0) * 1e3)
print("filters start -> last counter increment", int(fb[3] - fb[0]) if fb[3] else None, "| -> first conv observation", int(fb[4] - fb[0]) if fb[4] < 2**63 else None)
if fb[2]:
    print("marker -> filters start", int(fb[0] - fb[2]), "| marker -> conv first CTA", int(tg[:, 50].min() - fb[2]), "| marker -> conv end", int(tg[:, 51].max() - fb[2]))
print("pair start marks (alloc, prezero(w2), cluster sync, griddep):", np.median(rel[:, 2]), np.median(tr[:, 5] - tr[:, 0]), np.median(rel[:, 3]), np.median(rel[:, 4]))
print("first MMA start: median", np.median(first_mma), "griddep wait", np.median([r[2] for r in rows]),
      "filters ready", np.median([r[3] for r in rows]))
mma = [r[5][i] - r[4][i] for r in rows for i in range(r[1])]
epi = [r[7][i] - r[6][i] for r in rows for i in range(r[1])]
if fam == "conv_flat":
    e = rel[:, 24 + 1]
    print("epilogue tile 1 (cycles from acc_full): blocks read", np.median(rel[:, 44] - e), "published", np.median(rel[:, 46] - e), "barrier", np.median(rel[:, 47] - e), "exchanged",
          np.median(rel[:, 45] - e), "done", np.median(rel[:, 33] - e))
print("MMA issue->commit per tile: median", np.median(mma), " epilogue per tile: median", np.median(epi))
if fam == "conv_flat" and hasattr(lib, "gensor_dev_flat_warp"):
    fw = lib.gensor_dev_flat_warp
    fw.argtypes = [ctypes.POINTER(ctypes.c_longlong), ctypes.c_int]
    wb = (ctypes.c_longlong * (160 * 16 * 5))()
    assert fw(wb, 160 * 16 * 5) == 0
    w = np.array(wb, dtype=np.int64).reshape(160, 16, 5)[:148]
    print("per epilogue warp, tile 1 (cycles from CTA start; median over CTAs): got, TMEM read, at barrier, past barrier, done")
    for i in range(16):
        wi = i + 2
        print(f"  warp {wi:2d} (q={wi & 3}, h={(wi - 2) >> 2}, SP{wi % 4}):", [int(np.median(w[:, i, k])) for k in range(5)])
if fam == "conv_flat":
    print("pair start (cycles from CTA start, median): barriers initialised", np.median(rel[:, 5]), "| cluster barrier passed",
          np.median(rel[:, 6]), "| TMEM allocated (warp 1)", np.median(rel[:, 7]), "| block barrier passed", np.median(rel[:, 2]))

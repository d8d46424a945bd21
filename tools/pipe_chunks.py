"""Developer probe: the execute_host copy/compute pipeline of the headline conv emulated with
torch streams at different chunk counts (H2D chunk c || kernels of chunk c-1 || D2H chunk c-2),
using the real conv_flat kernels for the chunk shapes — to choose the pipeline's chunk size."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2502_11407_b200 as g
hw = g.HardwareSpec.b200(0)
N, C, H, W, F = 16, 64, 58, 58, 64
OH, OW = H - 2, W - 2
xin = torch.rand(N * C * H * W).pin_memory()
kin = torch.rand(F * C * 9).pin_memory()
hout = torch.empty(N * F * OH * OW).pin_memory()
din = torch.empty_like(xin, device="cuda"); dk = torch.empty_like(kin, device="cuda")
dout = torch.empty(N * F * OH * OW, device="cuda")
s_in, s_out, s_k = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.current_stream()
ui, uo = C * H * W, F * OH * OW
for chunks in (1, 2, 4, 8, 16):
    q = N // chunks
    op = g.TensorOpSpec.parse_text(json.dumps({"kind": "conv2d", "I": [q, C, H, W], "K": [F, C, 3, 3], "S": 1}))
    k = g.Kernel(op, g.optimize(op, hw, g.EngineConfig(mode="b200", top_k=1)), 0, "auto")
    def step():
        ev0 = torch.cuda.Event(); ev0.record(s_k)
        s_in.wait_event(ev0); s_out.wait_event(ev0)
        with torch.cuda.stream(s_in):
            dk.copy_(kin, non_blocking=True)
        for c in range(chunks):
            with torch.cuda.stream(s_in):
                din[c * q * ui:(c + 1) * q * ui].copy_(xin[c * q * ui:(c + 1) * q * ui], non_blocking=True)
                e_in = torch.cuda.Event(); e_in.record(s_in)
            s_k.wait_event(e_in)
            k.execute([din[c * q * ui:(c + 1) * q * ui], dk], dout[c * q * uo:(c + 1) * q * uo], s_k)
            e_k = torch.cuda.Event(); e_k.record(s_k)
            s_out.wait_event(e_k)
            with torch.cuda.stream(s_out):
                hout[c * q * uo:(c + 1) * q * uo].copy_(dout[c * q * uo:(c + 1) * q * uo], non_blocking=True)
        s_k.wait_stream(s_out)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(15):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s_k); step(); e1.record(s_k); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    print(json.dumps({"chunks": chunks, "images_per_chunk": q, "ms": round(statistics.median(ts), 4)}), flush=True)

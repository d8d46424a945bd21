"""Developer tool: cuDNN / cuBLAS times of the BASELINE shapes (library context for the roofline
fractions; never on the product path). Same timing discipline as bench.py: L2 flushed between
steps, CUDA events, median."""
import json, statistics, torch
torch.backends.cuda.matmul.allow_tf32 = True
torch.backends.cudnn.allow_tf32 = True
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn, n=20):
    for _ in range(3): fn()
    ts = []
    for _ in range(n):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
    return statistics.median(ts)
res = {}
x = torch.rand(16, 64, 58, 58, device="cuda"); w = torch.rand(64, 64, 3, 3, device="cuda")
us = t(lambda: torch.nn.functional.conv2d(x, w)); res["conv2d_C_tf32_cudnn"] = {"us": us, "tflops": 3.699376128e9 / us / 1e6}
xb, wb = x.bfloat16(), w.bfloat16()
us = t(lambda: torch.nn.functional.conv2d(xb, wb)); res["conv2d_C_bf16_cudnn"] = {"us": us, "tflops": 3.699376128e9 / us / 1e6}
a = torch.rand(1024, 1024, device="cuda"); b = torch.rand(1024, 1024, device="cuda")
us = t(lambda: a @ b); res["gemm_G_tf32_cublas"] = {"us": us, "tflops": 2 * 1024**3 / us / 1e6}
q = torch.rand(192, 512, 64, device="cuda").bfloat16(); k = torch.rand(192, 64, 512, device="cuda").bfloat16()
us = t(lambda: torch.bmm(q, k)); res["bgemm_B_bf16_cublas"] = {"us": us, "tflops": 6.442450944e9 / us / 1e6, "gbs": 125829120 / us / 1e3}
A = torch.rand(32768, 4096, device="cuda"); one = torch.ones(4096, device="cuda")
us = t(lambda: A @ one); res["rowsum_V_cublas_gemv"] = {"us": us, "gbs": 537018368 / us / 1e3}
us = t(lambda: torch.softmax(A, 1)); res["softmax_torch"] = {"us": us, "gbs": 1073741824 / us / 1e3}
print(json.dumps(res, indent=1))

"""Roofline denominators measured on this B200: FP32 FFMA (own probe kernel)
and dense TF32 tensor throughput (cuBLAS TF32 GEMM via torch, 8192^3)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_17001_b200 as P

out = {"gpu": torch.cuda.get_device_name(0)}
out["ffma_tflops"] = max(P.probe_ffma_tflops(0) for _ in range(5))
torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
a = torch.randn(n, n, device="cuda", dtype=torch.float32)
b = torch.randn(n, n, device="cuda", dtype=torch.float32)
for _ in range(3):
    a @ b
torch.cuda.synchronize()
best = 0.0
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); a @ b; e.record(); e.synchronize()
    best = max(best, 2 * n ** 3 / (s.elapsed_time(e) * 1e-3) / 1e12)
out["tf32_tflops_burst"] = best
t0 = time.time(); k = 0
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
while time.time() - t0 < 4.0:
    for _ in range(10):
        a @ b
    k += 10
    torch.cuda.synchronize()
e.record(); e.synchronize()
out["tf32_tflops_sustained"] = 2 * n ** 3 * k / (s.elapsed_time(e) * 1e-3) / 1e12
torch.backends.cuda.matmul.allow_tf32 = False
x = torch.empty(1 << 30, dtype=torch.uint8, device="cuda"); y = torch.empty_like(x)
bw = 0
for _ in range(10):
    s.record(); y.copy_(x); e.record(); e.synchronize()
    bw = max(bw, 2 * x.numel() / (s.elapsed_time(e) * 1e-3) / 1e9)
out["copy_gbs"] = bw
print(json.dumps(out))

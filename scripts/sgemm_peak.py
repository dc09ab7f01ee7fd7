"""cuBLAS FP32 SGEMM throughput (TF32 off) on this GPU: a library reference point for the FP32 path."""
import json, sys, torch
torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False
res = {}
for n in (4096, 8192):
    a = torch.randn(n, n, device="cuda"); b = torch.randn(n, n, device="cuda")
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0.record(); a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[n] = 2 * n ** 3 / best / 1e9
    print(f"sgemm {n}^3 fp32 (tf32 off): {res[n]:.1f} TFLOP/s (best of 10, {best:.2f} ms)")
# a 4 s back-to-back run (sustained)
n = 8192; a = torch.randn(n, n, device="cuda"); b = torch.randn(n, n, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); k = 0
import time; t = time.time()
while time.time() - t < 4: a @ b; k += 1
e1.record(); torch.cuda.synchronize()
print(f"sgemm 8192^3 sustained: {2 * n ** 3 * k / e0.elapsed_time(e1) / 1e9:.1f} TFLOP/s over {k} GEMMs")

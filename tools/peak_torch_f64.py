"""cuBLAS DGEMM yardstick: torch.matmul float64 8192^3, best of 10 and ~4 s sustained."""
import json, time, torch
n = 8192
a = torch.rand(n, n, dtype=torch.float64, device="cuda")
b = torch.rand(n, n, dtype=torch.float64, device="cuda")
c = a @ b
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(10):
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
reps = int(4000 / best) + 1
e0.record()
for _ in range(reps):
    c = a @ b
e1.record(); torch.cuda.synchronize()
tot = e0.elapsed_time(e1)
fl = 2.0 * n ** 3
print(json.dumps({"cublas_dgemm_8192_burst_tflops": fl / best / 1e9, "cublas_dgemm_8192_sustained_tflops": fl * reps / tot / 1e9}))

"""cuBLAS TF32 GEMM throughput on this GPU (library reference for the
tcgen05 tf32 kernel): torch.matmul on fp32 with TF32 allowed, CUDA events,
best of N after warm-up, 4096^3 (the tuned problem) and 8192^3."""
import json
import torch

torch.backends.cuda.matmul.allow_tf32 = True
torch.backends.cudnn.allow_tf32 = True
res = {}
for n in (4096, 8192):
    a = torch.rand(n, n, device="cuda")
    b = torch.rand(n, n, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    res[n] = {"ms": round(best, 4), "tflops": round(2 * n ** 3 / best / 1e9, 1)}
print(json.dumps({"cublas_tf32": res}))

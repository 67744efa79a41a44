"""cuBLAS DGEMM yardstick on the box (fp64 tensor pipe), for the batched path's roofline."""
import json, torch
torch.backends.cuda.matmul.allow_tf32 = False
def t(m, n, k, reps=20):
    a = torch.randn(m, k, dtype=torch.float64, device="cuda"); b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return dict(m=m, n=n, k=k, ms=ms, tflops=2 * m * n * k / ms / 1e9)
out = [t(8192, 8192, 8192, 5), t(16384, 16384, 16384, 2), t(840, 8192, 120), t(120, 8192, 720), t(8192, 840, 120)]
print(json.dumps(out))

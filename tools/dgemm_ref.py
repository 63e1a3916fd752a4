"""Measure cuBLAS DGEMM (library context only, never on the hot path) and clocks."""
import subprocess, time, torch
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active", "--format=csv,noheader", "-lms", "200"], stdout=open("gpurun_out/dgemm_clocks.csv", "w"))
for n in (4096, 8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10 if n < 16384 else 4
    e0.record()
    for _ in range(reps): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cuBLAS DGEMM n={n}: {2*n**3/ms/1e9:.1f} GF/s ({ms:.2f} ms)")
a = torch.randn(32768, 32768, dtype=torch.float64, device="cuda"); a = a @ a.T + 32768 * torch.eye(32768, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t = time.time()
    L = torch.linalg.cholesky(a)
    torch.cuda.synchronize(); dt = time.time() - t
    print(f"cuSOLVER potrf n=32768 (context only): {dt*1e3:.1f} ms = {32768**3/3/dt/1e9:.1f} GF/s")
smi.terminate()

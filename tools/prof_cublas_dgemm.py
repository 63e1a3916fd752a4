"""cuBLAS DGEMM (context only, never on the product path): C = A B^T with the
trailing-SYRK shape (m = n = 16384, K = 2048), device ms and TF/s."""
import sys

import torch

m = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
a = torch.rand(m, k, dtype=torch.float64, device="cuda")
c = torch.empty(m, m, dtype=torch.float64, device="cuda")
torch.matmul(a, a.T, out=c)
ms = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, a.T, out=c)
    e1.record()
    e1.synchronize()
    ms.append(e0.elapsed_time(e1))
print(f"cublas dgemm m=n={m} k={k}: ms {[round(x, 3) for x in ms]}, {2 * m * m * k / min(ms) / 1e9:.1f} TF/s")

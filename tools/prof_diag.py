"""One diagonal-block step of the mixed factorization (FP64 tree driver on a
bs x bs block, then the explicit inverse), for an ncu launch list."""
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_07311_b200.mixed as M  # noqa: E402
from paper_2604_07311_b200.control import flatten_cholesky, parse_tree, resolve_config  # noqa: E402
from paper_2604_07311_b200.engine import _lib  # noqa: E402
from paper_2604_07311_b200.views import DType, from_torch  # noqa: E402

bs = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
lib = _lib.lib()
tree = parse_tree(json.dumps(M.DIAG_TREE))
levels = flatten_cholesky(tree, resolve_config(tree, DType.F64))
arr = (_lib.BfCholLevel * len(levels))(*[_lib.BfCholLevel(v, 0, b, kc) for v, b, kc in levels])
g = torch.Generator(device="cuda")
g.manual_seed(1)
m = torch.rand(bs, bs, device="cuda", generator=g, dtype=torch.float64)
a0 = m @ m.T + bs * torch.eye(bs, device="cuda", dtype=torch.float64)
s = torch.cuda.current_stream().cuda_stream
info = torch.full((1,), -1, dtype=torch.int32, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for r in range(reps):
    a = a0.clone()
    x = torch.eye(bs, device="cuda", dtype=torch.float64)
    torch.cuda.synchronize()
    ev[0].record()
    assert lib.bf_cholesky_d(ctypes.byref(_lib.as_bfview(from_torch(a))), arr, len(levels), info.data_ptr(), s) == 0
    ev[1].record()
    assert lib.bf_trsm_rltn_d(1.0, ctypes.byref(_lib.as_bfview(from_torch(a))), ctypes.byref(_lib.as_bfview(from_torch(x))),
                              512, None, s) == 0
    ev[2].record()
    ev[2].synchronize()
    print(json.dumps({"bs": bs, "diag_ms": round(ev[0].elapsed_time(ev[1]), 3),
                      "inverse_ms": round(ev[1].elapsed_time(ev[2]), 3)}), flush=True)

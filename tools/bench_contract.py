"""Tensor-contraction benchmark (BASELINE configs[4]): abij,cdij->abcd with
dims d (C5: d=128, FP64), plus the non-foldable permuted layout
aibj,cjdi->abcd that exercises the gathered (block-scatter) operand path.

    python tools/bench_contract.py [d ...]

Prints one JSON line per (spec, d): GFLOP/s (2*M*N*K per contraction, device
time, inputs resident), and whether fold on/off give identical bits (the
folded run uses the strided TMA GEMM, the unfolded one the gather kernel, and
both must sum k in the reference's order).
"""
import hashlib
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.tensor import ContractionSpec, make_tensor  # noqa: E402


def run(spec_text: str, d: int, reps: int = 3):
    spec = ContractionSpec.parse(spec_text)
    g = torch.Generator(device="cuda")
    g.manual_seed(42)

    def rand(labels):
        t = make_tensor([d] * len(labels))
        t.storage.copy_(torch.rand(t.storage.numel(), dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
        return t

    a, b = rand(spec.labels_a), rand(spec.labels_b)
    c = make_tensor([d] * len(spec.labels_c))
    flops = 2.0 * d ** (len(set(spec.labels_a + spec.labels_b)))
    out = {}
    for fold in (True, False):
        bf.contract(1.0, a, b, 0.0, c, spec, fold=fold)  # warm
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            bf.contract(1.0, a, b, 0.0, c, spec, fold=fold)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out[fold] = (flops / (ms / 1e3) / 1e9, ms, hashlib.sha256(c.storage.cpu().numpy().tobytes()).hexdigest())
    print(json.dumps({"spec": spec_text, "d": d, "flops": flops,
                      "gflops_fold": round(out[True][0], 1), "ms_fold": round(out[True][1], 3),
                      "gflops_nofold": round(out[False][0], 1), "ms_nofold": round(out[False][1], 3),
                      "fold_bitwise_equal": out[True][2] == out[False][2]}), flush=True)


if __name__ == "__main__":
    dims = [int(x) for x in sys.argv[1:]] or [64, 128]
    for d in dims:
        for spec in ("abij,cdij->abcd", "aibj,cjdi->abcd"):
            run(spec, d, reps=3 if d <= 64 else 1)

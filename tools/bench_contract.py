"""Tensor-contraction benchmark (BASELINE configs[4]): abij,cdij->abcd with
dims d (C5: d=128, FP64), plus the non-foldable permuted layout
aibj,cjdi->abcd that exercises the gathered (block-scatter) operand path.

    python tools/bench_contract.py [d ...]

Prints one JSON line per (spec, d): GFLOP/s (2*M*N*K per contraction, device
time, inputs resident) for fold on/off x stage auto/never (auto: permuted
operands staged k-contiguous for the TMA GEMM when large; never: the
element-gathering GEMM), and whether every path gave identical bits (all must
sum k in the reference's order).
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
        for stage in ("auto", "never"):
            bf.contract(1.0, a, b, 0.0, c, spec, fold=fold, stage=stage)  # warm
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                bf.contract(1.0, a, b, 0.0, c, spec, fold=fold, stage=stage)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1) / reps
            key = ("fold" if fold else "nofold") + "_" + stage
            out[key] = (flops / (ms / 1e3) / 1e9, ms, hashlib.sha256(c.storage.cpu().numpy().tobytes()).hexdigest())
    line = {"spec": spec_text, "d": d, "flops": flops}
    for key, (gf, ms, _) in out.items():
        line["gflops_" + key] = round(gf, 1)
        line["ms_" + key] = round(ms, 3)
    line["all_paths_bitwise_equal"] = len({h for _, _, h in out.values()}) == 1
    print(json.dumps(line), flush=True)

if __name__ == "__main__":
    dims = [int(x) for x in sys.argv[1:]] or [64, 128]
    for d in dims:
        for spec in ("abij,cdij->abcd", "aibj,cjdi->abcd"):
            run(spec, d, reps=3 if d <= 64 else 1)

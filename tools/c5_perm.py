"""Permuted 4-index contractions at d=128 (FP64, C5 size): device ms and
TFLOP/s of the mode-group TMA path.  aibj,cidj->abcd: both operands through
4-D tensor maps (no copy); aibj,cjdi->abcd: A through 4-D maps, B (its k
order transposed w.r.t. the reference's) staged k-contiguous once."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.tensor import ContractionSpec, make_tensor  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 128
import os  # noqa: E402
from paper_2604_07311_b200.engine import _lib  # noqa: E402
for _kv in filter(None, os.environ.get("BF_OPTS", "").split(",")):  # library options for sweeps
    _k, _v = _kv.split("=")
    assert _lib.lib().bf_set_option(_k.encode(), int(_v)) == 0, _kv
g = torch.Generator(device="cuda")
g.manual_seed(42)
for text in ("abij,cdij->abcd", "aibj,cidj->abcd", "aibj,cjdi->abcd", "abij,cdij->acbd"):
    spec = ContractionSpec.parse(text)

    def rand(n):
        t = make_tensor([d] * n)
        t.storage.copy_(torch.rand(t.storage.numel(), dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
        return t

    a, b, c = rand(4), rand(4), make_tensor([d] * 4)
    bf.contract(1.0, a, b, 0.0, c, spec)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    ms = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        bf.contract(1.0, a, b, 0.0, c, spec)
        e1.record()
        e1.synchronize()
        ms.append(round(e0.elapsed_time(e1), 2))
    print(json.dumps({"spec": text, "d": d, "ms": ms, "tflops": round(2 * d ** 6 / (min(ms) / 1e3) / 1e12, 2),
                      "peak_alloc_gb": round(torch.cuda.max_memory_allocated() / 1e9, 2)}), flush=True)
    del a, b, c
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()

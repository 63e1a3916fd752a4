"""One folded contraction abij,cdij->abcd at d (for an ncu launch list)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.tensor import ContractionSpec, make_tensor  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 128
spec = ContractionSpec.parse("abij,cdij->abcd")
g = torch.Generator(device="cuda")
g.manual_seed(1)
ts = []
for labels in (spec.labels_a, spec.labels_b):
    t = make_tensor([d] * len(labels))
    t.storage.copy_(torch.rand(t.storage.numel(), dtype=torch.float64, device="cuda", generator=g))
    ts.append(t)
c = make_tensor([d] * 4)
bf.contract(1.0, ts[0], ts[1], 0.0, c, spec)
torch.cuda.synchronize()
print("ok")

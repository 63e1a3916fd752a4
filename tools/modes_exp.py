import ctypes, json, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2604_07311_b200 as bf
from paper_2604_07311_b200.engine import _lib
from paper_2604_07311_b200.tensor import ContractionSpec, make_tensor
d = 128
g = torch.Generator(device="cuda"); g.manual_seed(1)
def rand():
    t = make_tensor([d] * 4)
    t.storage.copy_(torch.rand(t.storage.numel(), dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
    return t
a, b, c = rand(), rand(), make_tensor([d] * 4)
N = d * d
def mv(t, rd, rs, cd, cs):
    v = _lib.BfModesView(); v.base = t.storage.data_ptr(); v.off = 0
    v.nr, v.nc = len(rd), len(cd)
    for i, (x, y) in enumerate(zip(rd, rs)): v.rdim[i], v.rstr[i] = x, y
    for i, (x, y) in enumerate(zip(cd, cs)): v.cdim[i], v.cstr[i] = x, y
    return v
lib = _lib.lib()
s = torch.cuda.current_stream().cuda_stream
variants = {
  "plain_kernel": None,
  "modes_all_single": (mv(a, [N], [N], [N], [1]), mv(b, [N], [1], [N], [N]), mv(c, [N], [N], [N], [1])),
  "modes_c_2groups": (mv(a, [N], [N], [N], [1]), mv(b, [N], [1], [N], [N]), mv(c, [d, d], [d**3, d**2], [d, d], [d, 1])),
  "modes_a_4d": (mv(a, [d, d], [d**3, d**2], [d, d], [d, 1]), mv(b, [N], [1], [N], [N]), mv(c, [N], [N], [N], [1])),
}
spec = ContractionSpec.parse("abij,cdij->abcd")
for name, v in variants.items():
    def run():
        if v is None:
            bf.contract(1.0, a, b, 0.0, c, spec)
        else:
            rc = lib.bf_contract_modes_d(1.0, ctypes.byref(v[0]), ctypes.byref(v[1]), 0.0, ctypes.byref(v[2]), 256, s)
            assert rc == 0, lib.bf_last_error()
    run(); torch.cuda.synchronize()
    ms = []
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); e1.synchronize(); ms.append(round(e0.elapsed_time(e1), 2))
    print(name, ms, flush=True)

"""Per-step timeline of the host-memory entry point (bf_cholesky_host_d:
lower triangle in by block columns, step 0 consuming each as it lands,
finished block columns streamed back) at the bench size."""
import ctypes, json, os, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
import paper_2604_07311_b200 as bf
from paper_2604_07311_b200.control import parse_tree
from paper_2604_07311_b200.engine import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
tree = parse_tree(json.dumps(bench.GPU_TREE))
lib = _lib.lib()
for kv in filter(None, os.environ.get("BF_OPTS", "").split(",")):
    k, v = kv.split("=")
    assert lib.bf_set_option(k.encode(), int(v)) == 0, kv
a0 = bench.make_spd(bf, torch, n, torch.device("cuda"))
pristine = a0.cpu()
host = torch.empty(n, n, dtype=torch.float64, pin_memory=True)
work = torch.empty_like(a0)
ms = []
for i in range(3):
    host.copy_(pristine)
    torch.cuda.synchronize()
    lib.bf_set_option(b"timeline", 1 if i == 2 else 0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bf.cholesky_host(host, "lower", tree, work=work)
    e1.record()
    e1.synchronize()
    ms.append(round(e0.elapsed_time(e1), 2))
print("opts", os.environ.get("BF_OPTS", ""), "e2e ms", ms)
steps = lib.bf_timeline(None, 0)
buf = (ctypes.c_float * (5 * steps))()
lib.bf_timeline(buf, steps)
print("step col_done rest_done panel_beg panel_end")
for i in range(steps):
    c, r, pb, pe, pd = buf[5 * i: 5 * i + 5]
    print(f"{i:4d} {c:9.2f} {r:10.2f} {pb:10.2f} {pe:10.2f}")

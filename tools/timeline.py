"""Per-step timeline of the lookahead schedule at the bench size."""
import ctypes, json, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
import paper_2604_07311_b200 as bf
from paper_2604_07311_b200.control import parse_tree
from paper_2604_07311_b200.engine import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
tree = parse_tree(sys.argv[2]) if len(sys.argv) > 2 else parse_tree(json.dumps(bench.GPU_TREE))
lib = _lib.lib()
import os
for kv in filter(None, os.environ.get("BF_OPTS", "").split(",")):  # e.g. BF_OPTS=tail_reserve=32,tail_rows=20480
    k, v = kv.split("=")
    assert lib.bf_set_option(k.encode(), int(v)) == 0, kv
a0 = bench.make_spd(bf, torch, n, torch.device("cuda"))
work = a0.clone()
bf.cholesky(bf.from_torch(work), "lower", tree)  # warm
plain = []
for _ in range(3):  # plain timings (no timeline events)
    work.copy_(a0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bf.cholesky(bf.from_torch(work), "lower", tree)
    e1.record()
    e1.synchronize()
    plain.append(round(e0.elapsed_time(e1), 2))
print("opts", os.environ.get("BF_OPTS", ""), "plain ms", plain)
work.copy_(a0)
lib.bf_set_option(b"timeline", 1)
torch.cuda.synchronize()
bf.cholesky(bf.from_torch(work), "lower", tree)
torch.cuda.synchronize()
steps = lib.bf_timeline(None, 0)
buf = (ctypes.c_float * (5 * steps))()
lib.bf_timeline(buf, steps)
prev_rest = 0.0
print("step  n_k   col_done  rest_done  panel_beg  panel_end  panel_ms  diag_ms  syrk_ms  exposed_ms")
tot_exp = 0.0
for i in range(steps):
    c, r, pb, pe, pd = buf[5 * i: 5 * i + 5]
    nk = n - (i + 1) * (tree.bs)
    exposed = max(0.0, pe - r)
    tot_exp += exposed
    print(f"{i:4d} {nk:6d} {c:9.2f} {r:10.2f} {pb:10.2f} {pe:10.2f} {pe - pb:9.2f} {pd - pb:8.2f} {r - c:8.2f} {exposed:10.2f}")
print(f"total {buf[5 * (steps - 1) + 3]:.2f} ms, panel exposed {tot_exp:.2f} ms")

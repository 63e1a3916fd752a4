import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import paper_2604_07311_b200 as bf
from paper_2604_07311_b200.control import parse_tree
from paper_2604_07311_b200.engine import _lib
from golden_inputs import digest, spd_int
TREE = ('{"op":"cholesky","variant":3,"bs":512,"kernel":{"kc":512},"child":{"op":"cholesky","variant":3,"bs":64,'
        '"child":{"op":"cholesky","variant":"unblocked3"}}}')
import oracle as O
for bn in (int(x) for x in sys.argv[1:]):
    _lib.lib().bf_set_option(b"tma_bn", bn)
    for n, uplo in [(3000, "lower"), (1700, "upper"), (1700, "lower")]:
        a0 = spd_int(41, n)
        tree = parse_tree(TREE)
        ds = []
        for rep in range(3):
            ref = bf.make_view(n, n, fill=a0)
            bf.cholesky(ref, uplo, tree)
            ds.append(digest(ref.to_numpy()))
        v = bf.make_view(n, n, fill=a0)
        try:
            g = bf.CholeskyGraph(v, uplo, tree)
        except Exception as e:
            print(bn, n, uplo, "capture failed:", str(e)[:200], flush=True)
            import torch; torch.cuda.synchronize()
            continue
        gs = []
        for _ in range(3):
            v.copy_from(a0)
            g()
            gs.append(digest(v.to_numpy()))
        print(bn, n, uplo, "direct", ds, "graph", gs, flush=True)

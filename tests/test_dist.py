"""Multi-rank 2D block-cyclic Cholesky.

CPU: world_size 2, 4 and 8 (grids 2x1, 2x2, 4x2) under gloo, the distribution/communication logic
driven with the oracle as the per-tile compute (test-side stand-in), checked
bit for bit against the single-process oracle factorization.
GPU: the 1x1 grid against bf.cholesky, and 2 ranks sharing one GPU with a
host-staged gloo transport (their kernels never wait on each other), both
bit for bit.
"""
from __future__ import annotations

import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from golden_inputs import digest, spd_int
from paper_2604_07311_b200.control import parse_tree
from paper_2604_07311_b200.dist import BlockCyclic2D, TorchComm, cholesky_distributed, grid_for

TREE = ('{"op":"cholesky","variant":3,"bs":48,"kernel":{"kc":32},"child":{"op":"cholesky","variant":3,"bs":16,'
        '"child":{"op":"cholesky","variant":"unblocked3"}}}')


def _meta(t: torch.Tensor) -> tuple[np.ndarray, dict]:
    base = t
    while base._base is not None:
        base = base._base
    flat = base.reshape(-1).numpy()
    return flat, {"off": t.storage_offset(), "m": t.shape[0], "n": t.shape[1], "rs": t.stride(0), "cs": t.stride(1)}


class OracleOps:
    """Test-side CPU compute for the distributed driver: the golden-pinned
    oracle applied to the same tiles the B200 kernels would receive."""

    def potrf(self, tile, levels, base, info):
        if int(info[0]) >= 0:
            return
        st, m = _meta(tile)
        bad = O.cholesky(st, m, levels)
        if bad >= 0:
            info[0] = base + bad

    def trsm(self, tri, b, kc, info):
        if int(info[0]) >= 0:
            return
        tri = tri.contiguous()
        O.trsm_rltn(1.0, _meta(tri), _meta(b), kc=kc)

    def gemm(self, a, bt, c, lower, kc, info):
        if int(info[0]) >= 0:
            return
        a, bt = a.contiguous(), bt.contiguous()
        sa, ma = _meta(a)
        sb, mb = _meta(bt)
        O.gemm(-1.0, (sa, ma), (sb, O.transposed(mb)), 1.0, _meta(c), kc=kc, lower_only=lower)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, nb, tree_doc, out_dir, use_gpu, npd_at):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pr, pc = grid_for(world)
    layout = BlockCyclic2D(n, nb, pr, pc)
    a0 = spd_int(321, n)
    if npd_at is not None:
        a0[npd_at, npd_at] = -1e9
    local = torch.from_numpy(layout.scatter(a0, rank).copy())
    tree = parse_tree(tree_doc)
    if use_gpu:
        from paper_2604_07311_b200.dist import B200Ops

        dev_local = local.cuda()

        class HostStagedComm(TorchComm):  # gloo carries CUDA data through host copies
            def bcast(self, t, root):
                host = t.cpu()
                dist.broadcast(host, src=root)
                t.copy_(host)

        bad = cholesky_distributed(dev_local, layout, tree, HostStagedComm(), B200Ops(), raise_on_failure=False)
        local = dev_local.cpu()
    else:
        bad = cholesky_distributed(local, layout, tree, TorchComm(), OracleOps(), raise_on_failure=False)
    np.save(os.path.join(out_dir, f"local{rank}.npy"), local.numpy())
    with open(os.path.join(out_dir, f"bad{rank}.json"), "w") as f:
        json.dump(bad, f)
    dist.barrier()
    dist.destroy_process_group()


def _run(world, n, nb, tmp_path, use_gpu=False, npd_at=None):
    mp.spawn(_worker, args=(world, _free_port(), n, nb, TREE, str(tmp_path), use_gpu, npd_at), nprocs=world, join=True)
    pr, pc = grid_for(world)
    layout = BlockCyclic2D(n, nb, pr, pc)
    locals_ = [np.load(tmp_path / f"local{r}.npy") for r in range(world)]
    bads = [json.load(open(tmp_path / f"bad{r}.json")) for r in range(world)]
    return layout.gather(locals_), bads


def _oracle_full(n, npd_at=None):
    a0 = spd_int(321, n)
    if npd_at is not None:
        a0[npd_at, npd_at] = -1e9
    st = a0.reshape(-1).copy()
    bad = O.cholesky(st, {"off": 0, "m": n, "n": n, "rs": n, "cs": 1}, O.levels_from_tree(json.loads(TREE), n, "f64"))
    return st.reshape(n, n), bad


def test_layout_roundtrip_and_ownership():
    lay = BlockCyclic2D(250, 48, 2, 3)
    full = np.random.default_rng(0).uniform(size=(250, 250))
    locs = [lay.scatter(full, r) for r in range(6)]
    back = lay.gather(locs, fill=np.zeros_like(full))
    for i in range(lay.tiles):
        for j in range(i + 1):
            sl = np.s_[i * 48:i * 48 + lay.tile_len(i), j * 48:j * 48 + lay.tile_len(j)]
            np.testing.assert_array_equal(back[sl], full[sl])
    assert sum(lay.local_shape(r)[0] * lay.local_shape(r)[1] for r in range(6)) >= 250 * 250
    assert [grid_for(p) for p in (1, 2, 4, 8)] == [(1, 1), (2, 1), (2, 2), (4, 2)]


@pytest.mark.parametrize("world,n", [(1, 150), (2, 200), (4, 250), (8, 400)])
def test_distributed_bitwise_equals_single_process_cpu(tmp_path, world, n):
    full, bads = _run(world, n, 48, tmp_path)
    ref, bad = _oracle_full(n)
    assert bad == -1 and bads == [-1] * world
    assert np.tril(full).tobytes() == np.tril(ref).tobytes()


def test_distributed_npd_index_all_ranks_cpu(tmp_path):
    full, bads = _run(4, 250, 48, tmp_path, npd_at=131)
    ref, bad = _oracle_full(250, npd_at=131)
    assert bad == 131 and bads == [131] * 4


@pytest.mark.gpu
def test_single_gpu_grid_matches_bf_cholesky(cuda):
    import paper_2604_07311_b200 as bf

    class Solo:
        rank, world = 0, 1

        def bcast(self, t, root):
            pass

    n = 1000
    tree_doc = ('{"op":"cholesky","variant":3,"bs":256,"kernel":{"kc":256},"child":{"op":"cholesky","variant":3,'
                '"bs":64,"child":{"op":"cholesky","variant":"unblocked3"}}}')
    a0 = spd_int(5, n)
    layout = BlockCyclic2D(n, 256, 1, 1)
    local = torch.from_numpy(layout.scatter(a0, 0).copy()).cuda()
    cholesky_distributed(local, layout, parse_tree(tree_doc), Solo())
    v = bf.make_view(n, n, fill=a0)
    bf.cholesky(v, "lower", parse_tree(tree_doc))
    got = layout.gather([local.cpu().numpy()])
    assert np.tril(got).tobytes() == np.tril(v.to_numpy()).tobytes()


@pytest.mark.gpu
def test_two_ranks_on_one_gpu_bitwise(cuda, tmp_path):
    full, bads = _run(2, 200, 48, tmp_path, use_gpu=True)
    ref, bad = _oracle_full(200)
    assert bads == [-1, -1]
    assert digest(np.tril(full)) == digest(np.tril(ref))


@pytest.mark.parametrize("world,n", [(1, 150), (2, 200)])
def test_lookahead_split_updates_bitwise_cpu(tmp_path, world, n, monkeypatch):
    """The lookahead schedule's split updates (block column k+1 first, then
    the rest) on CPU tensors, forced through the same code path as on the GPU
    by a stream-free stand-in: identical bits to the single-process oracle."""
    monkeypatch.setenv("BF_DIST_FORCE_SPLIT", "1")
    full, bads = _run(world, n, 48, tmp_path)
    ref, bad = _oracle_full(n)
    assert bads == [-1] * world
    assert np.tril(full).tobytes() == np.tril(ref).tobytes()

"""Benchmark: FP64 blocked Cholesky GFLOP/s at n=32768 on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[1]): FP64 Cholesky, n=32768, two-level
blocking.  One step = one in-place factorization of a fresh SPD matrix
A = M M^T + n I (M ~ U(-1,1), the reference generator cli.py:55-64, formed on
the device with this package's own SYRK).  Work per step is the reference's
flop count n^3/3 (cli.py:78-79).

* value      device time of K factorizations, inputs resident in HBM (8.6 GB,
             far larger than the 126 MB L2), CUDA events on the launch stream;
             the pristine input is restored between steps outside the events.
* e2e        the same metric through the public API from HOST memory:
             cholesky_host() on a pinned host matrix (its lower triangle goes
             to HBM by block columns on a copy stream while step 0 consumes
             each column as it lands, each finished block column of the
             factor comes back while later steps run), all inside the timed
             region.
* roofline   the dominant kernel (the DMMA GEMMT/SYRK of the trailing update),
             timed alone with CUDA events over every top-level trailing update
             of the factorization: algorithmic flops n_k(n_k+1)*bs per launch.
* cpu_baseline  the oracle port of the reference (oracle/, C++ restatement,
             bit-identical to the reference) on this host's cores on a bounded
             sample (a smaller n of the same algorithm).
--impl reference   times that CPU port alone (the reference's own code is
             Python + numba and is not installed on the GPU box).
N > 1 ranks factor ONE n=32768 matrix together (strong scaling): 2D
block-cyclic tiles over a grid_for(N) process grid, NCCL panel broadcasts,
bit-identical to the single-GPU factor (paper_2604_07311_b200/dist).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_DEFAULT = 32768
GPU_TREE = {
    "op": "cholesky", "variant": 3, "bs": 2048, "kernel": {"kc": 2048},
    "child": {"op": "cholesky", "variant": 3, "bs": 128, "kernel": {"kc": 128},
              "child": {"op": "cholesky", "variant": "unblocked3"}},
}
# FP64 roofline denominator.  MEASURED_PEAKS.json carries no FP64 entry and
# B200_PROFILING.md no FP64 fallback, so this is our own measurement on this
# pool (tools/fp64_peak.cu, profiles/r01_fp64_peak.txt): register-resident DMMA
# m8n8k4, 148 SMs, best and sustained 37.1 TFLOP/s at 1965 MHz.
FP64_PEAK_TFLOPS = 37.1
FP64_PEAK_SOURCE = "measured: tools/fp64_peak.cu DMMA register-resident, 37.1 TF/s (profiles/r01_fp64_peak.txt)"


def chol_flops(n: int) -> float:
    return n ** 3 / 3.0


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.samples: list[tuple] = []
        self._proc = None
        self._thread = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._thread = threading.Thread(target=self._read, daemon=True)
            self._thread.start()
        except OSError:
            self._proc = None
        return self

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._proc.kill()

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        smax = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[4 + i].lower() == "active"})
        power = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "power_w_max": max(power) if power else None, "samples": len(self.samples)}


# ------------------------------------------------------------- CPU oracle --
def cpu_baseline(n_target: int, budget_s: float = 15.0) -> dict:
    """The oracle port of the reference (bit-identical to it) on this host,
    all cores, on a bounded sample: the largest n (multiple of 1024) whose
    factorization fits the time budget, with the GPU arm's tree."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O

    O.build()
    threads = O.host_threads()
    # the GPU arm's own tree (BASELINE configs[1] two-level blocking), so the
    # sample differs from the GPU workload only in n
    levels = O.levels_from_tree(GPU_TREE, 0, "f64")

    def run(n):
        rng = np.random.default_rng(42)
        m = rng.integers(-4, 5, (n, n)).astype(np.float64)
        a = (m @ m.T + n * np.eye(n)).reshape(-1).copy()
        t0 = time.perf_counter()
        bad = O.cholesky(a, {"off": 0, "m": n, "n": n, "rs": n, "cs": 1}, levels, nthreads=threads)
        dt = time.perf_counter() - t0
        assert bad == -1
        return dt

    n = 2048
    dt = run(n)
    rate = chol_flops(n) / dt
    n_s = int((budget_s * rate * 3) ** (1 / 3) // 1024 * 1024)
    n_s = max(2048, min(n_s, n_target, 16384))
    if n_s != n:
        dt = run(n_s)
        n = n_s
    return {"value": chol_flops(n) / dt / 1e9, "unit": "GFLOP/s", "cores": threads, "kind": "port",
            "sample": f"oracle C++ port of the reference (bit-identical to it), n={n}, the bench tree "
                      f"(v3 bs2048 kc2048 -> v3 bs128 kc128 -> unblocked3), {threads} threads, one factorization "
                      f"({dt:.2f} s)"}


# ----------------------------------------------------------------- GPU arm --
def make_spd(bf, torch, n: int, device, seed: int = 42):
    """A = M M^T + n I (lower triangle) with this package's own SYRK."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    m = torch.rand(n, n, dtype=torch.float64, device=device, generator=g) * 2 - 1
    a = torch.zeros(n, n, dtype=torch.float64, device=device)
    va = bf.from_torch(a)
    vm = bf.from_torch(m)
    bf.syrk_lower(1.0, vm, 0.0, va, cfg=bf.KernelConfig(8, 6, 64, 4096, 2048, bf.DType.F64, bf.DType.F64))
    a.diagonal().add_(float(n))
    del m
    return a


def side_workloads(torch, a0, n: int, fp64_ms: float, l64=None) -> dict:
    """BASELINE configs[3] and [4], measured after the headline (not part of
    `value`): the mixed-precision solve of the same SPD matrix (bf16/fp32
    factor on tcgen05 + FP64 refinement to 10*n*eps), FP64-equivalent
    n^3/3 / time; the FP32 factorization of that matrix on the tensor cores
    (3xTF32); and the 4-index contraction abij,cdij->abcd at d=128."""
    from paper_2604_07311_b200.mixed import MixedWorkspace, posv_mixed
    from paper_2604_07311_b200.tensor import ContractionSpec, make_tensor
    import paper_2604_07311_b200 as bfp

    out = {}
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    b = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    bs = 2048  # 2048: 72.5 ms, 1024: 78.5 ms, same 5 iterations and 3e-15 forward error (tools/c4_bs_sweep.py)
    ws = MixedWorkspace(n, bs)
    a_full = a0 + a0.T  # a0 holds the lower triangle only; the solve needs the dense symmetric A
    a_full.diagonal().sub_(a0.diagonal())
    step_tol = 1e-11  # forward-error criterion: the error left after a step of 1e-11 is ~1e-13 << 1e-12
    posv_mixed(a_full, b, ws=ws, step_tol=step_tol)  # warm
    torch.cuda.synchronize()
    ms, fms = [], []
    from paper_2604_07311_b200.mixed import cholesky_mixed

    for _ in range(3):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        cholesky_mixed(a_full, bs, ws=ws)
        e1.record()
        res = posv_mixed(a_full, b, ws=ws, step_tol=step_tol)
        e2.record()
        e2.synchronize()
        fms.append(e0.elapsed_time(e1))
        ms.append(e1.elapsed_time(e2))
    t, tf = statistics.median(ms), statistics.median(fms)
    fwd = None
    if l64 is not None:  # the FP64 solution from the bench's own FP64 factor (outside every timed region)
        lo = torch.tril(l64)
        y = torch.linalg.solve_triangular(lo, b[:, None], upper=False)
        xref = torch.linalg.solve_triangular(lo.T, y, upper=True)[:, 0]
        fwd = float((res.x - xref).norm() / xref.norm())
        del lo, y, xref
    # roofline of the factorization: bf16 tensor flops (trailing GEMMTs + column and panel GEMMs,
    # ~n^3/3 + n^2 bs) against the sustained bf16 peak, and its fp32 trailing-matrix HBM traffic
    # (each step reads and writes the lower trailing triangle once: sum_k n_k^2 * 4 B)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    bf16_peak = peaks.get("bf16_tflops_sustained", 1391.6)
    hbm_peak = peaks.get("hbm_gbs", 6556.2)
    tc_flops = chol_flops(n) + float(n) * n * bs
    traffic = sum(float(n - k * bs) ** 2 * 4 for k in range(1, n // bs))
    out["c4_mixed_posv"] = {"n": n, "bs": bs, "ms": round(t, 3), "factor_ms": round(tf, 3),
                            "refine_ms": round(t - tf, 3),
                            "fp64_equiv_gflops": round(chol_flops(n) / (t / 1e3) / 1e9, 1),
                            "iterations": res.iterations, "backward_error": res.backward_error,
                            "fwd_err_vs_fp64_solution": fwd, "converged": bool(res.converged),
                            "tol": "backward <= 10*n*eps64 and ||dx||/||x|| <= 1e-11",
                            "roofline_factor": {"tensor_achieved_tflops": round(tc_flops / (tf / 1e3) / 1e12, 1),
                                                "tensor_peak_tflops": bf16_peak,
                                                "tensor_frac": round(tc_flops / (tf / 1e3) / 1e12 / bf16_peak, 4),
                                                "hbm_achieved_gbs": round(traffic / (tf / 1e3) / 1e9, 1),
                                                "hbm_peak_gbs": hbm_peak,
                                                "hbm_frac": round(traffic / (tf / 1e3) / 1e9 / hbm_peak, 4),
                                                "bound": "neither: the FP64 diagonal/inverse/panel chain "
                                                         "(~3.6 ms per 2048 block, 16 blocks) is the critical path"},
                            "time_ratio_vs_fp64_factor": round(fp64_ms / t, 2)}
    del ws, a_full
    # FP32 Cholesky of the same matrix on the tensor cores (3xTF32 tcgen05)
    from paper_2604_07311_b200.mixed import F32TcWorkspace, cholesky_f32_tc

    a32 = a0.float()
    w32 = torch.empty_like(a32)
    ws32 = F32TcWorkspace(n, 1024)
    ms = []
    for i in range(4):
        w32.copy_(a32)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cholesky_f32_tc(w32, bs=1024, ws=ws32)
        e1.record()
        e1.synchronize()
        if i:
            ms.append(e0.elapsed_time(e1))
    t = statistics.median(ms)
    xv = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    lf = torch.tril(w32).double()
    ax = a0 @ xv + a0.T @ xv - a0.diagonal() * xv  # a0 holds the lower triangle only
    rr = float(torch.linalg.vector_norm(ax - lf @ (lf.T @ xv)) / torch.linalg.vector_norm(ax))
    out["c2_f32_tensor_core"] = {"n": n, "ms": round(t, 3), "gflops": round(chol_flops(n) / (t / 1e3) / 1e9, 1),
                                 "method": "3xTF32 tcgen05 GEMMs, FP64 diagonal blocks (mixed.cholesky_f32_tc)",
                                 "rel_residual_Ax_vs_LLtx": rr}
    del a32, w32, ws32, lf, ax
    torch.cuda.empty_cache()
    d = 128
    spec = ContractionSpec.parse("abij,cdij->abcd")

    def rand(labels):
        tt = make_tensor([d] * len(labels))
        tt.storage.copy_(torch.rand(tt.storage.numel(), dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
        return tt

    ta, tb = rand(spec.labels_a), rand(spec.labels_b)
    tc = make_tensor([d] * 4)
    bfp.contract(1.0, ta, tb, 0.0, tc, spec)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bfp.contract(1.0, ta, tb, 0.0, tc, spec)
    e1.record()
    e1.synchronize()
    cms = e0.elapsed_time(e1)
    out["c5_contraction"] = {"spec": "abij,cdij->abcd", "d": d, "dtype": "f64", "ms": round(cms, 3),
                             "gflops": round(2.0 * d ** 6 / (cms / 1e3) / 1e9, 1),
                             "path": "folded facades: one TMA DMMA GEMM, C tile in TMEM across the 64 kc folds"}

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1)

    ms_bf16 = timed(lambda: bfp.contract(1.0, ta, tb, 0.0, tc, spec, precision="bf16"))
    out["c5_contraction_bf16"] = {"spec": "abij,cdij->abcd", "d": d, "ms": round(ms_bf16, 3),
                                  "gflops": round(2.0 * d ** 6 / (ms_bf16 / 1e3) / 1e9, 1),
                                  "path": "bf16 operands, fp32 TMEM accumulation on tcgen05, FP64 C (not bitwise)"}
    pspec = ContractionSpec.parse("aibj,cidj->abcd")
    ms_perm = timed(lambda: bfp.contract(1.0, ta, tb, 0.0, tc, pspec))
    out["c5_contraction_permuted"] = {"spec": "aibj,cidj->abcd", "d": d, "dtype": "f64", "ms": round(ms_perm, 3),
                                      "gflops": round(2.0 * d ** 6 / (ms_perm / 1e3) / 1e9, 1),
                                      "path": "permuted mode groups through 4-D TMA tensor maps, no copy"}
    del ta, tb, tc
    torch.cuda.empty_cache()
    return out


def roofline_syrk(bf, torch, a0, n: int, bs: int, kc: int) -> dict:
    """Time the dominant kernel alone: the trailing GEMMT of every top-level
    step (n_k = n - (k+1)*bs, K = bs), on the launch stream."""
    work = a0.clone()
    v = bf.from_torch(work)
    cfg = bf.KernelConfig(8, 6, 64, kc, 2048, bf.DType.F64, bf.DType.F64)
    stream = torch.cuda.current_stream()
    flops, ms = 0.0, 0.0
    launches = 0
    for k in range(n // bs - 1):
        r2 = (k + 1) * bs
        nk = n - r2
        a21 = v.subview(bf.Range(r2, nk), bf.Range(k * bs, bs))
        a22 = v.subview(bf.Range(r2, nk), bf.Range(r2, nk))
        bf.syrk_lower(-1.0, a21, 1.0, a22, cfg=cfg)  # warm
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        bf.syrk_lower(-1.0, a21, 1.0, a22, cfg=cfg)
        e1.record(stream)
        e1.synchronize()
        ms += e0.elapsed_time(e1)
        flops += float(nk) * (nk + 1) * bs
        launches += 1
    del work
    achieved = flops / (ms / 1e3) / 1e12
    traffic, traffic_note = None, None
    tpath = ROOT / "profiles" / "r02_syrk_traffic.json"
    if tpath.exists():
        t = json.loads(tpath.read_text())
        traffic = t["traffic_bytes"]
        traffic_note = (f"dram read+write of one launch ({t['launch']}) from {t['source']}; algorithmic "
                        f"{t['algorithmic_bytes'] / 1e9:.2f} GB for that launch")
    return {"bound": "tensor", "achieved": round(achieved, 3), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": round(achieved / FP64_PEAK_TFLOPS, 4), "traffic": traffic, "traffic_note": traffic_note,
            "kernel": "gemm_dmma_tma_kernel<m8n8k4, 2x16-k TMA boxes, 2 stages, BN=64>: two 8-warp groups per "
                      "CTA on 128x64 tiles (GEMMT lower, trailing SYRK)",
            "per_launch_flops": "n_k*(n_k+1)*bs, n_k = n-(k+1)*bs", "launches_timed": launches,
            "syrk_ms_total": round(ms, 3), "peak_source": FP64_PEAK_SOURCE}


def dist_tree(world: int) -> dict:
    """Tile size of the 2D block-cyclic layout = the root bs: 2048 (the bench
    tree) up to 2 GPUs, 1024 beyond, so the per-step panel chain (diagonal
    factor + panel TRSM + broadcasts) stays under each step's share of the
    trailing update on 4-8 GPUs."""
    doc = json.loads(json.dumps(GPU_TREE))
    if world > 2:
        doc["bs"], doc["kernel"]["kc"] = 1024, 1024
    return doc


def run_distributed(args, bf, torch, dist, dev, world: int, rank: int, n: int) -> int:
    """All ranks factor ONE n x n matrix with the native NCCL driver
    (bf_chol_dist_d): lower tiles only, 2D block-cyclic over grid_for(world),
    each rank generating its own tiles (no rank ever holds the whole matrix),
    row/column communicators, panel broadcasts under the trailing updates.
    At one rank (--dist) it is the same NCCL path on a 1x1 grid."""
    from paper_2604_07311_b200.control import parse_tree
    from paper_2604_07311_b200.dist import native
    from paper_2604_07311_b200.engine import _lib

    tree_doc = dist_tree(world) if args.tree == json.dumps(GPU_TREE) else json.loads(args.tree)
    tree = parse_tree(json.dumps(tree_doc))
    ctx = native.DistContext.from_torch_distributed()
    for kv in filter(None, os.environ.get("BF_DIST_OPTS", "").split(",")):  # e.g. BF_DIST_OPTS=fan=0,reserve=24
        k, v = kv.split("=")
        ctx.set_option(k, int(v))
    lp = ctx.layout(n, tree.bs)
    local0 = torch.empty(lp.local_elems(), dtype=torch.float64, device=dev)
    native.fill_synthetic(ctx, local0, n, tree.bs, seed=42)
    work = torch.empty_like(local0)
    stream = torch.cuda.current_stream()

    def one(timed):
        work.copy_(local0)  # restore outside the events
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        bad = native.cholesky_dist(ctx, work, n, tree)
        e1.record(stream)
        e1.synchronize()
        assert bad == -1
        if timed is not None:
            timed.append(e0.elapsed_time(e1))

    for _ in range(args.warmup):
        one(None)
    lib = _lib.lib()
    timed: list = []
    l0 = lib.bf_launch_count()
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clocks:
        for _ in range(args.steps):
            one(timed)
    launches = (lib.bf_launch_count() - l0) // max(1, args.steps)
    t = torch.tensor([sum(timed) / len(timed)], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = chol_flops(n) / (ms / 1e3) / 1e9
    e2e = None
    if not args.no_e2e:
        host = torch.empty(local0.numel(), dtype=torch.float64, pin_memory=True)
        host.copy_(local0)
        out = torch.empty_like(host).pin_memory()
        e2e_ms = []
        for i in range(1 + args.e2e_steps):
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            work.copy_(host, non_blocking=True)
            native.cholesky_dist(ctx, work, n, tree)
            out.copy_(work, non_blocking=True)
            e1.record(stream)
            e1.synchronize()
            if i:
                e2e_ms.append(e0.elapsed_time(e1))
        t2 = torch.tensor([sum(e2e_ms) / len(e2e_ms)], device=dev)
        dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        nbytes = local0.numel() * 8
        e2e = {"value": round(chol_flops(n) / (float(t2.item()) / 1e3) / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "ms_per_step": round(float(t2.item()), 3),
               "path": "per rank: pinned host lower panels -> HBM, bf_chol_dist_d (NCCL), HBM -> pinned host"}
        del host, out
    if rank == 0:
        line = {
            "metric": "Cholesky GFLOP/s (n=32768 FP64)", "value": round(value, 3), "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic SPD: A = S + n I, S symmetric U[-1,1) from a counter hash, each rank generating "
                    "its own lower tiles on device (bf_dist_fill_synthetic_d)",
            "config": {"workload": f"FP64 blocked Cholesky n={n}, 2D block-cyclic over {ctx.pr}x{ctx.pc} GPUs "
                                   "(BASELINE configs[1]/[2])",
                       "n": n, "tree": tree_doc, "parallelism": f"2D block-cyclic {ctx.pr}x{ctx.pc}, lower tiles "
                       "only, NCCL row/column broadcasts (bf_chol_dist_d)",
                       "local_elems_rank0": lp.local_elems(), "l2": "matrix >> L2"},
            "pct_of_fp64_peak": round(100 * value / world / 1e3 / FP64_PEAK_TFLOPS, 2),
            "roofline": None, "cpu_baseline": None, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clocks.summary(), "step_ms": [round(x, 3) for x in timed],
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()
    return 0


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    # --order (alias --n): under torchrun "--n" after the script name is taken
    # as an abbreviation of torchrun's own options
    ap.add_argument("--order", "--n", dest="n", type=int, default=N_DEFAULT)
    ap.add_argument("--tree", type=str, default=json.dumps(GPU_TREE))
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-roofline", action="store_true")
    ap.add_argument("--no-side", action="store_true", help="skip the C4 mixed / C5 contraction side measurements")
    ap.add_argument("--tiles-per-cta", type=int, default=None, help="library option (tuning)")
    ap.add_argument("--dist", action="store_true", help="use the distributed driver even at one rank")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = args.n
    workload = f"FP64 blocked Cholesky n={n}, two-level blocking (BASELINE configs[1])"

    if args.impl == "reference":
        if rank != 0:
            return 0
        steps = []
        base = None
        for i in range(args.warmup + args.steps):
            base = cpu_baseline(n, budget_s=8.0)
            if i >= args.warmup:
                steps.append(base["value"])
        value = statistics.median(steps)
        line = {"metric": "Cholesky GFLOP/s (n=32768 FP64)", "value": round(value, 3), "unit": "GFLOP/s",
                "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic SPD (integer M, exact M M^T + n I), seed 42",
                "config": {"workload": workload, "tree": GPU_TREE, "sample_n": base["sample"]},
                "cpu_baseline": dict(base, value=round(value, 3)),
                "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import torch.distributed as dist

    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.control import parse_tree
    from paper_2604_07311_b200.engine import _lib

    if args.tiles_per_cta is not None:
        _lib.lib().bf_set_option(b"tiles_per_cta", args.tiles_per_cta)
    for kv in filter(None, os.environ.get("BF_OPTS", "").split(",")):  # library options for sweeps (tools/)
        k, v = kv.split("=")
        _lib.check(_lib.lib().bf_set_option(k.encode(), int(v)), f"bf_set_option({k})")
    torch.cuda.set_device(local)
    if world > 1 or args.dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", init_method="env://", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    tree = parse_tree(args.tree)

    if world > 1 or args.dist:
        return run_distributed(args, bf, torch, dist, dev, world, rank, n)

    a0 = make_spd(bf, torch, n, dev)
    work = torch.empty_like(a0)
    torch.cuda.synchronize()

    def one_step(timed: list | None):
        work.copy_(a0)
        v = bf.from_torch(work)
        stream = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        info = bf.cholesky_async(v, "lower", tree)
        e1.record(stream)
        if timed is not None:
            timed.append((e0, e1, info))
        return info

    for _ in range(args.warmup):
        info = one_step(None)
    torch.cuda.synchronize()
    assert int(info.item()) == -1, "warm-up factorization failed"

    lib = _lib.lib()
    timed: list = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.bf_launch_count()
    with ClockSampler(local) as clocks:
        wall0 = time.perf_counter()
        for _ in range(args.steps):
            one_step(timed)
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    launches = (lib.bf_launch_count() - launches0) // max(1, args.steps)
    if world > 1:
        dist.barrier()
    for _, _, info in timed:
        assert int(info.item()) == -1
    step_ms = [e0.elapsed_time(e1) for e0, e1, _ in timed]
    ms = sum(step_ms) / len(step_ms)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = chol_flops(n) * world / (ms / 1e3) / 1e9

    # ---- end to end through the public API from host memory -------------
    e2e = None
    if not args.no_e2e:
        pristine = a0.cpu()
        host = torch.empty(n, n, dtype=torch.float64, pin_memory=True)
        dev_buf = work
        e2e_ms = []
        for i in range(1 + args.e2e_steps):
            host.copy_(pristine)  # reset outside the timed region
            torch.cuda.synchronize()
            stream = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            bf.cholesky_host(host, "lower", tree, work=dev_buf)  # syncs to read the pivot flag
            e1.record(stream)
            e1.synchronize()
            if i > 0:
                e2e_ms.append(e0.elapsed_time(e1))
        ems = sum(e2e_ms) / len(e2e_ms)
        bs_root = tree.bs or n
        nbytes = sum((n - c0) * min(bs_root, n - c0) * 8 for c0 in range(0, n, bs_root))
        e2e = {"value": round(chol_flops(n) * world / (ems / 1e3) / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "ms_per_step": round(ems, 3),
               "path": "paper_2604_07311_b200.cholesky_host(pinned host matrix): lower triangle to HBM by block "
                       "columns overlapped with step 0, factor, each finished block column back to the host under "
                       "the remaining steps"}
        del host, pristine

    roof = None
    if not args.no_roofline and rank == 0:
        bs = tree.bs or 128
        kc = (tree.kernel or {}).get("kc", 256)
        roof = roofline_syrk(bf, torch, a0, n, bs, kc)
        roof["share_of_step"] = round(roof["syrk_ms_total"] / ms, 4)

    cpu = None
    if not args.no_cpu and rank == 0 and world == 1:
        cpu = cpu_baseline(n)

    side = None
    if not args.no_side and rank == 0 and world == 1:
        side = side_workloads(torch, a0, n, ms, l64=work)

    if rank == 0:
        clk = clocks.summary()
        line = {
            "metric": "Cholesky GFLOP/s (n=32768 FP64)",
            "value": round(value, 3),
            "unit": "GFLOP/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms, 3),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic: A = M M^T + n I, M ~ U(-1,1) seed 42 (reference generator cli.py:55-64), formed on device",
            "config": {"workload": workload, "n": n, "tree": json.loads(args.tree),
                       "l2": "input 8.6 GB >> 126 MB L2 (no flush needed); pristine copy restored outside the events",
                       "parallelism": f"replicas x{world}" if world > 1 else "1 GPU"},
            "pct_of_fp64_peak": round(100 * value / world / 1e3 / FP64_PEAK_TFLOPS, 2),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "side_workloads": side,
            "gpu_launches": int(launches),
            "clocks": clk,
            "wall_s_timed": round(wall, 3),
            "step_ms": [round(x, 3) for x in step_ms],
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

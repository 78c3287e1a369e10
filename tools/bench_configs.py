#!/usr/bin/env python3
"""Reconstruction-level measurements for BASELINE.json configs 0, 2, 3 and 4.

bench.py is the driver's contract (config 1, the operator microbenchmark); this
tool measures the reconstructions the metric's "recon wall-time" half refers to
and checks them against the CPU oracle where the oracle finishes.

  python tools/bench_configs.py --config 0 [--oracle]
  python tools/bench_configs.py --config 3 [--oracle]
  torchrun --nproc-per-node N tools/bench_configs.py --config 2     (slices sharded, no collective)
  torchrun --nproc-per-node N tools/bench_configs.py --config 4     (coils sharded, NCCL all-reduce)

Each run prints one JSON line (rank 0); bench.py imports these functions for its `recon`
and `sharded` objects.  GPU times are CUDA events on the launching stream around the whole
call (so host work inside the call counts), max over ranks for N > 1; inputs are seeded
synthetic data with the config's shapes.
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def _dist():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SR_DIST_BACKEND=gloo exercises the multi-rank logic on a box with fewer GPUs than ranks
    # (ranks share devices round-robin; collectives through the host).  Timing runs use NCCL.
    backend = os.environ.get("SR_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
    return rank, world, dev


def _max_over_ranks(v, world, dev):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _nrmse(x, ref):
    return float(np.linalg.norm(np.abs(x) - np.abs(ref)) / np.linalg.norm(ref))


# ----------------------------------------------------------------------------- 2-D (configs 0 and 3)
def run_2d(cfgid: int, with_oracle: bool):
    import torch
    from oracle import sketch_oracle as O
    from paper_2305_06482_b200 import coil_sketch as cs
    from paper_2305_06482_b200 import forward_model as fm
    from paper_2305_06482_b200 import linops as lo
    from paper_2305_06482_b200 import sketching as sk
    from paper_2305_06482_b200 import solvers as so
    from paper_2305_06482_b200 import synth
    rank, world, dev = _dist()
    rng = np.random.default_rng(0)
    if cfgid == 0:
        dims, C, v, s, lam, T, K = (256, 256), 16, 4, 4, 1e-3, 10, 10
        mask = synth.vd_poisson_mask(dims, 4.0, 24, 0)
        pts = synth.mask_points(mask)
        traj = lo.Trajectory(pts, "cartesian-mask")
        weights = None
        okern = O.CartesianKernel(dims, pts)
        kern = None
        wdesc = "VD Poisson-disc R=4, 24x24 centre"
    else:
        dims, C, v, s, lam, T, K = (320, 320), 16, 4, 4, 5e-4, 15, 8
        pts = synth.golden_angle_radial(128, 640, dims)
        traj = lo.Trajectory(pts, "non-cartesian")
        weights = fm.radial_density_weights(traj)
        okern = O.GriddedKernel(dims, pts, 2.0, 4)
        from paper_2305_06482_b200.nufft import GriddedKernel
        kern = GriddedKernel(dims, pts, 2.0, 4)
        wdesc = "golden-angle radial 128 x 640, KB 2x / w4, ramp DCF"
    shape = lo.GridShape(dims)
    truth = synth.random_ellipses(dims, 10, rng).ravel()
    maps = synth.gaussian_coil_maps(dims, C, rng)
    clean = O.Sense(maps, okern).forward(truth).reshape(C, -1)
    data = clean + synth.complex_noise(clean.shape, 0.01 * np.abs(clean).max(), rng)
    reg = so.make_regularizer("l1-wavelet", lam, shape)
    cfg = cs.CoilSketchConfig(C, sk.SketchConfig(v + s, v, s, rademacher_scale=12 ** -0.5), reg, T, K)
    # warm-up (plans, workspaces, first-launch costs, the first CUDA-graph captures of the process:
    # 3 outers), then the timed reconstructions
    cs.coil_sketching_recon(fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps),
                            cs.CoilSketchConfig(C, cfg.sketch, reg, 3, 1), weights=weights, kernel=kern)
    compress = "lapack" if os.environ.get("SR_HOST_COMPRESS") else "device"
    runs = []
    rep = None
    for _ in range(3):
        # the previous run's report (and whatever else this process left behind: bench.py runs several
        # configurations and a CPU oracle in one process) is released and collected outside the timed
        # region
        rep = None
        gc.collect()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rep = cs.coil_sketching_recon(fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps), cfg,
                                      weights=weights, kernel=kern, compress=compress)
        e1.record()
        torch.cuda.synchronize()
        runs.append(e0.elapsed_time(e1) / 1e3)
    t_gpu = float(np.median(runs))
    if os.environ.get("SR_PROFILE_RECON"):
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
            cs.coil_sketching_recon(fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps), cfg,
                                    weights=weights, kernel=kern, compress=compress)
            torch.cuda.synchronize()
        evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
        busy = sum(e.time_range.end - e.time_range.start for e in evs)
        span = max(e.time_range.end for e in evs) - min(e.time_range.start for e in evs)
        print(f"GPU kernels+copies: {len(evs)} events, busy {busy / 1e3:.1f} ms of a {span / 1e3:.1f} ms span",
              flush=True)
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=14), flush=True)
    line = {"config": cfgid, "what": f"coil-sketched recon {dims} C={C} -> {v}+{s}, {T}x{K} FISTA, {wdesc}",
            "gpu_wall_s": t_gpu, "gpu_wall_s_runs": runs, "compress": compress, "counts": rep.counts.get("coil_transform"),
            "expected_counts": cs.expected_coil_transforms(cfg, so.SolverConfig(tol=0.0)),
            "objectives": [r.objective for r in rep.per_outer], "data": "synthetic"}
    if with_oracle:
        t0 = time.perf_counter()
        ref = O.coil_sketching_recon(data, maps, dims, lambda: okern, c_hat0=C, v=v, s=s, lam=lam, outer=T, inner=K,
                                     weights=None if weights is None else weights.w, rademacher_scale=12 ** -0.5)
        line["cpu_oracle_wall_s"] = time.perf_counter() - t0
        line["cpu_cores"] = 1
        line["nrmse_vs_oracle"] = _nrmse(rep.x_final.values, ref.x_final)
        line["rel_l2_vs_oracle"] = float(np.linalg.norm(rep.x_final.values - ref.x_final) / np.linalg.norm(ref.x_final))
        line["oracle_objectives"] = ref.objectives
        line["speedup"] = line["cpu_oracle_wall_s"] / t_gpu
    return line


# ----------------------------------------------------------------------------- config 2
def _oracle_slice(args):
    """One config-2 slice reconstruction through the oracle (process-pool worker)."""
    from oracle import sketch_oracle as O
    yh, mh, dims, pts, C, V, S = args
    okern = O.CartesianKernel(dims, pts)
    return O.coil_sketching_recon(yh, mh, dims, lambda: okern, c_hat0=C, v=V, s=S, lam=1e-3, outer=10, inner=10,
                                  rademacher_scale=12 ** -0.5).x_final


def run_cfg2(with_oracle: bool, nslices_total: int = 256, pool: int = 0):
    import torch
    from oracle import sketch_oracle as O
    from paper_2305_06482_b200 import coil_sketch as cs
    from paper_2305_06482_b200 import linops as lo
    from paper_2305_06482_b200 import sketching as sk
    from paper_2305_06482_b200 import solvers as so
    from paper_2305_06482_b200 import synth
    from paper_2305_06482_b200.cartesian import CartesianKernel
    from paper_2305_06482_b200.parallel_recon import ReadoutDecoupler, compress_slices, gather_slices, shard_range
    from paper_2305_06482_b200.plan import cartesian_plan
    rank, world, dev = _dist()
    NX, NY, NZ, C, V, S = 256, 256, 160, 32, 6, 6
    lo_s, hi_s = shard_range(nslices_total, rank, world)
    nloc = hi_s - lo_s
    dims = (NY, NZ)
    D = NY * NZ
    rng = np.random.default_rng(0)  # identical inputs on every rank
    mask = synth.vd_poisson_mask(dims, 8.0, 20, 0)
    pts = synth.mask_points(mask)
    N = len(pts)
    vol = synth.random_ellipses((NX, NY, NZ), 20, rng, planes=(lo_s, hi_s))  # this rank's slab only
    maps3 = synth.coil_maps_cylinder((NX, NY, NZ), C, rng, xp=torch, device=dev)  # (C, NX*NY*NZ)
    # this rank's slices: maps (nloc, C, D), acquisition through the 3-D Cartesian model
    maps = maps3.view(C, NX, D)[:, lo_s:hi_s].permute(1, 0, 2).contiguous()
    del maps3
    x_true = torch.from_numpy(vol.reshape(nloc, D).astype(np.complex64)).to(dev)
    kern = CartesianKernel(dims, [cartesian_plan(dims, pts)], batch=nloc)
    y2 = kern.forward(maps, x_true)  # (nloc, C, N) per-slice data
    sig = 0.01 * float(torch.abs(y2).max())
    gen = torch.Generator(dev).manual_seed(1234 + rank)
    y2 = y2 + (torch.randn(y2.shape, dtype=torch.complex64, device=dev, generator=gen) * sig)
    # 3-D k-space of this rank's slab along kx is not separable across ranks; the readout
    # decoupling (K8) is exercised per rank on its own slab (its slices' readout transform):
    kx = torch.fft.fftshift(torch.fft.fft(torch.fft.ifftshift(y2.permute(1, 0, 2), dim=1), dim=1, norm="ortho"), dim=1)
    dec = ReadoutDecoupler(nloc) if _lib_supported(nloc) else None
    reg = so.make_regularizer("l1-wavelet", 1e-3, lo.GridShape(dims))
    cfg = cs.CoilSketchConfig(C, sk.SketchConfig(V + S, V, S, rademacher_scale=12 ** -0.5), reg, 10, 10)
    # the pipeline runs twice; the first run (library handles, graph capture, allocator) is a warm-up
    for _rep in range(2):
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        y = dec(kx.contiguous()) if dec is not None else y2
        ev[1].record()
        maps0, y0, comp = compress_slices(maps, y, C)
        ev[2].record()
        res = cs.coil_sketching_recon_batched(kern, maps0, y0, cfg, dims)
        ev[3].record()
        torch.cuda.synchronize()
        t_start, t_dec, t_comp, t_end = 0.0, *(ev[0].elapsed_time(e) / 1e3 for e in ev[1:])
        t_solve0 = t_comp
    if os.environ.get("SR_PROFILE_RECON") and rank == 0:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            cs.coil_sketching_recon_batched(kern, maps0, y0, cfg, dims)
            torch.cuda.synchronize()
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=16), flush=True)
    full = gather_slices(res.x, nslices_total, rank, world)
    t_wall = _max_over_ranks(t_end - t_start, world, dev)
    t_solve = _max_over_ranks(t_end - t_solve0, world, dev)
    line = None
    if rank == 0:
        line = {"config": 2, "what": f"{nslices_total} readout-decoupled slices {dims}, C={C} -> {V}+{S}, 10x10 FISTA",
                "n_gpus": world, "scaling": "strong", "gpu_wall_s": t_wall, "gpu_solve_s": t_solve,
                "slices_per_s": nslices_total / t_wall, "k_decoupled_with_K8": dec is not None,
                "readout_idft_s": t_dec - t_start, "compression_s": t_comp - t_dec,
                "samples_per_slice": N, "data": "synthetic"}
    if with_oracle and rank == 0:
        # oracle on a bounded sample: the first 2 slices of rank 0 (same comp)
        xs = res.x.cpu().numpy()
        yh = y.cpu().numpy().astype(np.complex128)
        mh = maps.cpu().numpy().astype(np.complex128)
        okern = O.CartesianKernel(dims, pts)
        errs, tt = [], 0.0
        for sl in range(min(2, nloc)):
            t0 = time.perf_counter()
            ref = O.coil_sketching_recon(yh[sl], mh[sl], dims, lambda: okern, c_hat0=C, v=V, s=S, lam=1e-3,
                                         outer=10, inner=10, rademacher_scale=12 ** -0.5)
            tt += time.perf_counter() - t0
            errs.append(_nrmse(xs[sl], ref.x_final))
        line["oracle_slices"] = len(errs)
        line["nrmse_vs_oracle_max"] = max(errs)
        line["cpu_oracle_s_per_slice"] = tt / len(errs)
        line["cpu_oracle_extrapolated_s"] = tt / len(errs) * nslices_total
        if pool > 0:
            import multiprocessing as mp
            from concurrent.futures import ProcessPoolExecutor
            cores = len(os.sched_getaffinity(0))
            k = min(pool, nloc)
            tasks = [(yh[sl], mh[sl], dims, pts, C, V, S) for sl in range(k)]
            # single-threaded BLAS in the spawned workers (read when they import numpy)
            saved = {v: os.environ.get(v) for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")}
            for v in saved:
                os.environ[v] = "1"
            t0 = time.perf_counter()
            with ProcessPoolExecutor(max_workers=min(cores, k), mp_context=mp.get_context("spawn")) as ex:
                outs = list(ex.map(_oracle_slice, tasks))
            t_pool = time.perf_counter() - t0
            for v, val in saved.items():
                if val is None:
                    os.environ.pop(v, None)
                else:
                    os.environ[v] = val
            line["cpu_pool"] = {"slices": k, "processes": min(cores, k), "cores": cores, "wall_s": t_pool,
                                "extrapolated_s": t_pool * nslices_total / k,
                                "nrmse_max": max(_nrmse(xs[sl], outs[sl]) for sl in range(k))}
    return line


def _lib_supported(n):
    from paper_2305_06482_b200 import _lib
    return bool(_lib.lib().sr_fft_size_supported(n)) and n >= 2


# ----------------------------------------------------------------------------- config 4
def run_cfg4(with_oracle: bool, scale: float = 1.0, outer: int = 10, inner: int = 10):
    import torch
    from paper_2305_06482_b200 import synth
    from paper_2305_06482_b200.linops import CostCounter
    from paper_2305_06482_b200.nufft import GriddedKernel
    from paper_2305_06482_b200.parallel_recon import CoilShard
    from paper_2305_06482_b200.recon import SketchedReconEngine
    from paper_2305_06482_b200.sketching import SketchConfig, coil_contract
    rank, world, dev = _dist()
    dims = tuple(int(round(n * scale)) for n in (256, 256, 160))
    C, V, S = 32, 8, 8
    pts = synth.cones_3d(dims, n_readouts=int(18000 * scale * scale), n_samples=int(512 * scale))
    N = len(pts)
    rng = np.random.default_rng(0)
    GriddedKernel(dims, pts[:4096], 1.25, 4)  # warm-up (sort / allocator first use)
    torch.cuda.synchronize()
    t_plan0 = time.perf_counter()
    kern = GriddedKernel(dims, pts, 1.25, 4)  # device plan (csrc/nufft_plan.cu), host fp64 trajectory in
    torch.cuda.synchronize()
    t_plan = time.perf_counter() - t_plan0
    D = kern.D
    maps = synth.coil_maps_cylinder(dims, C, rng, xp=torch, device=dev).unsqueeze(0).contiguous()  # (1, C, D)
    vol = torch.from_numpy(synth.random_ellipses(dims, 20, rng).ravel().astype(np.complex64)).to(dev).view(1, -1)
    r = np.linalg.norm(pts, axis=1)
    w = np.where(r > 1e-12 * max(r.max(), 1.0), r, 0.5 * r[r > 1e-12 * max(r.max(), 1.0)].min())
    w = w / w.max()
    sqrt_w = torch.from_numpy(np.sqrt(w)).to(dev)
    # acquisition (unweighted) in coil chunks, then weighting, noise
    y = torch.empty(1, C, N, dtype=torch.complex64, device=dev)
    for c0 in range(0, C, 8):
        y[:, c0:c0 + 8] = kern.forward(maps[:, c0:c0 + 8].contiguous(), vol)
    sig = 0.01 * float(torch.abs(y).max())
    gen = torch.Generator(dev).manual_seed(7)
    y = y + torch.randn(y.shape, dtype=torch.complex64, device=dev, generator=gen) * sig
    y = y * sqrt_w.to(torch.float32)
    # PCA compression (keep = C) from the data Gram matrix on the device (phases differ from LAPACK;
    # this run is a timing, not a parity run)
    gram = (y[0] @ y[0].conj().T).to(torch.complex128)
    evals, evecs = torch.linalg.eigh(gram)
    comp = evecs.flip(-1).conj().T.to(torch.complex64)
    maps0 = coil_contract(maps, comp.unsqueeze(0))
    y0 = coil_contract(y, comp.unsqueeze(0))
    del maps, y
    shard = CoilShard(rank, world)
    sk = SketchConfig(V + S, V, S, rademacher_scale=12 ** -0.5)
    eng = SketchedReconEngine(kern, maps0, y0, dims=dims, sketch=sk, lam=1e-3, sqrt_w=sqrt_w, shard=shard,
                              counter=CostCounter())
    # one sketched normal-op apply (this rank's coils + all-reduce), timed
    from paper_2305_06482_b200.rng import child_seed
    from paper_2305_06482_b200.sketching import gen_sketch_matrix
    mat = gen_sketch_matrix(sk.with_seed(child_seed(0, 1)), C).mat
    smaps = eng._sketch(mat)
    xin = vol.clone()
    out = torch.empty_like(xin)
    eng._normal(smaps, xin, out)
    torch.cuda.synchronize()
    reps = 5
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        eng._normal(smaps, xin, out)
    e1.record()
    torch.cuda.synchronize()
    t_apply = _max_over_ranks(e0.elapsed_time(e1) / 1e3 / reps, world, dev)
    if os.environ.get("SR_PROFILE_APPLY") and rank == 0:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            eng._normal(smaps, xin, out)
            torch.cuda.synchronize()
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15), flush=True)
    if os.environ.get("SR_PROFILE_RECON") and rank == 0:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
            eng.run(2, inner)
            torch.cuda.synchronize()
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25), flush=True)
    if outer > 0:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = eng.run(outer, inner)
        e1.record()
        torch.cuda.synchronize()
        t_recon = _max_over_ranks(e0.elapsed_time(e1) / 1e3, world, dev)
    else:
        res, t_recon = None, None
    line = {"config": 4, "what": f"3-D cones {dims}, N={N}, KB 1.25x/w4, C={C} -> {V}+{S}, "
                                 f"{outer}x{inner} FISTA, coils sharded over {world} GPU(s)",
            "n_gpus": world, "scaling": "strong", "sketched_normal_apply_s": t_apply,
            "recon_wall_s": t_recon, "plan_build_s": t_plan,
            "objectives": None if res is None else res.objectives[:, 0].tolist(),
            "counts": None if res is None else res.counts, "data": "synthetic"}
    if with_oracle and rank == 0:
        # full-size CPU reference path on a bounded sample: the sketched normal op of ONE of the
        # 16 sketched coils through the oracle (numpy complex128, one core, tap tables per chunk of
        # 1 M samples to bound memory), timed and compared with the device result for that coil
        from oracle import sketch_oracle as O
        m1 = smaps[:, :1].contiguous()
        o1 = torch.empty_like(xin)
        kern.normal(m1, xin, o1, w=sqrt_w)
        okern = O.ChunkedGriddedKernel(dims, pts, 1.25, 4)
        osense = O.Sense(m1[0].cpu().numpy().astype(np.complex128), okern, w)
        t0 = time.perf_counter()
        ref = osense.normal(xin[0].cpu().numpy().astype(np.complex128))
        t_cpu = time.perf_counter() - t0
        # the reference builds its interpolator once (setup); the chunked oracle rebuilds the tap
        # tables in apply and in apply_adjoint, so that time is measured and taken out
        t0 = time.perf_counter()
        for s0 in range(0, okern.n_points, okern.chunk):
            okern._taps(okern.points[s0:s0 + okern.chunk])
        t_taps = time.perf_counter() - t0
        got = o1[0].cpu().numpy()
        line["oracle_one_coil_rel_l2"] = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
        line["cpu_oracle_one_coil_normal_s"] = t_cpu
        line["cpu_oracle_tap_tables_s"] = 2 * t_taps
        line["cpu_oracle_apply_extrapolated_s"] = (t_cpu - 2 * t_taps) * (V + S)
        line["cpu_oracle_sample"] = ("sketched normal op of 1 of the 16 sketched coils at full size (N = 9.2 M), "
                                     "numpy complex128, one core, interpolator construction excluded, x 16")
        line["cpu_cores"] = 1
        line["speedup_apply_vs_cpu"] = line["cpu_oracle_apply_extrapolated_s"] / t_apply
    return line if rank == 0 else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True, choices=[0, 2, 3, 4])
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--slices", type=int, default=256)
    ap.add_argument("--scale", type=float, default=1.0, help="config 4 geometry scale (1.0 = full size)")
    ap.add_argument("--oracle-pool", type=int, default=0,
                    help="config 2: also run this many slice reconstructions of the oracle in a process pool "
                         "(one per host core, OPENBLAS_NUM_THREADS=1) and extrapolate to all slices")
    ap.add_argument("--outer", type=int, default=10)
    ap.add_argument("--inner", type=int, default=10)
    a = ap.parse_args()
    if a.config in (0, 3):
        line = run_2d(a.config, a.oracle)
    elif a.config == 2:
        line = run_cfg2(a.oracle, a.slices, a.oracle_pool)
    else:
        line = run_cfg4(a.oracle, a.scale, a.outer, a.inner)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

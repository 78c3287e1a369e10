"""The config-4 coil-sharded device engine (coils sharded, image-domain coil
sum all-reduced, forward_model.py:180 being the sum it replaces) executed end to end: two
ranks in two processes, gloo on CUDA tensors (this box has one GPU; the collective goes
through the host, so no rank's kernels wait on another's), against the unsharded engine on
the same inputs.  Checks the final image, the per-outer objectives, the Lipschitz constant
and the coil-transform counters (each rank keeps the reference tally of the whole operator)."""

import os
import socket

import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _engine_inputs(g, dev):
    from paper_2305_06482_b200 import forward_model as fm
    from paper_2305_06482_b200 import linops as lo
    from paper_2305_06482_b200.nufft import GriddedKernel
    dims = tuple(int(n) for n in g["dims"])
    shape = lo.GridShape(dims)
    traj = lo.Trajectory(g["points"], "non-cartesian")
    kern = GriddedKernel(dims, g["points"], float(g["oversamp"]), int(g["width"]))
    w = fm.DensityWeights(g["weights"])
    maps0, data0, _, _ = fm.coil_compress_device(fm.KSpaceData(traj, g["data"]), fm.SensitivityMaps(shape, g["maps"]),
                                                 int(g["chat0"]))
    sqrt_w = torch.from_numpy(np.sqrt(w.w)).to(dev, torch.float32)
    y = (data0 * sqrt_w.to(torch.complex64)).view(1, int(g["chat0"]), -1).contiguous()
    return dims, kern, maps0.view(1, int(g["chat0"]), -1).contiguous(), y, sqrt_w


def _run(g, dev, shard):
    from paper_2305_06482_b200.recon import SketchedReconEngine
    from paper_2305_06482_b200.sketching import SketchConfig
    dims, kern, maps0, y, sqrt_w = _engine_inputs(g, dev)
    v, s = int(g["v"]), int(g["s"])
    eng = SketchedReconEngine(kern, maps0, y, dims=dims, sketch=SketchConfig(v + s, v, s, rademacher_scale=float(g["scale"])),
                              lam=float(g["lam"]), sqrt_w=sqrt_w, shard=shard)
    res = eng.run(int(g["outer"]), int(g["inner"]))
    return res


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_06482_b200.parallel_recon import CoilShard
        g = golden("recon_cones3d")
        res = _run(g, torch.device("cuda", 0), CoilShard(rank, world))
        q.put((rank, res.x.cpu().numpy(), np.asarray(res.objectives), float(res.lipschitz[0]),
               int(res.counts["coil_transform"])))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, repr(e), None, None, None))
        raise
    finally:
        dist.destroy_process_group()


def test_coil_sharded_engine_world2_matches_unsharded(cuda):
    import torch.multiprocessing as mp
    g = golden("recon_cones3d")
    ref = _run(g, cuda, None)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    xr = ref.x.cpu().numpy()
    for rank, x, objs, lip, cnt in outs:
        assert not isinstance(x, str), x
        assert np.linalg.norm(x - xr) / np.linalg.norm(xr) < 1e-5, rank
        np.testing.assert_allclose(objs, ref.objectives, rtol=1e-5)
        assert abs(lip - float(ref.lipschitz[0])) < 1e-5 * abs(lip)
        assert cnt == int(ref.counts["coil_transform"])
    # both ranks hold the same (replicated) image
    assert np.array_equal(outs[0][1], outs[1][1])


# --- slab-pipelined all-reduce (the coil sum of a 3-D NUFFT normal op finished one slab of image
# planes at a time, each slab's all-reduce overlapping the next slab's inverse passes)
SLAB_DIMS = (128, 96, 32)  # 128 x 96 = 12288 image rows: the fused row pass, so slabs apply


def _slab_problem(dev, coils=6):
    from paper_2305_06482_b200 import synth
    from paper_2305_06482_b200.nufft import GriddedKernel
    pts = synth.cones_3d(SLAB_DIMS, n_readouts=300, n_samples=200)
    kern = GriddedKernel(SLAB_DIMS, pts, 1.25, 4)
    g = torch.Generator(dev).manual_seed(7)
    D = kern.D
    maps = torch.randn(1, coils, D, dtype=torch.complex64, device=dev, generator=g) * 0.3
    x = torch.randn(1, D, dtype=torch.complex64, device=dev, generator=g)
    return kern, maps, x, pts


def test_nufft_normal_slabs_equal_normal(cuda):
    """head + per-slab tails == the one-call normal op (same kernels per output row; the gridding
    flush's float atomics make two calls of either agree to fp32 rounding, not bitwise), with and
    without the solver epilogue; a partial slab on a grid too small for it is refused."""
    kern, maps, x, _ = _slab_problem(cuda)
    assert kern.slab_planes() == SLAB_DIMS[0]
    a = torch.randn_like(x) * 0.1
    coef = torch.tensor([[0.5, -1.0, 0.25, 0.0]], device=cuda)
    dd = torch.randn_like(x)
    for kw in ({}, dict(anchor=a, coef=coef, u=x, d=dd)):
        ref = torch.empty_like(x)
        kern.normal(maps, x, ref, **kw)
        for nslab in (1, 3, 4):
            n0 = SLAB_DIMS[0]
            bounds = [(n0 * k // nslab, n0 * (k + 1) // nslab) for k in range(nslab)]
            seen = []
            out = torch.full_like(x, float("nan"))
            kern.normal_slabs(maps, x, out, bounds, lambda lo, hi: seen.append((lo, hi)), **kw)
            assert seen == bounds
            err = float(torch.linalg.vector_norm(out - ref) / torch.linalg.vector_norm(ref))
            assert err < 1e-6, (kw.keys(), nslab, err)
    from paper_2305_06482_b200 import synth
    from paper_2305_06482_b200.nufft import GriddedKernel
    small = GriddedKernel((16, 24, 16), synth.cones_3d((16, 24, 16), n_readouts=40, n_samples=60), 1.25, 4)
    assert small.slab_planes() == 0
    m2 = torch.ones(1, 1, small.D, dtype=torch.complex64, device=cuda)
    x2 = torch.ones(1, small.D, dtype=torch.complex64, device=cuda)
    with pytest.raises(ValueError):
        small.normal_slabs(m2, x2, torch.empty_like(x2), [(0, 10), (10, 20)], lambda lo, hi: None)


def test_nufft_coil_looped_embed_equals_one_shot(cuda):
    """The embed + row FFT pass with the coils looped inside the CTA (several coils, enough image rows)
    == the one-shot pass (taken for a single coil): the normal op over C coils equals the sum of the
    C single-coil normal ops, with and without the anchor."""
    kern, maps, x, _ = _slab_problem(cuda)
    a = torch.randn_like(x) * 0.1
    for kw in ({}, dict(anchor=a)):
        full = torch.empty_like(x)
        kern.normal(maps, x, full, **kw)
        acc = torch.zeros_like(x)
        one = torch.empty_like(x)
        for j in range(maps.shape[1]):
            kern.normal(maps[:, j:j + 1].contiguous(), x, one, **kw)
            acc += one
        err = float(torch.linalg.vector_norm(full - acc) / torch.linalg.vector_norm(acc))
        assert err < 2e-6, (list(kw), err)


def test_nufft_normal_pingpong_equals_normal(cuda):
    """The normal op with two spread grids used in turn (the idle one zeroed on a library stream while
    the gridding kernel runs, sr_nufft_normal_pp) == the one-grid normal op, over a run of calls with
    other workspace users (forward / adjoint, another coil count, the slab pipeline) in between."""
    kern, maps, x, _ = _slab_problem(cuda)
    ref = torch.empty_like(x)
    kern.normal(maps, x, ref)  # small grid: the plain path
    assert kern._pp is None
    x2 = torch.randn_like(x)
    ref2 = torch.empty_like(x)
    kern.normal(maps, x2, ref2)
    kern.PP_MIN_BYTES = 0  # force the ping-pong path on this small grid
    try:
        def close(a, b):
            return float(torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b)) < 1e-6
        out = torch.empty_like(x)
        for k in range(5):
            xin, want = (x, ref) if k % 2 == 0 else (x2, ref2)
            out.fill_(float("nan"))
            kern.normal(maps, xin, out)
            assert kern._pp == (maps.shape[1], (k + 1) % 2)
            assert close(out, want), k
        # other users of the workspace reset the state; the next call zeroes its own grid
        y = kern.forward(maps, x)
        assert kern._pp is None
        kern.adjoint(maps, y, torch.empty_like(x))
        kern.normal(maps, x, out)
        assert close(out, ref)
        kern.normal(maps[:, :2].contiguous(), x, torch.empty_like(x))  # another coil count
        kern.normal(maps, x2, out)
        assert close(out, ref2)
        n0 = SLAB_DIMS[0]
        kern.normal_slabs(maps, x, torch.empty_like(x), [(0, n0 // 2), (n0 // 2, n0)], lambda lo, hi: None)
        kern.normal(maps, x, out)
        kern.normal(maps, x2, out)
        assert close(out, ref2)
    finally:
        del kern.PP_MIN_BYTES  # back to the class default


def _slab_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_06482_b200.parallel_recon import CoilShard
        res = _slab_engine(torch.device("cuda", 0), CoilShard(rank, world))
        q.put((rank, res.x.cpu().numpy(), np.asarray(res.objectives), float(res.lipschitz[0])))
    except Exception as e:
        q.put((rank, repr(e), None, None))
        raise
    finally:
        dist.destroy_process_group()


def _slab_engine(dev, shard):
    from paper_2305_06482_b200.recon import SketchedReconEngine
    from paper_2305_06482_b200.sketching import SketchConfig
    kern, maps, x, pts = _slab_problem(dev, coils=8)
    g = torch.Generator(dev).manual_seed(11)
    y = torch.zeros(1, 8, kern.nmax, dtype=torch.complex64, device=dev)
    y[:, :, : kern.n_points] = torch.randn(1, 8, kern.n_points, dtype=torch.complex64, device=dev, generator=g)
    eng = SketchedReconEngine(kern, maps, y, dims=SLAB_DIMS, sketch=SketchConfig(4, 2, 2), lam=1e-3, shard=shard)
    return eng.run(2, 3)


def test_coil_sharded_slab_pipeline_world2_matches_unsharded(cuda):
    """Two gloo ranks run the engine whose sketched normal op all-reduces its coil sum slab by slab
    (async collectives); the image, objectives and step size match the unsharded engine."""
    import torch.multiprocessing as mp
    ref = _slab_engine(cuda, None)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    xr = ref.x.cpu().numpy()
    for rank, x, objs, lip in outs:
        assert not isinstance(x, str), x
        assert np.linalg.norm(x - xr) / np.linalg.norm(xr) < 1e-5, rank
        np.testing.assert_allclose(objs, ref.objectives, rtol=1e-5)
        assert abs(lip - float(ref.lipschitz[0])) < 1e-5 * abs(lip)

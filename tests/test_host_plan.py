"""CPU tests of the host side: C-ABI exports, perm-order layout tables.

The kernels' data flow (perm-order spectrum, mask, sample gather/scatter with
centering phases) is emulated here in numpy with the SAME host tables the GPU
consumes, and compared with the oracle -- so a layout bug is caught without a GPU.
"""

import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden, rel
from oracle import sketch_oracle as O
from paper_2305_06482_b200 import _lib, plan


def header_symbols():
    text = (ROOT / "include" / "sketchrecon_b200.h").read_text()
    return sorted(set(re.findall(r"\b(?:int|long long)\s+(sr_\w+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.exported_symbols())


def test_fft_split_table():
    for n in (256, 320, 160, 640, 200, 16, 20, 8):
        p, q = _lib.fft_split(n)
        assert p * q == n
        pos = plan.perm_positions(n)
        assert sorted(pos) == list(range(n))
    with pytest.raises(ValueError):
        _lib.fft_split(7 * 11)


def _emulate(dims, points, maps, x, y):
    pl = plan.cartesian_plan(dims, points)
    ny, nx = plan.grid2d(dims)
    D = ny * nx
    maskpp = pl.maskT.reshape(nx, ny).T  # [pos_y, pos_x]
    to_pp = lambda s: plan.to_perm_spectrum(s, ny, nx)  # noqa: E731
    py = plan.perm_positions(ny) if ny > 1 else np.zeros(1, int)
    px = plan.perm_positions(nx)
    from_pp = lambda s: s[..., py[:, None], px[None, :]]  # noqa: E731
    imgs = maps.reshape(-1, ny, nx) * x.reshape(ny, nx)
    spec = to_pp(np.fft.fft2(imgs))
    # forward: gather with phase, 1/sqrt(D)
    fwd = (spec.reshape(len(maps), -1)[:, pl.spos] * pl.ph) / np.sqrt(D)
    # normal: mask / D, inverse, conj coil sum
    nrm = np.fft.ifft2(from_pp(spec * maskpp / D)) * D
    nrm = np.sum(np.conj(maps.reshape(-1, ny, nx)) * nrm, axis=0).ravel()
    # adjoint: scatter (write list), conj phase, 1/sqrt(D)
    sp = np.zeros((len(maps), D), complex)
    yy = y.reshape(len(maps), -1)
    sp[:, pl.spos[pl.wlist]] = yy[:, pl.wlist] * np.conj(pl.ph[pl.wlist]) / np.sqrt(D)
    adj = np.fft.ifft2(from_pp(sp.reshape(-1, ny, nx))) * D
    adj = np.sum(np.conj(maps.reshape(-1, ny, nx)) * adj, axis=0).ravel()
    return fwd.ravel(), nrm, adj


@pytest.mark.parametrize("name", ["sense_cart", "sense_cart_b", "sense_cart_1d"])
def test_perm_layout_emulation_matches_reference(name):
    g = golden(name)
    dims = tuple(int(n) for n in g["dims"])
    fwd, nrm, adj = _emulate(dims, g["points"], g["maps"], g["x"], g["y"])
    assert rel(fwd, g["Ax"]) < 1e-12
    assert rel(nrm, g["AHAx"]) < 1e-12
    assert rel(adj, g["AHy"]) < 1e-12


def test_duplicate_bins_last_write_wins():
    pts = np.array([[0, 0], [1, 2], [0, 0], [-3, 1], [1, 2]], float)
    pl = plan.cartesian_plan((8, 8), pts)
    assert list(pl.wlist) == [2, 3, 4]
    assert pl.maskT.sum() == 3


def test_oracle_kernel_parity_small():
    # oracle self-consistency: adjointness of the Cartesian SENSE operator
    rng = np.random.default_rng(1)
    dims = (16, 12)
    pts = np.argwhere(rng.random(dims) < 0.4) - np.array([8, 6])
    maps = rng.standard_normal((3, 192)) + 1j * rng.standard_normal((3, 192))
    a = O.Sense(maps, O.CartesianKernel(dims, pts))
    u = rng.standard_normal(192) + 1j * rng.standard_normal(192)
    v = rng.standard_normal(3 * len(pts)) + 1j * rng.standard_normal(3 * len(pts))
    assert abs(np.vdot(v, a.forward(u)) - np.vdot(a.adjoint(v), u)) < 1e-10 * np.linalg.norm(u) * np.linalg.norm(v)


def test_support_safe_frac_keeps_float64_decisions():
    """fp32 KB offsets make the same keep/drop decision per tap as the reference's fp64
    (linops.py:404-410), including samples on grid lines up to 1e-16."""
    import numpy as np
    from paper_2305_06482_b200.nufft import support_safe_frac
    rng = np.random.default_rng(0)
    for w in (4, 5, 6):
        edge = np.array([5e-16, -5e-16, 0.0, 1e-12, -1e-12, 2.0, 2.0 - 4e-16, 3.0 + 1e-15, 0.5, 0.5 + 1e-16])
        u = np.concatenate([rng.uniform(-40, 40, 20000), edge, edge + 17.0]) * 1.25
        b = np.ceil(u - w / 2.0)
        t = support_safe_frac(u, b, w)
        assert t.dtype == np.float32
        assert np.max(np.abs(t.astype(np.float64) - (u - b))) < 1e-6
        for k in range(w):
            ref = (1.0 - (2.0 * (u - (b + k)) / w) ** 2) > 0
            dev = np.abs((np.float32(2.0) * (t - np.float32(k))) / np.float32(w)) < np.float32(1.0)
            assert np.array_equal(ref, dev), (w, k)


def _build_c_example(tmp_path):
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    out = tmp_path / "c_abi_normal"
    libdir = ROOT / "paper_2305_06482_b200" / "_native"
    cmd = [gcc, "-O2", "-std=c11", f"-I{ROOT / 'include'}", "-I/usr/local/cuda/include", "-o", str(out),
           str(ROOT / "examples" / "c_abi_normal.c"), f"-L{libdir}", "-lsketchrecon_b200",
           "-L/usr/local/cuda/lib64", "-lcudart", "-lm", f"-Wl,-rpath,{libdir}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_c_abi_example_compiles_and_links(tmp_path):
    """The header is plain C and the library exports what a C caller links (examples/)."""
    assert _build_c_example(tmp_path).exists()


@pytest.mark.gpu
def test_c_abi_example_runs(tmp_path):
    """A pure-C caller (no Python / torch): library-owned Cartesian plan + normal op vs a direct
    CPU DFT (examples/c_abi_normal.c exits 0 when the relative L2 error is below 1e-4)."""
    import subprocess
    exe = _build_c_example(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr

"""Build the sm_100a shared library in-tree: ``python -m paper_2305_06482_b200.build``.

Runs the DFT code generator, compiles every ``csrc/*.cu`` with
``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` in parallel and
links ``_native/libsketchrecon_b200.so`` (static cudart, C ABI only -- no torch
types cross the boundary).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_native"
LIB = OUT_DIR / "libsketchrecon_b200.so"
INCLUDE = ROOT / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
         "-Xptxas", "-O3", f"-I{INCLUDE}", f"-I{CSRC}"] + os.environ.get("SR_NVCC_EXTRA", "").split()


def _sources():
    # largest translation units first so the parallel build's critical path is short
    srcs = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp"))
    return sorted(srcs, key=lambda p: (-p.stat().st_size * (3 if "_inst_" in p.name else 1), p.name))


FLAGS_FILE = OUT_DIR / "build_flags.txt"


def _flag_line() -> str:
    return " ".join([NVCC, *ARCH, *FLAGS])


def _needs_build() -> bool:
    if not LIB.exists():
        return True
    # a library built with other flags (e.g. an SR_NVCC_EXTRA measurement knob) is rebuilt
    if not FLAGS_FILE.exists() or FLAGS_FILE.read_text().strip() != _flag_line():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + list(INCLUDE.glob("*.h"))
    return any(p.stat().st_mtime > t for p in deps if p.is_file())


def _compile(src: Path, verbose: bool) -> Path:
    obj = OUT_DIR / (src.stem + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr.strip():
        print(r.stderr, flush=True)
    return obj


def build(force: bool = False, verbose: bool = False) -> Path:
    subprocess.run([sys.executable, str(CSRC / "gen_dft.py"), str(CSRC / "dft_gen.cuh")], check=True)
    if not force and not _needs_build():
        return LIB
    OUT_DIR.mkdir(exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    FLAGS_FILE.write_text(_flag_line() + "\n")
    return LIB


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(p)

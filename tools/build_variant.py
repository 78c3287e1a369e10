#!/usr/bin/env python3
"""Build an A/B variant of the library: recompile the named csrc files with extra nvcc flags and
link them with the default build's other objects into _native/variants/lib<NAME>.so (load it with
SR_LIB_PATH).  python tools/build_variant.py NAME "-DSPREAD_G=2 ..." nufft.cu [more.cu]"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2305_06482_b200 import build as B  # noqa: E402


def main():
    name, extra, files = sys.argv[1], sys.argv[2].split(), sys.argv[3:]
    B.build()
    vdir = B.OUT_DIR / "variants"
    vdir.mkdir(exist_ok=True)
    objs = {p.stem: p for p in B.OUT_DIR.glob("*.o")}
    for f in files:
        src = B.CSRC / f
        obj = vdir / f"{name}_{src.stem}.o"
        subprocess.run([B.NVCC, *B.ARCH, *B.FLAGS, *extra, "-c", str(src), "-o", str(obj)], check=True)
        objs[src.stem] = obj
    out = vdir / f"lib{name}.so"
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", str(out), *map(str, objs.values())], check=True)
    print(out)


if __name__ == "__main__":
    main()

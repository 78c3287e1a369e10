#!/usr/bin/env python3
"""Code generator for the register-resident small DFTs used by every FFT kernel.

Emits ``dft_gen.cuh``: one ``__device__ __forceinline__`` function per
(size, direction) that transforms ``float2 v[N]`` in place, natural order in
and natural order out.  Sizes with two coprime factors use the prime-factor
(Good-Thomas) algorithm -- the index maps are free register renaming, and there
are no inter-stage twiddles (20 = 4 x 5: 272 -> ~224 FP instructions); prime
powers are unrolled four-step (Cooley-Tukey) factorizations whose inner
twiddles are literal constants computed here in float64 and rounded once to
float32, so no sin/cos is evaluated on the device for the in-register stages.

Convention (matches numpy.fft, which the reference uses at
/root/reference/pkg/src/sketchrecon/linops.py:304-309):
    forward  X[k] = sum_n x[n] exp(-2 pi i n k / N)
    inverse  x[n] = sum_k X[k] exp(+2 pi i n k / N)     (unnormalised)
"""

from __future__ import annotations

import math
import sys
from pathlib import Path

SIZES = (1, 2, 3, 4, 5, 6, 8, 9, 10, 12, 15, 16, 18, 20, 24, 25, 30, 32)


def _fmt(v: float) -> str:
    f = float(v)
    if f == 0.0:
        return "0.0f"
    return f"{f:.9e}f"


class _Emitter:
    def __init__(self):
        self.lines: list[str] = []
        self.n = 0

    def tmp(self, expr: str) -> str:
        name = f"t{self.n}"
        self.n += 1
        self.lines.append(f"  const float2 {name} = {expr};")
        return name

    # complex helpers ------------------------------------------------------
    def add(self, a, b):
        return self.tmp(f"make_float2({a}.x + {b}.x, {a}.y + {b}.y)")

    def sub(self, a, b):
        return self.tmp(f"make_float2({a}.x - {b}.x, {a}.y - {b}.y)")

    def muli(self, a, sgn):
        # multiply by sgn * i
        if sgn > 0:
            return self.tmp(f"make_float2(-{a}.y, {a}.x)")
        return self.tmp(f"make_float2({a}.y, -{a}.x)")

    def scale(self, a, c):
        return self.tmp(f"make_float2({_fmt(c)} * {a}.x, {_fmt(c)} * {a}.y)")

    def twiddle(self, a, num: int, den: int, sign: int):
        """a * exp(sign * 2 pi i num / den), with exact special angles."""
        num %= den
        if num == 0:
            return a
        g = math.gcd(num, den)
        num, den = num // g, den // g
        if den == 2:
            return self.tmp(f"make_float2(-{a}.x, -{a}.y)")
        if den == 4:
            # exp(sign*i*pi/2 * num) : num==1 -> sign*i ; num==3 -> -sign*i
            return self.muli(a, sign if num == 1 else -sign)
        ang = sign * 2.0 * math.pi * num / den
        c, s = math.cos(ang), math.sin(ang)
        if den == 8:
            r = math.sqrt(0.5)
            # (x + iy)(c + is) with |c| = |s| = r
            cs = 1 if c > 0 else -1
            ss = 1 if s > 0 else -1
            # real = r*(cs*x - ss*y), imag = r*(cs*y + ss*x)
            re = f"({'' if cs > 0 else '-'}{a}.x {'-' if ss > 0 else '+'} {a}.y)"
            im = f"({'' if cs > 0 else '-'}{a}.y {'+' if ss > 0 else '-'} {a}.x)"
            return self.tmp(f"make_float2({_fmt(r)} * {re}, {_fmt(r)} * {im})")
        return self.tmp(
            f"make_float2(fmaf({_fmt(c)}, {a}.x, {_fmt(-s)} * {a}.y), "
            f"fmaf({_fmt(c)}, {a}.y, {_fmt(s)} * {a}.x))"
        )

    # DFT kernels ------------------------------------------------------------
    def dft(self, xs: list[str], sign: int) -> list[str]:
        n = len(xs)
        if n == 1:
            return list(xs)
        if n == 2:
            return [self.add(xs[0], xs[1]), self.sub(xs[0], xs[1])]
        if n == 3:
            a0, a1, a2 = xs
            s = self.add(a1, a2)
            d = self.sub(a1, a2)
            y0 = self.add(a0, s)
            m = self.tmp(f"make_float2(fmaf(-0.5f, {s}.x, {a0}.x), fmaf(-0.5f, {s}.y, {a0}.y))")
            r = self.scale(d, math.sqrt(3.0) / 2.0)
            ir = self.muli(r, sign)
            return [y0, self.add(m, ir), self.sub(m, ir)]
        if n == 4:
            a0, a1, a2, a3 = xs
            s02 = self.add(a0, a2)
            d02 = self.sub(a0, a2)
            s13 = self.add(a1, a3)
            d13 = self.sub(a1, a3)
            w = self.muli(d13, sign)
            return [self.add(s02, s13), self.add(d02, w), self.sub(s02, s13), self.sub(d02, w)]
        if n == 5:
            a0, a1, a2, a3, a4 = xs
            c1, c2 = math.cos(2 * math.pi / 5), math.cos(4 * math.pi / 5)
            s1, s2 = math.sin(2 * math.pi / 5), math.sin(4 * math.pi / 5)
            p1 = self.add(a1, a4)
            m1 = self.sub(a1, a4)
            p2 = self.add(a2, a3)
            m2 = self.sub(a2, a3)
            y0 = self.tmp(f"make_float2({a0}.x + {p1}.x + {p2}.x, {a0}.y + {p1}.y + {p2}.y)")
            r1 = self.tmp(
                f"make_float2(fmaf({_fmt(c1)}, {p1}.x, fmaf({_fmt(c2)}, {p2}.x, {a0}.x)), "
                f"fmaf({_fmt(c1)}, {p1}.y, fmaf({_fmt(c2)}, {p2}.y, {a0}.y)))"
            )
            r2 = self.tmp(
                f"make_float2(fmaf({_fmt(c2)}, {p1}.x, fmaf({_fmt(c1)}, {p2}.x, {a0}.x)), "
                f"fmaf({_fmt(c2)}, {p1}.y, fmaf({_fmt(c1)}, {p2}.y, {a0}.y)))"
            )
            q1 = self.tmp(
                f"make_float2(fmaf({_fmt(s1)}, {m1}.x, {_fmt(s2)} * {m2}.x), "
                f"fmaf({_fmt(s1)}, {m1}.y, {_fmt(s2)} * {m2}.y))"
            )
            q2 = self.tmp(
                f"make_float2(fmaf({_fmt(s2)}, {m1}.x, {_fmt(-s1)} * {m2}.x), "
                f"fmaf({_fmt(s2)}, {m1}.y, {_fmt(-s1)} * {m2}.y))"
            )
            iq1 = self.muli(q1, sign)
            iq2 = self.muli(q2, sign)
            return [y0, self.add(r1, iq1), self.add(r2, iq2), self.sub(r2, iq2), self.sub(r1, iq1)]
        a, b = _coprime_split(n)
        if a > 1:
            # prime-factor (Good-Thomas) algorithm, gcd(a, b) = 1: input x[(b n1 + a n2) mod n],
            # output X[(k1 b (b^-1 mod a) + k2 a (a^-1 mod b)) mod n]; no twiddle multiplications
            inner = [self.dft([xs[(b * n1 + a * n2) % n] for n2 in range(b)], sign) for n1 in range(a)]
            ea, eb = b * pow(b, -1, a), a * pow(a, -1, b)
            out = [None] * n
            for k2 in range(b):
                col = self.dft([inner[n1][k2] for n1 in range(a)], sign)
                for k1 in range(a):
                    out[(k1 * ea + k2 * eb) % n] = col[k1]
            return out
        # composite: n = a * b, x[a_i + a*b_i]
        a = _pick_factor(n)
        b = n // a
        # inner DFTs of length b over stride-a subsequences
        inner = []
        for ai in range(a):
            sub = [xs[ai + a * bi] for bi in range(b)]
            inner.append(self.dft(sub, sign))
        # twiddles W_n^{ai * kb}
        for ai in range(a):
            for kb in range(b):
                inner[ai][kb] = self.twiddle(inner[ai][kb], ai * kb, n, sign)
        out = [None] * n
        for kb in range(b):
            col = self.dft([inner[ai][kb] for ai in range(a)], sign)
            for ka in range(a):
                out[kb + b * ka] = col[ka]
        return out


def _coprime_split(n: int) -> tuple[int, int]:
    """n = a * b with gcd(a, b) = 1 and a a prime power (the largest one), or (1, n)."""
    pp, m, f = [], n, 2
    while m > 1:
        if m % f == 0:
            q = 1
            while m % f == 0:
                m //= f
                q *= f
            pp.append(q)
        f += 1
    if len(pp) < 2:
        return 1, n
    a = max(pp)
    return a, n // a


def _pick_factor(n: int) -> int:
    for f in (4, 5, 3, 2):
        if n % f == 0 and n != f:
            return f
    raise ValueError(f"cannot factor {n}")


def gen_function(n: int, inverse: bool) -> str:
    e = _Emitter()
    sign = 1 if inverse else -1
    xs = []
    for i in range(n):
        xs.append(f"v{i}")
    e.lines.append("  " + " ".join(f"const float2 v{i} = v[{i}];" for i in range(n)))
    outs = e.dft(xs, sign)
    body = "\n".join(e.lines)
    stores = "\n".join(f"  v[{i}] = {o};" for i, o in enumerate(outs))
    name = f"dft{n}_{'inv' if inverse else 'fwd'}"
    return (
        f"__device__ __forceinline__ void {name}(float2* v) {{\n"
        f"{body}\n{stores}\n}}\n"
    )


def generate() -> str:
    parts = [
        "// AUTO-GENERATED by gen_dft.py -- do not edit.\n"
        "// In-register DFTs, natural order in/out, literal twiddles (float64 -> float32).\n"
        "#pragma once\n#include <cuda_runtime.h>\n",
    ]
    for n in SIZES:
        parts.append(gen_function(n, False))
        parts.append(gen_function(n, True))
    # compile-time dispatch
    parts.append("template <int N, bool INV> struct RegDFT;\n")
    for n in SIZES:
        parts.append(
            f"template <> struct RegDFT<{n}, false> {{ __device__ __forceinline__ static void run(float2* v) {{ dft{n}_fwd(v); }} }};\n"
            f"template <> struct RegDFT<{n}, true> {{ __device__ __forceinline__ static void run(float2* v) {{ dft{n}_inv(v); }} }};\n"
        )
    return "\n".join(parts)


def fft_sizes() -> list[tuple[int, int, int]]:
    """(N, P, Q) of the SR_FFT_SIZES table in fft2step.cuh (single source of truth)."""
    import re
    text = Path(__file__).with_name("fft2step.cuh").read_text()
    lines = text[text.index("#define SR_FFT_SIZES(X)"):].splitlines()
    n = next(i for i, ln in enumerate(lines) if not ln.rstrip().endswith("\\"))
    body = "\n".join(lines[: n + 1])
    return [tuple(int(v) for v in m) for m in re.findall(r"X\((\d+),\s*(\d+),\s*(\d+)\)", body)]


def generate_twiddles() -> str:
    """Inter-stage twiddle tables of the two-level FFT, float64 -> float32 once:
    t1[k2*P + p] = W_N^{p k2},  t2[m1*Q + k2] = W_N^{m1 k2},  W_N = exp(-2 pi i / N)."""
    parts = [
        "// AUTO-GENERATED by gen_dft.py -- do not edit.\n"
        "// Two-level FFT twiddle tables (see fft2step.cuh), float64 -> float32.\n"
        "#pragma once\n#include <cuda_runtime.h>\n",
        "template <int P, int Q> struct TwTab;\n",
    ]
    for n, p, q in fft_sizes():
        if p == 1:
            continue

        def w(k):
            a = -2.0 * math.pi * (k % n) / n
            return f"{{{_fmt(math.cos(a))}, {_fmt(math.sin(a))}}}"

        t1 = ", ".join(w(pp * k2) for k2 in range(q) for pp in range(p))
        t2 = ", ".join(w(m1 * k2) for m1 in range(p) for k2 in range(q))
        parts.append(f"static __device__ const float2 sr_tw1_{n}[{n}] = {{{t1}}};\n"
                     f"static __device__ const float2 sr_tw2_{n}[{n}] = {{{t2}}};\n"
                     f"template <> struct TwTab<{p}, {q}> {{\n"
                     f"  __device__ __forceinline__ static const float2* t1() {{ return sr_tw1_{n}; }}\n"
                     f"  __device__ __forceinline__ static const float2* t2() {{ return sr_tw2_{n}; }}\n}};\n")
    return "\n".join(parts)


CART_BUCKETS = 6


def generate_buckets() -> tuple[str, dict[str, str]]:
    """Split SR_FFT_SIZES into CART_BUCKETS round-robin lists (largest sizes first) so the
    Cartesian kernels of each list compile in their own translation unit."""
    sizes = sorted(fft_sizes(), key=lambda t: -t[0])
    buckets = [[] for _ in range(CART_BUCKETS)]
    for i, t in enumerate(sizes):
        buckets[i % CART_BUCKETS].append(t)
    lines = ["// AUTO-GENERATED by gen_dft.py -- do not edit.",
             "// Size buckets of the Cartesian kernel instantiations (one translation unit each).",
             "#pragma once", ""]
    lines.append("#define SR_CART_BUCKETS(X) " + " ".join(f"X({k})" for k in range(CART_BUCKETS)))
    for k, b in enumerate(buckets):
        lines.append(f"#define SR_FFT_SIZES_B{k}(X) " + " ".join(f"X({n}, {p}, {q})" for n, p, q in sorted(b)))
    wrappers = {}
    for k in range(CART_BUCKETS):
        wrappers[f"fft_axis_inst_{k}.cu"] = (
            "// AUTO-GENERATED by gen_dft.py -- do not edit.\n"
            f"// NUFFT per-axis FFT kernels, size bucket {k} (see fft_axis_inst.cuh).\n"
            '#include "fft_buckets_gen.cuh"\n'
            f"#define SR_BUCKET_ID {k}\n"
            f"#define SR_BUCKET_SIZES SR_FFT_SIZES_B{k}\n"
            '#include "fft_axis_inst.cuh"\n')
        wrappers[f"cart_inst_{k}.cu"] = (
            "// AUTO-GENERATED by gen_dft.py -- do not edit.\n"
            f"// Cartesian kernels, size bucket {k} (see cart_inst.cuh).\n"
            '#include "fft_buckets_gen.cuh"\n'
            f"#define SR_BUCKET_ID {k}\n"
            f"#define SR_BUCKET_SIZES SR_FFT_SIZES_B{k}\n"
            '#include "cart_inst.cuh"\n')
    return "\n".join(lines) + "\n", wrappers


def _write(out: Path, text: str) -> None:
    if not out.exists() or out.read_text() != text:
        out.write_text(text)


def main(argv):
    out = Path(argv[1]) if len(argv) > 1 else Path(__file__).with_name("dft_gen.cuh")
    _write(out, generate())
    _write(out.with_name("tw_gen.cuh"), generate_twiddles())
    hdr, wrappers = generate_buckets()
    _write(out.with_name("fft_buckets_gen.cuh"), hdr)
    for name, text in wrappers.items():
        _write(out.with_name(name), text)


if __name__ == "__main__":
    main(sys.argv)

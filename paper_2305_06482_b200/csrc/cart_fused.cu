// K1 (fused): the whole Cartesian sketched normal operator in ONE persistent launch.
//
//   out_b = e( sum_j conj(c_bj) . F^H M'_b F (c_bj . (x_b - a_b)) )
//
// Reference: SenseOperator._forward/_adjoint (forward_model.py:168-180) over
// _CartesianMaskKernel (linops.py:344-364); the solvers call it as
// adjoint(forward(.)) (coil_sketch.py:126,133,197; solvers.py:175,248).
//
// Design (B200): the three passes of cart.cu (row FFT, column FFT-mask-IFFT,
// row IFFT + conjugate coil sum) become three kinds of work items of one
// persistent kernel, pulled in a fixed ticket order that staggers slices:
//     round r = { A items of slice r, B items of slice r-1, C items of slice r-2 }
//   A(s, row tile, coil)  u = c_j (x - a) on 16 rows, row FFT      -> ws
//   B(s, col tile, coil)  16 columns: FFT, mask/D, IFFT           (ws in place)
//   C(s, row tile)        16 rows: for every coil, row IFFT, acc += conj(c_j) (.),
//                         then the epilogue (FISTA / CG combination)
// Only ~3 slices are in flight, so the coil workspace (9.8 MB per 320^2 slice
// at C_hat = 12) and the re-read maps stay in the 126 MB L2: HBM sees ~the
// compulsory bytes (maps + x + out) instead of 5 workspace sweeps.  Measured
// on this part: L2-resident reads ~18.5 TB/s vs HBM ~7 TB/s vs DSMEM <= 4.8
// TB/s (tools/membw_probe.cu), which is why the exchange goes through L2 and
// not through cluster shared memory.
//
// Dependencies are per (slice, coil) counters with release/acquire at gpu
// scope; an item only waits on items with smaller tickets, which are already
// owned by resident CTAs, so the schedule cannot deadlock.  Workspace reads
// use ld.global.cg (L1 is not coherent across CTAs); counters are zeroed by a
// memset in the same stream before each launch.
#include "fft2step.cuh"

namespace {

constexpr int MAX_SLOTS = 8;  // workspace ring capacity (runtime `slots` <= MAX_SLOTS): slice s
                              // lives in slot s % slots, stays in L2, and its dirty lines are
                              // overwritten before they would be evicted

// optional wait statistics (sr_fused_stats): spin iterations per wait site, clock64 per item type
__device__ unsigned long long* g_fused_stats = nullptr;

__device__ __forceinline__ void spin_until(const int* c, int target, int site) {
  unsigned long long n = 0;
  int v;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
    if (v >= target) break;
    ++n;
    __nanosleep(64);
  }
  if (g_fused_stats && n) atomicAdd(g_fused_stats + site, n);
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// L2 residency hints: the workspace ring is kept (evict_last); maps are read
// twice (A, then C) and dropped after the second read (evict_first).
__device__ __forceinline__ uint64_t pol_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float2 ld_ws(const float2* ptr, uint64_t pol) {
  float2 v;
  asm volatile("ld.global.cg.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;"
               : "=f"(v.x), "=f"(v.y) : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_ws(float2* ptr, float2 v, uint64_t pol) {
  asm volatile("st.global.cg.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;"
               :: "l"(ptr), "f"(v.x), "f"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ float2 ld_ro_hint(const float2* ptr, uint64_t pol) {
  float2 v;
  asm("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(ptr), "l"(pol));
  return v;
}

template <int P, int QY, int QX, int TILE>
struct FusedCfg {
  using SX = RowShape<P, QX>;   // row tiles (A, C): 16-byte aligned groups
  using SY = FftShape<P, QY>;   // column tiles (B): odd stride over columns
  static constexpr int NX = P * QX, NY = P * QY;
  static constexpr int T = TILE * P;
  static constexpr int VSX = SX::VS;
  static constexpr int VSPY = SY::VS0 | 1;
  static constexpr int XS = NX + ((((P % 16) - (NX % 16)) % 16 + 16) % 16);  // staged x rows (A)
  static constexpr int ROWT = TILE * VSX;
  static constexpr int COLT = TILE * VSPY;
  // buffer region: A = [row tile | x rows], B = [column tile], C = [row tile | row tile]
  static constexpr int A_NEED = ROWT + TILE * XS, C_NEED = 2 * ROWT;
  static constexpr int BUF0 = A_NEED > C_NEED ? A_NEED : C_NEED;
  static constexpr int BUF1 = BUF0 > COLT ? BUF0 : COLT;
  static constexpr int BUF = BUF1 + (BUF1 & 1);
  static constexpr int OFF_TX1 = 0, OFF_TX2 = NX, OFF_TY1 = 2 * NX, OFF_TY2 = 2 * NX + NY;
  static constexpr int OFF_BUF = 2 * NX + 2 * NY + ((2 * NX + 2 * NY) & 1);
  static constexpr size_t SMEM = sizeof(float2) * (OFF_BUF + BUF) + 16;  // + round table (ints)
};

struct FusedArgs {
  const float2* x;
  const float2* anchor;
  const float2* maps;
  long long map_bstride;
  const uint8_t* maskT;
  long long mask_bstride;
  float2* out;
  float2* ws;     // ring of `slots` slice slots of (C, ny, nx), then the partial-sum ring
  int* sync;      // [0] ticket, [1..] cntA[S*C], cntB[S*C], cntC[S], cntT[S*nrt]
  int batch, ncoils;
  int lagB, lagC, slots;  // schedule: round r = {A(r), B(r - lagB), C(r - lagC)}
  float oscale;           // 1/D of the unitary FFT pair, applied once per pixel
  const float4* coef;
  const float2* u;
  const float2* d;
};

constexpr int COILS_PER_A = 4;  // coils per A item (x staged once, maps prefetched one coil ahead)
constexpr int COILS_PER_C = 3;  // coils per C item (partial coil sums, last arriver combines)

// ---------------------------------------------------------------- A items
// rows [rt*TILE, +TILE) of coils [j0, j1): u = c_j (x - a), row FFT -> workspace ring;
// cntA[s, j] is released after every coil so B items of that coil can start early.
template <int P, int QY, int QX, int TILE>
__device__ void item_rowfwd(const FusedArgs& a, int s, int rt, int j0, int j1, float2* sm, int* cntA) {
  using F = FusedCfg<P, QY, QX, TILE>;
  using SX = typename F::SX;
  constexpr int NX = F::NX, NY = F::NY, T = F::T, XS = F::XS;
  const int tid = threadIdx.x;
  const int lr = tid / P, p = tid - lr * P;
  const int row = rt * TILE + lr;
  const bool valid = row < NY;
  const long long D = (long long)NX * NY;
  const float2* tx1 = sm + F::OFF_TX1;
  float2* buf = sm + F::OFF_BUF;
  float2* xs = buf + F::ROWT;
  const int nrows = min(TILE, NY - rt * TILE);
  const int nvalid = nrows * NX;
  {
    const float2* xb = a.x + (long long)s * D + (long long)rt * TILE * NX;
    const float2* ab = a.anchor ? a.anchor + (long long)s * D + (long long)rt * TILE * NX : xb;
    for (int e = tid; e < TILE * NX; e += T) {
      const int l3 = e / NX, pos = e - l3 * NX;
      float2 v = make_float2(0.f, 0.f);
      if (e < nvalid) {
        v = __ldg(xb + e);
        if (a.anchor) v = csub(v, __ldg(ab + e));
      }
      xs[l3 * XS + pos] = v;
    }
  }
  const float2* mb = a.maps + s * a.map_bstride + (long long)row * NX + p;
  float2 mcur[QX];
#pragma unroll
  for (int q = 0; q < QX; ++q) mcur[q] = valid ? __ldg(mb + (long long)j0 * D + P * q) : make_float2(0.f, 0.f);
  __syncthreads();
  const float2* xr = xs + lr * XS + p;
  const uint64_t keep = pol_evict_last();
  for (int j = j0; j < j1; ++j) {
    float2 r[QX];
#pragma unroll
    for (int q = 0; q < QX; ++q) r[q] = cmul(mcur[q], xr[P * q]);
    if (j + 1 < j1 && valid) {
#pragma unroll
      for (int q = 0; q < QX; ++q) mcur[q] = __ldg(mb + (long long)(j + 1) * D + P * q);
    }
    fft_s1_fwd<P, QX>(r, p, tx1);
#pragma unroll
    for (int k2 = 0; k2 < QX; ++k2) buf[lr * F::VSX + SX::GS * k2 + p] = r[k2];
    __syncthreads();
    for (int it = tid; it < TILE * QX; it += T) {
      const int l2 = it / QX, k2 = it - l2 * QX;
      float2 g[P];
      float2* gp = buf + l2 * F::VSX + SX::GS * k2;
      lds_group<P, SX::VEC>(g, gp);
      fft_s2_fwd<P>(g);
      sts_group<P, SX::VEC>(gp, g);
    }
    __syncthreads();
    float2* wj = a.ws + ((long long)(s % a.slots) * a.ncoils + j) * D + (long long)rt * TILE * NX;
    for (int e = tid; e < nvalid; e += T) {
      const int l3 = e / NX, pos = e - l3 * NX;
      st_ws(wj + e, buf[l3 * F::VSX + SX::pad(pos)], keep);
    }
    __syncthreads();
    if (tid == 0) red_release_add(cntA + s * a.ncoils + j, 1);
  }
}

// ---------------------------------------------------------------- B items
template <int P, int QY, int QX, int TILE>
__device__ void item_colpass(const FusedArgs& a, int s, int ct, int j, float2* sm) {
  using F = FusedCfg<P, QY, QX, TILE>;
  using SY = typename F::SY;
  constexpr int NX = F::NX, NY = F::NY, T = F::T;
  const int tid = threadIdx.x;
  const int c = tid % TILE, p = tid / TILE;
  const int c0 = ct * TILE;
  const int ncols = min(TILE, NX - c0);
  const bool cvalid = c < ncols;
  const long long D = (long long)NX * NY;
  const float2* ty1 = sm + F::OFF_TY1;
  const float2* ty2 = sm + F::OFF_TY2;
  float2* buf = sm + F::OFF_BUF;
  float2* img = a.ws + ((long long)(s % a.slots) * a.ncoils + j) * D;
  const uint64_t keep = pol_evict_last();
  float2 r[QY];
#pragma unroll
  for (int q = 0; q < QY; ++q)
    r[q] = cvalid ? ld_ws(img + (long long)(p + P * q) * NX + c0 + c, keep) : make_float2(0.f, 0.f);
  fft_s1_fwd<P, QY>(r, p, ty1);
#pragma unroll
  for (int k2 = 0; k2 < QY; ++k2) buf[c * F::VSPY + SY::GS * k2 + p] = r[k2];
  __syncthreads();
  const uint8_t* mcol = a.maskT + s * a.mask_bstride;
  for (int it = tid; it < TILE * QY; it += T) {
    const int cc = it % TILE, k2 = it / TILE;
    if (cc >= ncols) continue;
    float2 g[P];
    float2* gp = buf + cc * F::VSPY + SY::GS * k2;
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) g[k1] = gp[k1];
    fft_s2_fwd<P>(g);
    const uint8_t* mk = mcol + (long long)(c0 + cc) * NY + P * k2;
    if ((P % 4) == 0) {
#pragma unroll
      for (int w4 = 0; w4 < P / 4; ++w4) {
        const uint32_t m4 = __ldg(reinterpret_cast<const uint32_t*>(mk) + w4);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          g[4 * w4 + i] = ((m4 >> (8 * i)) & 0xffu) ? g[4 * w4 + i] : make_float2(0.f, 0.f);
      }
    } else {
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) g[k1] = mk[k1] ? g[k1] : make_float2(0.f, 0.f);
    }
    fft_s2_inv<P, QY>(g, k2, ty2);
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) gp[k1] = g[k1];
  }
  __syncthreads();
#pragma unroll
  for (int k2 = 0; k2 < QY; ++k2) r[k2] = buf[c * F::VSPY + SY::GS * k2 + p];
  fft_s1_inv<QY>(r);
  if (cvalid) {
#pragma unroll
    for (int q = 0; q < QY; ++q) st_ws(img + (long long)(p + P * q) * NX + c0 + c, r[q], keep);
  }
}

// ---------------------------------------------------------------- C items
__device__ __forceinline__ int atom_add_acqrel(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// C(s, rt, g): coils [g*CG, g*CG + CG) of TILE rows; workspace tiles double-buffered with
// cp.async (L2 -> smem), maps prefetched before the FFT work; partial sums go to the
// partial ring, the last group to finish a row tile sums the G partials in a fixed order
// (deterministic) and writes the epilogue.  Returns true when this item finalised the tile.
template <int P, int QY, int QX, int TILE>
__device__ bool item_rowinv(const FusedArgs& a, int s, int rt, int g, int G, int CG, int* cntB,
                            int* cntT, int ncoltiles, float2* sm, int* s_flag) {
  using F = FusedCfg<P, QY, QX, TILE>;
  using SX = typename F::SX;
  constexpr int NX = F::NX, NY = F::NY, T = F::T;
  const int tid = threadIdx.x;
  const int lr = tid / P, p = tid - lr * P;
  const int row = rt * TILE + lr;
  const bool valid = row < NY;
  const long long D = (long long)NX * NY;
  const float2* tx2 = sm + F::OFF_TX2;
  float2* bufs = sm + F::OFF_BUF;
  const int nrows = min(TILE, NY - rt * TILE);
  const int nvalid = nrows * NX;
  const int slot = s % a.slots;
  float2 acc[QX];
#pragma unroll
  for (int q = 0; q < QX; ++q) acc[q] = make_float2(0.f, 0.f);
  const int j0 = g * CG, j1 = min(a.ncoils, j0 + CG);
  auto wait_coil = [&](int j) {
    if (tid == 0) spin_until(cntB + s * a.ncoils + j, ncoltiles, 2);
    __syncthreads();
  };
  auto issue_tile = [&](int j) {
    const float2* wj = a.ws + ((long long)slot * a.ncoils + j) * D + (long long)rt * TILE * NX;
    float2* dst = bufs + ((j - j0) & 1) * F::ROWT;
    for (int e = 2 * tid; e < nvalid; e += 2 * T) {
      const int l3 = e / NX, pos = e - l3 * NX;
      cp_async16(dst + l3 * F::VSX + SX::pad(pos), wj + e);
    }
    cp_async_commit();
  };
  wait_coil(j0);
  issue_tile(j0);
  for (int j = j0; j < j1; ++j) {
    if (j + 1 < j1) {
      wait_coil(j + 1);
      issue_tile(j + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    float2* buf = bufs + ((j - j0) & 1) * F::ROWT;
    float2 mreg[QX];
    {
      const float2* mr = a.maps + s * a.map_bstride + (long long)j * D + (long long)row * NX + p;
      const uint64_t drop = pol_evict_first();
#pragma unroll
      for (int q = 0; q < QX; ++q) mreg[q] = valid ? ld_ro_hint(mr + P * q, drop) : make_float2(0.f, 0.f);
    }
    for (int it = tid; it < TILE * QX; it += T) {
      const int l2 = it / QX, k2 = it - l2 * QX;
      float2 gg[P];
      float2* gp = buf + l2 * F::VSX + SX::GS * k2;
      lds_group<P, SX::VEC>(gg, gp);
      fft_s2_inv<P, QX>(gg, k2, tx2);
      sts_group<P, SX::VEC>(gp, gg);
    }
    __syncthreads();
    float2 r[QX];
#pragma unroll
    for (int k2 = 0; k2 < QX; ++k2) r[k2] = buf[lr * F::VSX + SX::GS * k2 + p];
    fft_s1_inv<QX>(r);
#pragma unroll
    for (int q = 0; q < QX; ++q) cfma_conj(acc[q], mreg[q], r[q]);
    __syncthreads();
  }
  const long long roff = (long long)row * NX + p;
  const uint64_t keep = pol_evict_last();
  if (G > 1) {
    float2* part = a.ws + (long long)a.slots * a.ncoils * D + ((long long)slot * G + g) * D;
    if (valid) {
#pragma unroll
      for (int q = 0; q < QX; ++q) st_ws(part + roff + P * q, acc[q], keep);
    }
    __syncthreads();
    if (tid == 0) *s_flag = (atom_add_acqrel(cntT + s * ((NY + TILE - 1) / TILE) + rt, 1) == G - 1);
    __syncthreads();
    if (!*s_flag) return false;
    const float2* pb = a.ws + (long long)a.slots * a.ncoils * D + (long long)slot * G * D;
#pragma unroll
    for (int q = 0; q < QX; ++q) acc[q] = make_float2(0.f, 0.f);
    if (valid) {
      const uint64_t drop = pol_evict_first();
      for (int gg = 0; gg < G; ++gg) {
#pragma unroll
        for (int q = 0; q < QX; ++q) acc[q] = cadd(acc[q], ld_ws(pb + (long long)gg * D + roff + P * q, drop));
      }
    }
  }
  if (!valid) return true;
#pragma unroll
  for (int q = 0; q < QX; ++q) acc[q] = cscale(acc[q], a.oscale);
  const long long off = (long long)s * D + roff;
  if (a.coef == nullptr) {
#pragma unroll
    for (int q = 0; q < QX; ++q) a.out[off + P * q] = acc[q];
  } else {
    const float4 cf = a.coef[s];
#pragma unroll
    for (int q = 0; q < QX; ++q) {
      float2 v = cscale(acc[q], cf.x);
      if (a.u) { const float2 uu = a.u[off + P * q]; v.x = fmaf(cf.y, uu.x, v.x); v.y = fmaf(cf.y, uu.y, v.y); }
      if (a.d) { const float2 dd = a.d[off + P * q]; v.x = fmaf(cf.z, dd.x, v.x); v.y = fmaf(cf.z, dd.y, v.y); }
      a.out[off + P * q] = v;
    }
  }
  return true;
}

// ---------------------------------------------------------------- scheduler

template <int P, int QY, int QX, int TILE>
__global__ void __launch_bounds__(FusedCfg<P, QY, QX, TILE>::T, (TILE >= 16 ? 1 : 3))
k_cart_normal_fused(FusedArgs a) {
  using F = FusedCfg<P, QY, QX, TILE>;
  constexpr int NX = F::NX, NY = F::NY, T = F::T;
  extern __shared__ __align__(16) float2 sm[];
  __shared__ int s_ticket, s_flag;
  const int tid = threadIdx.x;
  const int S = a.batch, C = a.ncoils;
  const int nrt = (NY + TILE - 1) / TILE, nct = (NX + TILE - 1) / TILE;
  const int G = (C + COILS_PER_C - 1) / COILS_PER_C;
  const int GA = (C + COILS_PER_A - 1) / COILS_PER_A;
  const int nA = nrt * GA, nB = nct * C, nC = nrt * G;
  const int LB = a.lagB, LC = a.lagC;
  const int R = S + LC;  // rounds
  int* rstart = reinterpret_cast<int*>(sm + F::OFF_BUF + F::BUF);  // R + 1 round offsets
  init_tw_s1<P, QX>(sm + F::OFF_TX1, tid, T);
  init_tw_s2<P, QX>(sm + F::OFF_TX2, tid, T);
  init_tw_s1<P, QY>(sm + F::OFF_TY1, tid, T);
  init_tw_s2<P, QY>(sm + F::OFF_TY2, tid, T);
  if (tid == 0) {
    int acc = 0;
    for (int r = 0; r < R; ++r) {
      rstart[r] = acc;
      acc += (r < S ? nA : 0) + (r >= LB && r < S + LB ? nB : 0) + (r >= LC ? nC : 0);
    }
    rstart[R] = acc;
  }
  __syncthreads();
  const int total = rstart[R];
  int* cntA = a.sync + 1;
  int* cntB = cntA + S * C;
  int* cntC = cntB + S * C;     // finalised row tiles per slice
  int* cntT = cntC + S;         // finished coil groups per (slice, row tile)
  for (;;) {
    if (tid == 0) s_ticket = atomicAdd(a.sync, 1);
    __syncthreads();
    const int t = s_ticket;
    __syncthreads();
    if (t >= total) break;
    // round = last r with rstart[r] <= t (binary search)
    int lo = 0, hi = R - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (rstart[mid] <= t) lo = mid; else hi = mid - 1;
    }
    const int r = lo;
    int it = t - rstart[r];
    const long long t_item0 = g_fused_stats ? clock64() : 0LL;
    if (r < S && it < nA) {
      const int s = r, rt = it % nrt, ga = it / nrt;
      if (s >= a.slots) {  // slot reuse: every row tile of slice s - slots is final
        if (tid == 0) {
          const int* c = cntC + (s - a.slots);
          spin_until(c, nrt, 0);
        }
        __syncthreads();
      }
      item_rowfwd<P, QY, QX, TILE>(a, s, rt, ga * COILS_PER_A, min(C, (ga + 1) * COILS_PER_A), sm, cntA);
      if (g_fused_stats && tid == 0) atomicAdd(g_fused_stats + 4, (unsigned long long)(clock64() - t_item0));
      continue;
    }
    if (r < S) it -= nA;
    if (r >= LB && r < S + LB && it < nB) {
      const int s = r - LB, ct = it % nct, j = it / nct;
      if (tid == 0) {
        const int* c = cntA + s * C + j;
        spin_until(c, nrt, 1);
      }
      __syncthreads();
      item_colpass<P, QY, QX, TILE>(a, s, ct, j, sm);
      __syncthreads();
      if (tid == 0) red_release_add(cntB + s * C + j, 1);
      if (g_fused_stats && tid == 0) atomicAdd(g_fused_stats + 5, (unsigned long long)(clock64() - t_item0));
      continue;
    }
    if (r >= LB && r < S + LB) it -= nB;
    {
      const int s = r - LC, rt = it % nrt, g = it / nrt;
      const bool fin = item_rowinv<P, QY, QX, TILE>(a, s, rt, g, G, COILS_PER_C, cntB, cntT, nct, sm, &s_flag);
      __syncthreads();
      if (fin && tid == 0) red_release_add(cntC + s, 1);
      if (g_fused_stats && tid == 0) atomicAdd(g_fused_stats + 6, (unsigned long long)(clock64() - t_item0));
    }
    __syncthreads();
  }
}

struct FusedConfig {
  int lagB = 1, lagC = 2, slots = 4, tile = 8;
};
FusedConfig g_cfg;

template <int P, int QY, int QX, int TILE>
int launch_fused(FusedArgs a, cudaStream_t st) {
  using F = FusedCfg<P, QY, QX, TILE>;
  static int per = 0, nsm = 0;
  const size_t smem = F::SMEM + sizeof(int) * (a.batch + a.lagC + 2);
  static size_t configured = 0;
  if (smem > configured) {
    if (cudaFuncSetAttribute(k_cart_normal_fused<P, QY, QX, TILE>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return SR_ECUDA;
    configured = smem;
    per = 0;
  }
  if (per == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cart_normal_fused<P, QY, QX, TILE>, F::T, smem);
    if (per < 1) return SR_ECUDA;
  }
  k_cart_normal_fused<P, QY, QX, TILE><<<nsm * per, F::T, smem, st>>>(a);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

}  // namespace

// (ny, nx) pairs with a fused instantiation: X(P, QY, QX)
#define SR_FUSED_SIZES(X)                                                                  \
  X(20, 16, 16) X(16, 16, 16) X(16, 16, 10) X(16, 10, 16) X(16, 10, 10) X(16, 8, 8)        \
  X(20, 10, 10) X(20, 16, 10) X(20, 10, 16) X(16, 4, 4) X(16, 8, 16) X(16, 16, 8)

int sr_fused_normal_supported(int ny, int nx) {
#define X(P, QY, QX) if (ny == P * QY && nx == P * QX) return 1;
  SR_FUSED_SIZES(X)
#undef X
  return 0;
}

static int fused_tile(int ny, int nx) {
  (void)ny; (void)nx;
  return g_cfg.tile;
}

long long sr_fused_sync_ints(int batch, int ncoils, int ny) {
  return 1 + 2LL * batch * ncoils + batch + (long long)batch * ((ny + 7) / 8);
}
// complex64 elements of workspace: coil ring + partial-sum ring
long long sr_fused_ws_elems(int batch, int ncoils, long long D) {
  const long long G = (ncoils + COILS_PER_C - 1) / COILS_PER_C;
  const long long slots = batch < g_cfg.slots ? batch : g_cfg.slots;
  return slots * ncoils * D + (G > 1 ? slots * G * D : 0);
}

extern "C" int sr_fused_stats(unsigned long long* dev_buf) {
  // dev_buf: 8 device counters [spin A-slot, spin B, spin C, -, cycles A, cycles B, cycles C, -] or NULL
  return cudaMemcpyToSymbol(g_fused_stats, &dev_buf, sizeof(dev_buf)) == cudaSuccess ? SR_OK : SR_ECUDA;
}

extern "C" int sr_fused_config(int lagB, int lagC, int slots, int tile) {
  if (lagB < 1 || lagC <= lagB || slots < lagC + 1 || slots > MAX_SLOTS || (tile != 8 && tile != 16))
    return SR_EINVAL;
  g_cfg.lagB = lagB; g_cfg.lagC = lagC; g_cfg.slots = slots; g_cfg.tile = tile;
  return SR_OK;
}

int sr_fused_normal(const float2* x, const float2* anchor, const float2* maps, long long map_bstride,
                    const uint8_t* maskT, long long mask_bstride, float2* out, float2* ws, int* sync,
                    int batch, int ncoils, int ny, int nx, const float4* coef, const float2* u,
                    const float2* d, cudaStream_t st) {
  const int slots = batch < g_cfg.slots ? batch : g_cfg.slots;
  FusedArgs a{x, anchor, maps, map_bstride, maskT, mask_bstride, out, ws, sync, batch, ncoils,
              g_cfg.lagB, g_cfg.lagC, slots < 1 ? 1 : slots, (float)(1.0 / ((double)ny * nx)), coef, u, d};
  // defaults: tile 8 (T = 8 P threads, 3 CTAs / SM)
  if (cudaMemsetAsync(sync, 0, sizeof(int) * sr_fused_sync_ints(batch, ncoils, ny), st) != cudaSuccess)
    return SR_ECUDA;
  const int tile = fused_tile(ny, nx);
#define X(P, QY, QX)                                                        \
  if (ny == P * QY && nx == P * QX)                                         \
    return tile == 8 ? launch_fused<P, QY, QX, 8>(a, st) : launch_fused<P, QY, QX, 16>(a, st);
  SR_FUSED_SIZES(X)
#undef X
  return SR_EUNSUPPORTED;
}

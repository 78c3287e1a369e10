// K1 (group schedule): the Cartesian sketched normal operator with the coil
// images exchanged through L2 inside small groups of co-resident CTAs.
//
//   out_b = e( sum_j conj(c_bj) . F^H M'_b F (c_bj . (x_b - a_b)) )
//
// Reference: SenseOperator._forward/_adjoint (forward_model.py:168-180) over
// _CartesianMaskKernel (linops.py:344-364), called as adjoint(forward(.)) by
// the solvers (coil_sketch.py:126,133,197; solvers.py:175,248).
//
// Design (B200).  The three-pass schedule of cart.cu streams every coil image
// through HBM twice (written after the row FFT, read + written by the column
// pass, read by the row IFFT: ~3.8 GB per config-1 apply against 0.73 GB of
// compulsory maps + x + out).  Here one persistent launch puts G CTAs (one per
// SM) on each coil image at a time:
//   CTA r of a group owns rows [r*R, r*R + R) and columns [r*CC, r*CC + CC).
//   A(u)  rows:    v = c_j (x - a) ; row FFT            -> scratch[u % 2]
//   B(u)  columns: column FFT, mask, column IFFT         (scratch in place)
//   C(u)  rows:    row IFFT ; acc += conj(c_j) (.)       (acc in shared memory)
// The scratch images of a group (2 x 0.8 MB at 320^2) stay in the 126 MB L2
// (evict_last stores), so HBM sees the maps once (the re-read in C hits L2),
// x and out.  Phases are ordered by two monotonic counters per group
// (gpu-scope release add / acquire spin); each CTA runs  B(u), A(u+1), C(u),
// so every wait is on work its peers issued one phase earlier:
//   wait A(u) < B(u) ; arrive B(u) ; A(u+1) ; arrive A(u+1) ; wait B(u) < C(u).
// Double buffering is enough: a CTA overwrites its rows of buffer u%2 in
// A(u+2) only after it has waited for B(u+1) <- everyone finished A(u+1) <-
// everyone finished C(u) (and B(u) before that).  Scratch is read with
// ld.global.cg / cp.async.cg (L1 is not coherent across SMs).
//
// Work split: the U = batch * ncoils (slice, coil) units are divided into
// contiguous ranges, one per group (balanced to one unit).  A group
// accumulates the coils of a slice in shared memory; a slice that lies wholly
// in one range is finished in place (epilogue -> out); a slice split between
// groups leaves one partial per group and the last CTA to arrive (per row
// band, counted atomically) sums the partials in group order, so the result is
// deterministic.
#include "fft2step.cuh"

namespace {

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ float2 ld_cg2(const float2* p) {
  float2 v;
  asm volatile("ld.global.cg.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_cg2(float2* p, float2 v) {
  asm volatile("st.global.cg.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void st_cg4(void* p, float4 v) {
  asm volatile("st.global.cg.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w) : "memory");
}

// L2 residency: the group scratch, x and the maps (read again in phase C) are kept
// (evict_last); the maps' second read and the results are streamed (evict_first)
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float2 ld_nc_hint(const float2* p, uint64_t pol) {
  float2 v;
  asm("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float2 ld_cg_hint(const float2* p, uint64_t pol) {
  float2 v;
  asm volatile("ld.global.cg.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_cg2_hint(float2* p, float2 v, uint64_t pol) {
  asm volatile("st.global.cg.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_cg4_hint(void* p, float4 v, uint64_t pol) {
  asm volatile("st.global.cg.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async16_hint(void* smem_dst, const void* gmem_src, uint64_t pol) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(d), "l"(gmem_src), "l"(pol)
               : "memory");
}

// the CTA's global writes precede the barrier; thread 0's gpu-scope fence + release-add is
// cumulative over them (the pattern of cooperative-groups grid sync), so only one warp pays
// for the fence and the others move on to the next phase
__device__ __forceinline__ void group_arrive(int* cnt) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    red_release_gpu(cnt, 1);
  }
}
__device__ __forceinline__ void group_wait(const int* cnt, int target) {
  if (threadIdx.x == 0) {
    while (ld_acquire_gpu(cnt) < target) __nanosleep(32);
    __threadfence();
  }
  __syncthreads();
}

template <int PY, int QY, int PX, int QX, int G>
struct GrpCfg {
  static constexpr int NY = PY * QY, NX = PX * QX;
  static constexpr int R = NY / G, CC = NX / G;
  static constexpr int T = R * PX;  // one thread per (row, p) of the row passes
  using SX = RowShape<PX, QX>;
  using SY = FftShape<PY, QY>;
  static constexpr int VSX = SX::VS;
  static constexpr int VSPY = SY::VS0 | 1;
  static constexpr int ACCS = NX + ((((PX % 16) - (NX % 16)) % 16 + 16) % 16);  // = PX (mod 16)
  static constexpr int ROWT = R * VSX, COLT = CC * VSPY;
  static constexpr int BUF0 = ROWT > COLT ? ROWT : COLT;
  static constexpr int BUF = BUF0 + (BUF0 & 1);
  static constexpr int OFF_TX1 = 0, OFF_TX2 = NX, OFF_TY1 = 2 * NX, OFF_TY2 = 2 * NX + NY;
  static constexpr int OFF_ACC0 = 2 * NX + 2 * NY;
  static constexpr int OFF_ACC = OFF_ACC0 + (OFF_ACC0 & 1);
  static constexpr int OFF_BUF0 = OFF_ACC + R * ACCS;
  static constexpr int OFF_BUF = OFF_BUF0 + (OFF_BUF0 & 1);
  static constexpr size_t SMEM = sizeof(float2) * (OFF_BUF + BUF);
  // CTAs per SM: as many as shared memory allows while keeping >= 96 registers per thread
  static constexpr int MB_SMEM = (int)(232448 / (SMEM + 1024)), MB_REG = 65536 / (96 * T);
  static constexpr int MB0 = MB_SMEM < MB_REG ? MB_SMEM : MB_REG;
  static constexpr int MINB = MB0 < 1 ? 1 : (MB0 > 4 ? 4 : MB0);
  static_assert(NY % G == 0 && NX % G == 0, "G must divide both dimensions");
  static_assert(T % 32 == 0 && T <= 1024, "R * PX must be a whole number of warps");
  static_assert(SX::VEC, "row tiles need an even P");
  static_assert(CC * PY <= T && R * QX <= T, "one task per thread in every phase");
};

struct GroupArgs {
  const float2* x;
  const float2* anchor;
  const float2* maps;
  long long map_bstride;
  const uint8_t* maskT;
  long long mask_bstride;
  float2* out;
  float2* scratch;  // ngroups x 2 x D
  float2* partial;  // ngroups x 2 x D
  int* sync;        // ngroups x 32 counters (A at +0, B at +16), then batch x G arrival counts
  int batch, ncoils, ngroups;
  float oscale;
  const float4* coef;
  const float2* u;
  const float2* d;
};

// unit u -> group owning it, for the balanced split [U g / n, U (g+1) / n)
__device__ __forceinline__ int group_of(long long u, long long U, int n) {
  return (int)((n * (u + 1) + U - 1) / U) - 1;
}

template <int PY, int QY, int PX, int QX, int G>
__global__ void __launch_bounds__(GrpCfg<PY, QY, PX, QX, G>::T, GrpCfg<PY, QY, PX, QX, G>::MINB)
k_cart_group(const GroupArgs a) {
  using Cf = GrpCfg<PY, QY, PX, QX, G>;
  using SX = typename Cf::SX;
  using SY = typename Cf::SY;
  constexpr int NX = Cf::NX, NY = Cf::NY, R = Cf::R, CC = Cf::CC, T = Cf::T;
  constexpr int VSX = Cf::VSX, VSPY = Cf::VSPY, ACCS = Cf::ACCS;
  constexpr long long D = (long long)NX * NY;
  extern __shared__ __align__(16) float2 dsm[];
  __shared__ int s_last;
  float2* tx1 = dsm + Cf::OFF_TX1;
  float2* tx2 = dsm + Cf::OFF_TX2;
  float2* ty1 = dsm + Cf::OFF_TY1;
  float2* ty2 = dsm + Cf::OFF_TY2;
  float2* acc = dsm + Cf::OFF_ACC;
  float2* buf = dsm + Cf::OFF_BUF;

  const int tid = threadIdx.x;
  const int grp = blockIdx.x / G, rank = blockIdx.x - grp * G;
  const int n = a.ngroups;
  if (grp >= n) return;
  const long long U = (long long)a.batch * a.ncoils;
  const long long ub = U * grp / n, ue = U * (grp + 1) / n;
  if (ub >= ue) return;
  const int ncoils = a.ncoils;
  const int row0 = rank * R, col0 = rank * CC;
  init_tw_s1<PX, QX>(tx1, tid, T);
  init_tw_s2<PX, QX>(tx2, tid, T);
  init_tw_s1<PY, QY>(ty1, tid, T);
  init_tw_s2<PY, QY>(ty2, tid, T);
  for (int e = tid; e < R * ACCS; e += T) acc[e] = make_float2(0.f, 0.f);
  int* cntA = a.sync + grp * 32;
  int* cntB = cntA + 16;
  int* scnt = a.sync + n * 32;
  float2* scr0 = a.scratch + (long long)grp * 2 * D;
  // row-pass thread coordinates: (row lr of the band, p)
  const int lr = tid / PX, p = tid - lr * PX;
  const int row = row0 + lr;
  __syncthreads();

  // ------------------------------------------------------------ phase A
  auto phaseA = [&](long long uu, float2* scr) {
    const int b = (int)(uu / ncoils), j = (int)(uu - (long long)b * ncoils);
    const long long xo = (long long)b * D + (long long)row * NX + p;
    const float2* mr = a.maps + b * a.map_bstride + j * D + (long long)row * NX + p;
    const uint64_t keep = pol_last();
    const float2* abase = a.anchor ? a.anchor : a.x;  // never null-based, even if hoisted
    float2 r[QX];
#pragma unroll
    for (int q = 0; q < QX; ++q) {
      float2 v = ld_nc_hint(a.x + xo + PX * q, keep);
      if (a.anchor) v = csub(v, ld_nc_hint(abase + xo + PX * q, keep));
      r[q] = cmul(ld_nc_hint(mr + PX * q, keep), v);
    }
    fft_s1_fwd<PX, QX>(r, p, tx1);
#pragma unroll
    for (int k2 = 0; k2 < QX; ++k2) buf[lr * VSX + SX::GS * k2 + p] = r[k2];
    __syncthreads();
    if (tid < R * QX) {
      const int l2 = tid / QX, k2 = tid - l2 * QX;
      float2 g[PX];
      float2* gp = buf + l2 * VSX + SX::GS * k2;
      lds_group<PX, true>(g, gp);
      fft_s2_fwd<PX>(g);
      sts_group<PX, true>(gp, g);
    }
    __syncthreads();
    float2* dst = scr + (long long)row0 * NX;
    for (int e = 2 * tid; e < R * NX; e += 2 * T) {
      const int l3 = e / NX, pos = e - l3 * NX;
      st_cg4_hint(dst + e, *reinterpret_cast<const float4*>(buf + l3 * VSX + SX::pad(pos)), keep);
    }
  };

  // ------------------------------------------------------------ phase B
  auto phaseB = [&](long long uu, float2* scr) {
    const int b = (int)(uu / ncoils);
    const int c = tid % CC, pc = tid / CC;
    const bool act = tid < CC * PY;
    const uint64_t keep = pol_last();
    float2* scol = scr + (long long)pc * NX + col0 + c;
    if (act) {
      float2 r[QY];
#pragma unroll
      for (int q = 0; q < QY; ++q) r[q] = ld_cg_hint(scol + (long long)(PY * q) * NX, keep);
      fft_s1_fwd<PY, QY>(r, pc, ty1);
#pragma unroll
      for (int k2 = 0; k2 < QY; ++k2) buf[c * VSPY + SY::GS * k2 + pc] = r[k2];
    }
    __syncthreads();
    if (tid < CC * QY) {
      const int cc = tid % CC, k2 = tid / CC;
      float2 g[PY];
      float2* gp = buf + cc * VSPY + SY::GS * k2;
#pragma unroll
      for (int k1 = 0; k1 < PY; ++k1) g[k1] = gp[k1];
      fft_s2_fwd<PY>(g);
      const uint8_t* mk = a.maskT + b * a.mask_bstride + (long long)(col0 + cc) * NY + PY * k2;
      if constexpr ((PY % 4) == 0) {
#pragma unroll
        for (int w4 = 0; w4 < PY / 4; ++w4) {
          const uint32_t m4 = __ldg(reinterpret_cast<const uint32_t*>(mk) + w4);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (!((m4 >> (8 * i)) & 0xffu)) g[4 * w4 + i] = make_float2(0.f, 0.f);
        }
      } else {
#pragma unroll
        for (int k1 = 0; k1 < PY; ++k1)
          if (!mk[k1]) g[k1] = make_float2(0.f, 0.f);
      }
      fft_s2_inv<PY, QY>(g, k2, ty2);
#pragma unroll
      for (int k1 = 0; k1 < PY; ++k1) gp[k1] = g[k1];
    }
    __syncthreads();
    if (act) {
      float2 r[QY];
#pragma unroll
      for (int k2 = 0; k2 < QY; ++k2) r[k2] = buf[c * VSPY + SY::GS * k2 + pc];
      fft_s1_inv<QY>(r);
#pragma unroll
      for (int q = 0; q < QY; ++q) st_cg2_hint(scol + (long long)(PY * q) * NX, r[q], keep);
    }
  };

  // ------------------------------------------------------------ phase C
  auto phaseC = [&](long long uu, float2* scr) {
    const int b = (int)(uu / ncoils), j = (int)(uu - (long long)b * ncoils);
    const float2* src = scr + (long long)row0 * NX;
    const uint64_t keep = pol_last(), drop = pol_first();
    for (int e = 2 * tid; e < R * NX; e += 2 * T) {
      const int l3 = e / NX, pos = e - l3 * NX;
      cp_async16_hint(buf + l3 * VSX + SX::pad(pos), src + e, keep);
    }
    cp_async_commit();
    const float2* mr = a.maps + b * a.map_bstride + j * D + (long long)row * NX + p;
    float2 m[QX];
#pragma unroll
    for (int q = 0; q < QX; ++q) m[q] = ld_nc_hint(mr + PX * q, drop);
    cp_async_wait<0>();
    __syncthreads();
    if (tid < R * QX) {
      const int l2 = tid / QX, k2 = tid - l2 * QX;
      float2 g[PX];
      float2* gp = buf + l2 * VSX + SX::GS * k2;
      lds_group<PX, true>(g, gp);
      fft_s2_inv<PX, QX>(g, k2, tx2);
      sts_group<PX, true>(gp, g);
    }
    __syncthreads();
    float2 r[QX];
#pragma unroll
    for (int k2 = 0; k2 < QX; ++k2) r[k2] = buf[lr * VSX + SX::GS * k2 + p];
    fft_s1_inv<QX>(r);
    float2* ar = acc + lr * ACCS + p;
#pragma unroll
    for (int q = 0; q < QX; ++q) {
      float2 v = ar[PX * q];
      cfma_conj(v, m[q], r[q]);
      ar[PX * q] = v;
    }
    __syncthreads();  // buf is reused by the next phase
  };

  auto epilogue = [&](int b, float2 v, long long off) {
    v = cscale(v, a.oscale);
    if (a.coef) {
      const float4 cf = a.coef[b];
      v = cscale(v, cf.x);
      if (a.u) { const float2 uu = a.u[off]; v.x = fmaf(cf.y, uu.x, v.x); v.y = fmaf(cf.y, uu.y, v.y); }
      if (a.d) { const float2 dd = a.d[off]; v.x = fmaf(cf.z, dd.x, v.x); v.y = fmaf(cf.z, dd.y, v.y); }
    }
    a.out[off] = v;
  };

  // slice b's coils [b*ncoils, (b+1)*ncoils) are done in this group's range
  auto finish = [&](int b) {
    const long long s0 = (long long)b * ncoils, s1 = s0 + ncoils;
    const long long band = (long long)b * D + (long long)row0 * NX;
    if (s0 >= ub && s1 <= ue) {
      for (int e = tid; e < R * NX; e += T) {
        const int l3 = e / NX, pos = e - l3 * NX;
        float2* ap = acc + l3 * ACCS + pos;
        epilogue(b, *ap, band + e);
        *ap = make_float2(0.f, 0.f);
      }
      __syncthreads();
      return;
    }
    const int slot = (b == (int)(ub / ncoils)) ? 0 : 1;
    float2* pp = a.partial + (long long)(grp * 2 + slot) * D + (long long)row0 * NX;
    for (int e = tid; e < R * NX; e += T) {
      const int l3 = e / NX, pos = e - l3 * NX;
      float2* ap = acc + l3 * ACCS + pos;
      st_cg2(pp + e, *ap);
      *ap = make_float2(0.f, 0.f);
    }
    __threadfence();
    __syncthreads();
    const int g0 = group_of(s0, U, n), g1 = group_of(s1 - 1, U, n);
    if (tid == 0) {
      const int old = atomicAdd(scnt + b * G + rank, 1);
      s_last = (old == g1 - g0);
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      for (int e = tid; e < R * NX; e += T) {
        float2 v = make_float2(0.f, 0.f);
        for (int g = g0; g <= g1; ++g) {
          const int sl = (b == (int)((U * g / n) / ncoils)) ? 0 : 1;
          v = cadd(v, ld_cg2(a.partial + (long long)(g * 2 + sl) * D + (long long)row0 * NX + e));
        }
        epilogue(b, v, band + e);
      }
    }
    __syncthreads();
  };

  // two scratch buffers: iteration k runs B(k), A(k+1), C(k)
  const int nu = (int)(ue - ub);
  auto scr_of = [&](int k) { return scr0 + (k & 1) * D; };
  phaseA(ub, scr_of(0));
  group_arrive(cntA);
  for (int k = 0; k < nu; ++k) {
    group_wait(cntA, G * (k + 1));
    phaseB(ub + k, scr_of(k));
    group_arrive(cntB);
    if (k + 1 < nu) {
      phaseA(ub + k + 1, scr_of(k + 1));
      group_arrive(cntA);
    }
    group_wait(cntB, G * (k + 1));
    const long long uu = ub + k;
    phaseC(uu, scr_of(k));
    const int b = (int)(uu / ncoils);
    if (uu - (long long)b * ncoils == ncoils - 1 || uu + 1 == ue) finish(b);
  }
}

// X(NY, PY, QY, NX, PX, QX, G): the first entry of a size is its default; sr_group_select(G)
// picks another instantiated group size (tuning)
#define SR_GROUP_CFGS(X)                 \
  X(320, 20, 16, 320, 20, 16, 20)        \
  X(320, 20, 16, 320, 20, 16, 40)        \
  X(320, 20, 16, 320, 20, 16, 10)        \
  X(256, 16, 16, 256, 16, 16, 16)        \
  X(256, 16, 16, 256, 16, 16, 8)         \
  X(256, 16, 16, 160, 16, 10, 16)        \
  X(256, 16, 16, 160, 16, 10, 8)         \
  X(64, 16, 4, 64, 16, 4, 4)

int g_group_pref = 0;

int group_G(int ny, int nx) {
  int first = 0;
#define X(NY, PY, QY, NX, PX, QX, G)                 \
  if (ny == NY && nx == NX) {                          \
    if (G == g_group_pref) return G;                   \
    if (!first) first = G;                             \
  }
  SR_GROUP_CFGS(X)
#undef X
  return first;
}

template <int PY, int QY, int PX, int QX, int G>
int group_ngroups() {
  using Cf = GrpCfg<PY, QY, PX, QX, G>;
  static int cached = 0;
  if (cached) return cached;
  int dev = 0, nsm = 0, occ = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  if (cudaFuncSetAttribute(k_cart_group<PY, QY, PX, QX, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)Cf::SMEM) != cudaSuccess)
    return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cart_group<PY, QY, PX, QX, G>, Cf::T,
                                                    Cf::SMEM) != cudaSuccess)
    return 0;
  cached = (nsm * occ) / G;  // every CTA of the grid is co-resident
  return cached;
}

int ngroups_for(int ny, int nx) {
  const int g = group_G(ny, nx);
#define X(NY, PY, QY, NX, PX, QX, G) \
  if (ny == NY && nx == NX && g == G) return group_ngroups<PY, QY, PX, QX, G>();
  SR_GROUP_CFGS(X)
#undef X
  return 0;
}

template <int PY, int QY, int PX, int QX, int G>
int launch_group(const GroupArgs& a, cudaStream_t st) {
  using Cf = GrpCfg<PY, QY, PX, QX, G>;
  k_cart_group<PY, QY, PX, QX, G><<<a.ngroups * G, Cf::T, Cf::SMEM, st>>>(a);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// entry points (sr_cart_normal in cart.cu dispatches chunk == -2 here)

extern "C" int sr_group_select(int g) {
  g_group_pref = g;
  return SR_OK;
}

extern "C" int sr_group_normal_supported(int ny, int nx) { return group_G(ny, nx) > 0 ? 1 : 0; }

extern "C" int sr_group_ngroups(int ny, int nx) { return group_G(ny, nx) > 0 ? ngroups_for(ny, nx) : 0; }

long long sr_group_ws_bytes(int batch, int ny, int nx) {
  const int n = sr_group_ngroups(ny, nx);
  const int G = group_G(ny, nx);
  if (n <= 0) return 0;
  const long long D = (long long)ny * nx;
  return 8LL * 4 * n * D + 4LL * (32LL * n + (long long)batch * G) + 256;
}

int sr_group_normal(const float2* x, const float2* anchor, const float2* maps, long long map_bstride,
                    const uint8_t* maskT, long long mask_bstride, float2* out, void* ws, int batch,
                    int ncoils, int ny, int nx, const float4* coef, const float2* u, const float2* d,
                    cudaStream_t st) {
  const int nmax = sr_group_ngroups(ny, nx);
  const int G = group_G(ny, nx);
  if (nmax <= 0) return SR_EUNSUPPORTED;
  const long long D = (long long)ny * nx;
  // at most one group per unit: every range is then non-empty, which the partial-sum
  // arrival count (groups g0..g1 of a slice) relies on
  const long long U = (long long)batch * ncoils;
  const int n = (int)(U < nmax ? U : nmax);
  GroupArgs a;
  a.x = x; a.anchor = anchor; a.maps = maps; a.map_bstride = map_bstride;
  a.maskT = maskT; a.mask_bstride = mask_bstride; a.out = out;
  a.scratch = (float2*)ws;
  a.partial = a.scratch + 2LL * nmax * D;
  a.sync = (int*)(a.partial + 2LL * nmax * D);
  a.batch = batch; a.ncoils = ncoils; a.ngroups = n;
  a.oscale = (float)(1.0 / (double)D);
  a.coef = coef; a.u = u; a.d = d;
  if (cudaMemsetAsync(a.sync, 0, 4LL * (32LL * n + (long long)batch * G), st) != cudaSuccess)
    return SR_ECUDA;
#define X(NY, PY, QY, NX, PX, QX, G_) \
  if (ny == NY && nx == NX && G == G_) return launch_group<PY, QY, PX, QX, G_>(a, st);
  SR_GROUP_CFGS(X)
#undef X
  return SR_EUNSUPPORTED;
}

// K1 single-pass schedule: one 4-CTA thread-block cluster holds a whole coil image on chip.
//
// Reference path (the same operator as cart.cu's three-pass schedule):
//   SenseOperator._forward/_adjoint  /root/reference/pkg/src/sketchrecon/forward_model.py:168-180
//   _CartesianMaskKernel.apply/apply_adjoint  /root/reference/pkg/src/sketchrecon/linops.py:344-364
//   out_b = sum_j conj(c_bj) . F^H M' F (c_bj . (x_b - a_b))      [+ epilogue]
//
// The three-pass schedule moves every coil image through HBM three times (row FFT -> workspace
// -> column pass -> workspace -> row IFFT): 3.78 GB per config-1 apply for 0.73 GB of
// compulsory traffic.  Here the coil image never leaves the chip.  A cluster of CL = 4 CTAs (one
// per SM, ~206 KB of shared memory each) owns one slice; CTA s keeps the image rows
// y = s + 4 n (n < NL = ny / 4) for one coil at a time and loops over the coils:
//
//   F   row FFT step 1 of coil j straight from HBM (u = c_j (x - a)), fused with the row IFFT
//       step 1' of coil j-1 and its conj(c_{j-1}) accumulation (same thread, same positions)
//   R   row FFT step 2 (groups of P in shared memory)
//   C   local column DFT of length NL per column, one thread per column, in registers:
//         A_s[k1] = sum_n u[s + 4 n] W_NL^{n k1}
//   X   the only cross-CTA step, through distributed shared memory.  For ky = k1 + NL k2,
//         U[ky] = sum_r W_ny^{r k1} W_4^{r k2} A_r[k1]        (twiddle + DFT_4 over the CTAs)
//       so a "group" (column, k1) couples exactly one value per CTA: the owner CTA of k1 reads
//       the 4 values, applies twiddle . DFT_4 . mask . IDFT_4 . conj twiddle and writes the 4
//       results back; a group whose 4 mask bits are all 0 moves nothing (every CTA zeroes its
//       own slot), so the exchange is pruned by the undersampling.
//   C'  local column IDFT, R' row IFFT step 2', then F of the next coil.
// Shared memory per CTA holds the NL rows (pitch NX + 2 float2: 16-byte rows, and the 128-bit
// row-group accesses of R / R' with lanes over rows are bank-conflict free), the row twiddles
// and the exchange twiddles.  The coil sum accumulates in an L2-resident buffer (ws) owned by the
// CTA's rows, so out may alias x, u or d as in the three-pass schedule.  HBM traffic is the maps
// (read for u and again for the conj sum), x and out: ~1.3 GB per config-1 apply.
#include <cooperative_groups.h>

#include "fft2step.cuh"

namespace cg = cooperative_groups;

int sr_g_cluster_min_batch = 16;  // slices per launch from which sr_cart_normal takes this path (0 = never)
static long long* sr_g_cluster_prof = nullptr;  // device buffer of 7 phase clock sums (probe only)

namespace {

constexpr int CL = 4;

template <int NL, int P, int Q>
struct ClCfg {
  static constexpr int NX = P * Q;
  static constexpr int NY = NL * CL;
  static constexpr int T = NX;           // one thread per column in the column phases
  static constexpr int PITCH = NX + 2;   // float2; 2*PITCH = 4 (mod 32) for NX = 0 (mod 16)
  static constexpr int KO = NL / CL;     // groups owned per column
  static constexpr size_t SMEM = sizeof(float2) * ((size_t)NL * PITCH + 2 * NX + 3 * NL);
  static_assert(NX % 32 == 0, "one thread per column: whole warps");
  static_assert(NX % 16 == 0 && P % 2 == 0, "16-byte row groups");
  static_assert(NL % (4 * CL) == 0 && NL / CL <= 32, "owned group ranges: whole 32-bit mask words");
};

// grp[b][c][k1] = bit k2 set iff ky = k1 + NL k2 is sampled in column (perm position) c
__global__ void k_cl_groups(const uint8_t* __restrict__ maskT, long long mbs, uint8_t* __restrict__ grp,
                            int ny, int nx, int nl, int py, int qy) {
  const int b = blockIdx.y;
  const uint8_t* mk = maskT + b * mbs;
  uint8_t* g = grp + (long long)b * nx * nl;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nx * nl; e += gridDim.x * blockDim.x) {
    const int c = e / nl, k1 = e - c * nl;
    unsigned bits = 0;
#pragma unroll
    for (int k2 = 0; k2 < CL; ++k2) {
      const int ky = k1 + nl * k2;
      const int pos = py * (ky % qy) + ky / qy;
      bits |= (mk[(long long)c * ny + pos] ? 1u : 0u) << k2;
    }
    g[e] = (uint8_t)bits;
  }
}

template <int NL, int P, int Q>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(P * Q, 1)
k_cart_cluster(const float2* __restrict__ x, const float2* __restrict__ anchor, const float2* __restrict__ maps,
               const uint8_t* __restrict__ grp, float2* __restrict__ accb, float2* out, int ncoils,
               long long xbs, long long mbs, const float4* __restrict__ coef, const float2* u, const float2* d,
               float oscale, long long* prof) {
  using C = ClCfg<NL, P, Q>;
  constexpr int NX = C::NX, NY = C::NY, T = C::T, PITCH = C::PITCH, KO = C::KO;
  extern __shared__ __align__(16) float2 sm[];
  float2* img = sm;
  float2* t1 = sm + NL * PITCH;
  float2* t2 = t1 + NX;
  float2* tx = t2 + NX;  // tx[(r - 1) * NL + k1] = W_NY^{r k1}
  cg::cluster_group cl = cg::this_cluster();
  const int s = (int)cl.block_rank();
  const int b = blockIdx.x / CL;
  const int tid = threadIdx.x;
  init_tw_s1<P, Q>(t1, tid, T);
  init_tw_s2<P, Q>(t2, tid, T);
  for (int e = tid; e < (CL - 1) * NL; e += T) {
    const int r = e / NL + 1, k1 = e - (r - 1) * NL;
    double sn, cs;
    sincospi(-2.0 * (double)((r * k1) % NY) / (double)NY, &sn, &cs);
    tx[e] = make_float2((float)cs, (float)sn);
  }
  float2* rimg[CL];
#pragma unroll
  for (int r = 0; r < CL; ++r) rimg[r] = cl.map_shared_rank(img, r);
  __syncthreads();

  constexpr long long D = (long long)NY * NX;
  const float2* xb = x + b * xbs;
  const float2* axb = anchor ? anchor + b * xbs : xb;
  const float2* mb = maps + b * mbs;
  float2* ab = accb + b * D;
  const uint8_t* gcol = grp + ((long long)b * NX + tid) * NL;

  // optional per-phase clocks (thread 0, summed over CTAs): F-inv, F-fwd, R, C, X, C', R'
  __shared__ long long pcs[8];  // [0, 7): phase sums, [7]: last stamp
  if (prof && tid == 0) {
#pragma unroll
    for (int i = 0; i < 7; ++i) pcs[i] = 0;
    pcs[7] = clock64();
  }
  auto tick = [&](int ph) {
    if (prof && tid == 0) {
      const long long t = clock64();
      pcs[ph] += t - pcs[7];
      pcs[7] = t;
    }
  };
  // the next coil's map rows go to L2 ahead of their use (one bulk prefetch per row)
  auto prefetch_maps = [&](int jj) {
    if (jj < ncoils && tid < NL)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(mb + (long long)jj * D +
                                                                        (long long)(s + CL * tid) * NX),
                   "r"(NX * 8)
                   : "memory");
  };
  prefetch_maps(0);

  for (int j = 0; j <= ncoils; ++j) {
    // ---- F (inverse half): row IFFT step 1' of coil j-1 and the conj(c_{j-1}) coil sum
    if (j > 0) {
      for (int task = tid; task < NL * P; task += T) {
        const int n = task / P, p = task - n * P;
        const long long ro = (long long)(s + CL * n) * NX + p;
        const float2* irow = img + n * PITCH + p;
        const float2* cm = mb + (long long)(j - 1) * D + ro;
        float2 cv[Q], av[Q];
#pragma unroll
        for (int m2 = 0; m2 < Q; ++m2) cv[m2] = __ldcs(cm + P * m2);
        if (j > 1) {
#pragma unroll
          for (int m2 = 0; m2 < Q; ++m2) av[m2] = ab[ro + P * m2];
        } else {
#pragma unroll
          for (int m2 = 0; m2 < Q; ++m2) av[m2] = make_float2(0.f, 0.f);
        }
        float2 r[Q];
#pragma unroll
        for (int k2 = 0; k2 < Q; ++k2) r[k2] = irow[P * k2];
        fft_s1_inv<Q>(r);
#pragma unroll
        for (int m2 = 0; m2 < Q; ++m2) cfma_conj(av[m2], cv[m2], r[m2]);
        if (j < ncoils) {
#pragma unroll
          for (int m2 = 0; m2 < Q; ++m2) ab[ro + P * m2] = av[m2];
        } else {
          const float4 cf = coef ? coef[b] : make_float4(1.f, 0.f, 0.f, 0.f);
          const long long oo = b * xbs + ro;
#pragma unroll
          for (int m2 = 0; m2 < Q; ++m2) {
            float2 a = cscale(av[m2], oscale);
            if (coef) {
              a = cscale(a, cf.x);
              if (u) { const float2 uu = u[oo + P * m2]; a.x = fmaf(cf.y, uu.x, a.x); a.y = fmaf(cf.y, uu.y, a.y); }
              if (d) { const float2 dd = d[oo + P * m2]; a.x = fmaf(cf.z, dd.x, a.x); a.y = fmaf(cf.z, dd.y, a.y); }
            }
            out[oo + P * m2] = a;
          }
        }
      }
    }
    tick(0);
    if (j == ncoils) break;
    // ---- F (forward half): u = c_j (x - a), row FFT step 1 (same tasks -> in place per thread)
    for (int task = tid; task < NL * P; task += T) {
      const int n = task / P, p = task - n * P;
      const long long ro = (long long)(s + CL * n) * NX + p;
      float2* irow = img + n * PITCH + p;
      const float2* cj = mb + (long long)j * D + ro;
      float2 r[Q], xv[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) r[q] = __ldg(cj + P * q);
#pragma unroll
      for (int q = 0; q < Q; ++q) xv[q] = xb[ro + P * q];
      if (anchor) {
#pragma unroll
        for (int q = 0; q < Q; ++q) xv[q] = csub(xv[q], axb[ro + P * q]);
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) r[q] = cmul(r[q], xv[q]);
      fft_s1_fwd<P, Q>(r, p, t1);
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) irow[P * k2] = r[k2];
    }
    prefetch_maps(j + 1);
    __syncthreads();
    tick(1);

    // ---- R: row FFT step 2, one (row, k2) group per task, lanes over rows
    for (int task = tid; task < NL * Q; task += T) {
      const int n = task % NL, k2 = task / NL;
      float2 g[P];
      float2* gp = img + n * PITCH + P * k2;
      lds_group<P, true>(g, gp);
      fft_s2_fwd<P>(g);
      sts_group<P, true>(gp, g);
    }
    __syncthreads();
    tick(2);

    // ---- C: local column DFT of length NL (one thread per column)
    {
      float2 v[NL];
#pragma unroll
      for (int n = 0; n < NL; ++n) v[n] = img[n * PITCH + tid];
      RegDFT<NL, false>::run(v);
#pragma unroll
      for (int k = 0; k < NL; ++k) img[k * PITCH + tid] = v[k];
    }
    cl.sync();
    tick(3);

    // ---- X: cross-CTA radix-4 step with the mask, pruned to the sampled groups
    {
      const int c = tid;
      uint32_t gw[NL / 4];
#pragma unroll
      for (int w = 0; w < NL / 16; ++w) {
        const uint4 q4 = __ldg(reinterpret_cast<const uint4*>(gcol) + w);
        gw[4 * w] = q4.x; gw[4 * w + 1] = q4.y; gw[4 * w + 2] = q4.z; gw[4 * w + 3] = q4.w;
      }
      // empty groups: every CTA zeroes its own slot
#pragma unroll
      for (int w = 0; w < NL / 4; ++w) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (((gw[w] >> (8 * i)) & 0xffu) == 0u) img[(4 * w + i) * PITCH + c] = make_float2(0.f, 0.f);
      }
      // owned non-empty groups, four at a time so their remote loads are in flight together;
      // their mask nibbles packed in two 64-bit words (no dynamically indexed register arrays)
      const int k0 = s * KO;
      uint32_t live = 0;
      unsigned long long nib[2] = {0ull, 0ull};
#pragma unroll
      for (int w = 0; w < KO / 4; ++w) {
        const uint32_t ow = __ldg(reinterpret_cast<const uint32_t*>(gcol + k0) + w);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int o = 4 * w + i;
          const uint32_t bits = (ow >> (8 * i)) & 0xfu;
          live |= (bits ? 1u : 0u) << o;
          nib[o / 16] |= (unsigned long long)bits << (4 * (o % 16));
        }
      }
      while (live) {
        int kk[4];
        uint32_t kb[4];
        bool ok[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          ok[t] = live != 0u;
          const int i = ok[t] ? __ffs(live) - 1 : 0;
          live &= live - 1u;
          kk[t] = k0 + i;
          kb[t] = (unsigned)((i < 16 ? nib[0] >> (4 * i) : nib[1] >> (4 * (i - 16))) & 0xfull);
        }
        float2 v[4][CL];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
#pragma unroll
          for (int r = 0; r < CL; ++r)
            v[t][r] = ok[t] ? rimg[r][kk[t] * PITCH + c] : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (!ok[t]) continue;
          const int k1 = kk[t];
          const uint32_t bits = kb[t];
#pragma unroll
          for (int r = 1; r < CL; ++r) v[t][r] = cmul(v[t][r], tx[(r - 1) * NL + k1]);
          RegDFT<CL, false>::run(v[t]);
#pragma unroll
          for (int k2 = 0; k2 < CL; ++k2)
            if (!((bits >> k2) & 1u)) v[t][k2] = make_float2(0.f, 0.f);
          RegDFT<CL, true>::run(v[t]);
#pragma unroll
          for (int r = 1; r < CL; ++r) v[t][r] = cmulc(tx[(r - 1) * NL + k1], v[t][r]);
#pragma unroll
          for (int r = 0; r < CL; ++r) rimg[r][k1 * PITCH + c] = v[t][r];
        }
      }
    }
    cl.sync();
    tick(4);

    // ---- C': local column IDFT
    {
      float2 v[NL];
#pragma unroll
      for (int k = 0; k < NL; ++k) v[k] = img[k * PITCH + tid];
      RegDFT<NL, true>::run(v);
#pragma unroll
      for (int n = 0; n < NL; ++n) img[n * PITCH + tid] = v[n];
    }
    __syncthreads();
    tick(5);

    // ---- R': row IFFT step 2'
    for (int task = tid; task < NL * Q; task += T) {
      const int n = task % NL, k2 = task / NL;
      float2 g[P];
      float2* gp = img + n * PITCH + P * k2;
      lds_group<P, true>(g, gp);
      fft_s2_inv<P, Q>(g, k2, t2);
      sts_group<P, true>(gp, g);
    }
    __syncthreads();
    tick(6);
  }
  if (prof && tid == 0) {
#pragma unroll
    for (int i = 0; i < 7; ++i) atomicAdd(reinterpret_cast<unsigned long long*>(prof) + i, (unsigned long long)pcs[i]);
  }
}

template <int NL, int P, int Q>
int launch_cluster_t(const float2* x, const float2* anchor, const float2* maps, long long mbs,
                     const uint8_t* maskT, long long mask_bstride, float2* out, void* ws, int batch,
                     int ncoils, const float4* coef, const float2* u, const float2* d, float oscale,
                     cudaStream_t st) {
  using C = ClCfg<NL, P, Q>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(k_cart_cluster<NL, P, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)C::SMEM) != cudaSuccess)
      return SR_ECUDA;
    configured = true;
  }
  const long long D = (long long)C::NY * C::NX;
  // ws: group table (batch * nx * NL bytes, 256-byte rounded), then the coil-sum buffer (batch * D)
  uint8_t* grp = (uint8_t*)ws;
  const long long gbytes = (((long long)batch * C::NX * NL) + 255) / 256 * 256;
  float2* acc = (float2*)((uint8_t*)ws + gbytes);
  int py = 0, qy = 0;
  if (sr_fft_split(C::NY, &py, &qy) != SR_OK) return SR_EUNSUPPORTED;
  dim3 gg((C::NX * NL + 255) / 256, batch);
  k_cl_groups<<<gg, 256, 0, st>>>(maskT, mask_bstride, grp, C::NY, C::NX, NL, py, qy);
  SR_CHECK_LAUNCH();
  k_cart_cluster<NL, P, Q><<<batch * CL, C::T, C::SMEM, st>>>(x, anchor, maps, grp, acc, out, ncoils, D, mbs,
                                                              coef, u, d, oscale, sr_g_cluster_prof);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

}  // namespace

// Returns SR_EUNSUPPORTED when no cluster instantiation covers (ny, nx) (the caller then runs
// the three-pass schedule).
int sr_cart_cluster_normal(const float2* x, const float2* anchor, const float2* maps, long long mbs,
                           const uint8_t* maskT, long long mask_bstride, float2* out, void* ws, int batch,
                           int ncoils, int ny, int nx, const float4* coef, const float2* u, const float2* d,
                           float oscale, cudaStream_t st) {
#define SR_CL_CASE(NY_, NX_, NL_, P_, Q_)                                                              \
  if (ny == NY_ && nx == NX_)                                                                          \
    return launch_cluster_t<NL_, P_, Q_>(x, anchor, maps, mbs, maskT, mask_bstride, out, ws, batch, ncoils, \
                                         coef, u, d, oscale, st);
  SR_CL_CASE(320, 320, 80, 20, 16)
  SR_CL_CASE(256, 256, 64, 16, 16)
  SR_CL_CASE(256, 160, 64, 16, 10)
#undef SR_CL_CASE
  return SR_EUNSUPPORTED;
}

extern "C" int sr_cart_cluster_profile(void* buf) {
  sr_g_cluster_prof = (long long*)buf;
  return SR_OK;
}

long long sr_cart_cluster_ws_bytes(int batch, int ncoils, int ny, int nx) {
  (void)ncoils;
  const long long D = (long long)ny * nx;
  return ((long long)batch * D / 4 + 255) / 256 * 256 + 8LL * batch * D;
}

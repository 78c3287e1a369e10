// Cartesian three-pass kernels (K1/K2) and their launchers, shared by the size-bucket
// translation units cart_inst_<k>.cu (split so nvcc compiles the instantiations in parallel).
// See cart.cu for the algorithm and the reference mapping.
#pragma once
#include <type_traits>

#include "fft2step.cuh"

extern int sr_g_col_jc;  // coils per CTA of k_colnormal (0 = use k_colpass); cart.cu
extern int sr_g_col_pf;  // k_colnormal: 1 = next coil's strip prefetched in registers (2 CTAs/SM), 0 = not (3 CTAs/SM)
extern int sr_g_row_bulk, sr_g_row_bulk_min_n;  // rowfwd TMA bulk stores (on, min row length); cart.cu
extern int sr_g_carveout;  // preferred shared-memory carveout (percent, -1 = driver default) of the column pass; cart.cu

// apply the carveout knob to a kernel once per value (the L1 / shared split decides how many
// CTAs of a pass fit an SM: the driver's default picked 135 KB for the column pass = 2 CTAs)
template <typename K>
inline int apply_carveout(K kern, int& applied) {
  if (applied == sr_g_carveout) return SR_OK;
  const int v = sr_g_carveout < 0 ? -1 : sr_g_carveout;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, v) != cudaSuccess) return SR_ECUDA;
  applied = sr_g_carveout;
  return SR_OK;
}

enum { COL_NORMAL = 0, COL_FWD = 1, COL_INV = 2, COL_FWD_G = 3, COL_INV_S = 4 };

// K2 sample I/O fused into the column pass (modes COL_FWD_G / COL_INV_S): the samples of slice b
// whose perm-order x position falls in column block k are bidx[bptr[b][k] .. bptr[b][k+1]) (indices
// within the slice; spos / ph / y as in k_gather / k_scatter).
struct SampleIO {
  const int* spos;
  const float2* ph;
  const long long* soff;
  const int* bptr;  // (batch, nblk + 1), absolute offsets into bidx
  const int* bidx;
  float2* y;          // COL_FWD_G output
  const float2* yin;  // COL_INV_S input
  const float2* ymeas;
  double* partial;
  long long ystride;
  float scale;
  int nblk, pblocks;
};

namespace {

// ------------------------------------------------------------------- pass A
constexpr int cgcd(int a, int b) { return b == 0 ? a : cgcd(b, a % b); }
__host__ __device__ constexpr int pow2_floor(int n) { return n < 2 ? 1 : 2 * pow2_floor(n / 2); }

// ROWS rows per CTA, one thread per (row, p): T = ROWS * P is a whole number
// of warps and at least 128 threads.
template <int P, int Q>
struct RowCfg {
  static constexpr int BASE = 32 / cgcd(P, 32);
  static constexpr int ROWS0 = BASE * ((128 / (BASE * P)) > 1 ? (128 / (BASE * P)) : 1);
  static constexpr int ROWS = ROWS0 > 64 ? 64 : ROWS0;
  static constexpr int T = ROWS * P;
  static constexpr int MINB0 = (T <= 160) ? 4 : 3, MINB0_INV = (T <= 128) ? 4 : 3;
  static constexpr int MAXB = 2048 / T;  // resident threads per SM
  static constexpr int MINB = MINB0 < MAXB ? MINB0 : (MAXB > 0 ? MAXB : 1);
  static constexpr int MINB_INV = MINB0_INV < MAXB ? MINB0_INV : (MAXB > 0 ? MAXB : 1);
  static constexpr int N = P * Q;
  static constexpr int XS = N + ((((P % 16) - (N % 16)) % 16 + 16) % 16);  // x row stride = P (mod 16)
  // dynamic smem (float2): twiddles N | work rows ROWS*VS | [fwd only] staged x ROWS*XS
  static constexpr size_t SMEM_FWD = sizeof(float2) * (N + ROWS * RowShape<P, Q>::VS + ROWS * XS);
  static constexpr size_t SMEM_INV = sizeof(float2) * (N + 2 * ROWS * RowShape<P, Q>::VS);
};

template <int P, int Q>
__global__ void __launch_bounds__(RowCfg<P, Q>::T, RowCfg<P, Q>::MINB)
k_rowfwd(const float2* __restrict__ x, const float2* __restrict__ anchor,
         const float2* __restrict__ maps, float2* __restrict__ ws,
         int ncoils, int ny, long long x_bstride, long long map_bstride, int bulk, int cpg) {
  using S = RowShape<P, Q>;
  constexpr int N = S::N, ROWS = RowCfg<P, Q>::ROWS, T = RowCfg<P, Q>::T;
  constexpr int XS = RowCfg<P, Q>::XS;
  extern __shared__ __align__(16) float2 dsm[];
  float2* t1 = dsm;
  float2* buf = dsm + N;
  float2* xs = buf + ROWS * S::VS;
  const int tid = threadIdx.x;
  const int b = blockIdx.y;
  const int row0 = blockIdx.x * ROWS;
  const int lr = tid / P, p = tid % P;
  const int row = row0 + lr;
  const bool valid = row < ny;
  const long long D = (long long)ny * N;
  const int nvalid = min(ROWS, ny - row0) * N;
  init_tw_s1<P, Q>(t1, tid, T);
  // coils [jb, je) of this CTA (blockIdx.z = coil group: small batches spread coils over CTAs)
  const int jb = blockIdx.z * cpg, je = min(ncoils, jb + cpg);
  const float2* mb = maps + b * map_bstride + (long long)row * N + p;
  float2* wb = ws + (long long)b * ncoils * D + (long long)row0 * N;
  // software pipeline: coil j+1's map values are loaded while coil j is transformed
  float2 mcur[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) mcur[q] = valid ? __ldg(mb + jb * D + P * q) : make_float2(0.f, 0.f);
  // stage u = x - anchor for the CTA's rows once (reused by every coil); all loads of a
  // thread are issued before the first use so their latencies overlap (T * Q = ROWS * N)
  {
    const float2* xb = x + b * x_bstride + (long long)row0 * N;
    // never a null-based address, even for loads the compiler hoists above the anchor test
    const float2* ab = anchor ? anchor + b * x_bstride + (long long)row0 * N : xb;
    float2 v[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      const int e = tid + i * T;
      v[i] = e < nvalid ? __ldg(xb + e) : make_float2(0.f, 0.f);
    }
    if (anchor) {
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        const int e = tid + i * T;
        if (e < nvalid) v[i] = csub(v[i], __ldg(ab + e));
      }
    }
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      const int e = tid + i * T;
      const int l3 = e / N, pos = e - l3 * N;
      xs[l3 * XS + pos] = v[i];
    }
  }
  __syncthreads();
  const float2* xr = xs + lr * XS + p;
  for (int j = jb; j < je; ++j) {
    float2 r[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) r[q] = cmul(mcur[q], xr[P * q]);
    if (j + 1 < je && valid) {
      const float2* mn = mb + (j + 1) * D;
#pragma unroll
      for (int q = 0; q < Q; ++q) mcur[q] = __ldg(mn + P * q);
    }
    fft_s1_fwd<P, Q>(r, p, t1);
    float2* wj = wb + j * D;
    if (S::VEC && bulk) {
      // the previous coil's bulk stores must have read buf before it is overwritten
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncthreads();
    }
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) buf[lr * S::VS + S::GS * k2 + p] = r[k2];
    __syncthreads();
    if (S::VEC && bulk) {
      // step 2: each perm-order group (P contiguous values, 16-byte aligned in shared and
      // global memory) goes to the workspace as one TMA bulk store, no copy-out pass
      for (int it = tid; it < ROWS * Q; it += T) {
        const int l2 = it / Q, k2 = it - l2 * Q;
        float2 g[P];
        float2* gp = buf + l2 * S::VS + S::GS * k2;
        lds_group<P, true>(g, gp);
        fft_s2_fwd<P>(g);
        sts_group<P, true>(gp, g);
        if (l2 * N < nvalid) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          const unsigned src = (unsigned)__cvta_generic_to_shared(gp);
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                       :: "l"(wj + (long long)l2 * N + P * k2), "r"(src), "r"(P * 8) : "memory");
        }
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      continue;
    }
    if (P > 1) {
      for (int it = tid; it < ROWS * Q; it += T) {
        const int l2 = it / Q, k2 = it - l2 * Q;
        float2 g[P];
        float2* gp = buf + l2 * S::VS + S::GS * k2;
        lds_group<P, S::VEC>(g, gp);
        fft_s2_fwd<P>(g);
        sts_group<P, S::VEC>(gp, g);
      }
      __syncthreads();
    }
    if constexpr (S::VEC) {
      for (int e = 2 * tid; e < nvalid; e += 2 * T) {
        const int l3 = e / N, pos = e - l3 * N;
        *reinterpret_cast<float4*>(wj + e) = *reinterpret_cast<const float4*>(buf + l3 * S::VS + S::pad(pos));
      }
    } else {
      for (int e = tid; e < nvalid; e += T) {
        const int l3 = e / N, pos = e - l3 * N;
        wj[e] = buf[l3 * S::VS + S::pad(pos)];
      }
    }
    __syncthreads();
  }
  if (S::VEC && bulk) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------------- pass C
// Epilogue: out = s_acc * acc + s_u * u + s_d * d, coefficients per slice
// (coef[b] = {s_acc, s_u, s_d, unused}); coef == nullptr -> out = acc.
template <int P, int Q>
__global__ void __launch_bounds__(RowCfg<P, Q>::T, RowCfg<P, Q>::MINB_INV)
k_rowinv(float2* __restrict__ ws, const float2* __restrict__ maps,
         float2* __restrict__ out, int ncoils, int ny, long long x_bstride,
         long long map_bstride, const float4* __restrict__ coef,
         const float2* __restrict__ u, const float2* __restrict__ d, float oscale, int cpg) {
  // Rows contiguous in shared memory (one bulk copy per row) where the unpadded groups of P cost at
  // most 2-way bank conflicts in the 128-bit group loads (P = 20, 12); other even P (16: 8-way)
  // keep the padded groups filled by 16-byte cp.async (256 x 160 slices: 0.31 -> 0.275 s recon).
  static constexpr bool BULK = (P == 20 || P == 12);
  using S = typename std::conditional<BULK, RowShapeNP<P, Q>, RowShape<P, Q>>::type;
  constexpr int N = S::N, ROWS = RowCfg<P, Q>::ROWS, T = RowCfg<P, Q>::T;
  extern __shared__ __align__(16) float2 dsm[];
  float2* t2 = dsm;
  float2* bufs = dsm + N;  // two tiles of ROWS * VS (double buffer)
  const int tid = threadIdx.x;
  const int b = blockIdx.y;
  const int row0 = blockIdx.x * ROWS;
  const int lr = tid / P, p = tid % P;
  const int row = row0 + lr;
  const bool valid = row < ny;
  const long long D = (long long)ny * N;
  init_tw_s2<P, Q>(t2, tid, T);
  float2 acc[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = make_float2(0.f, 0.f);
  // coils [jb, je) of this CTA; with several coil groups (small batches) the CTA leaves its raw
  // partial sum in coil jb's rows of the workspace (rows only it reads) for k_rowinv_sum
  const int jb = blockIdx.z * cpg, je = min(ncoils, jb + cpg);
  const float2* mb = maps + b * map_bstride + (long long)row * N + p;
  float2* wb = ws + (long long)b * ncoils * D + (long long)row0 * N;
  const int nvalid = min(ROWS, ny - row0) * N;
  // Coil tiles are double-buffered.  BULK: every row of the tile is one bulk-async copy global ->
  // shared on the TMA unit (no register staging, no per-element LDGSTS), completing on the
  // buffer's mbarrier; otherwise 16-byte (even P) or 8-byte cp.async.
  __shared__ __align__(8) uint64_t tbar[2];
  const int nrows = min(ROWS, ny - row0);
  if constexpr (BULK) {
    if (tid == 0) {
      mbar_init(&tbar[0], 1);
      mbar_init(&tbar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  auto issue_tile = [&](int j) {
    const float2* wj = wb + j * D;
    float2* dst = bufs + (j & 1) * (ROWS * S::VS);
    if constexpr (BULK) {
      // the buffer was last read through the generic proxy (previous coil, behind a barrier)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (tid == 0) mbar_arrive_expect(&tbar[j & 1], (unsigned)(nrows * N * 8));
      if (tid < nrows) bulk_g2s(dst + tid * S::VS, wj + (long long)tid * N, N * 8, &tbar[j & 1]);
    } else if constexpr (S::VEC) {
      for (int e = 2 * tid; e < nvalid; e += 2 * T) {
        const int l3 = e / N, pos = e - l3 * N;
        cp_async16(dst + l3 * S::VS + S::pad(pos), wj + e);
      }
      cp_async_commit();
    } else {
      for (int e = tid; e < nvalid; e += T) {
        const int l3 = e / N, pos = e - l3 * N;
        cp_async8(dst + l3 * S::VS + S::pad(pos), wj + e);
      }
      cp_async_commit();
    }
  };
  issue_tile(jb);
  for (int j = jb; j < je; ++j) {
    if (j + 1 < je) issue_tile(j + 1);
    if constexpr (BULK) {
      mbar_wait(&tbar[j & 1], ((j - jb) >> 1) & 1);
    } else {
      if (j + 1 < je) cp_async_wait<1>();
      else cp_async_wait<0>();
    }
    __syncthreads();
    float2* buf = bufs + (j & 1) * (ROWS * S::VS);
    float2 mreg[Q];
    {
      const float2* mr = mb + j * D;
#pragma unroll
      for (int q = 0; q < Q; ++q) mreg[q] = valid ? __ldg(mr + P * q) : make_float2(0.f, 0.f);
    }
    if (P > 1) {
      for (int it = tid; it < ROWS * Q; it += T) {
        const int l2 = it / Q, k2 = it - l2 * Q;
        float2 g[P];
        float2* gp = buf + l2 * S::VS + S::GS * k2;
        lds_group<P, S::VEC>(g, gp);
        fft_s2_inv<P, Q>(g, k2, t2);
        sts_group<P, S::VEC>(gp, g);
      }
      __syncthreads();
    }
    float2 r[Q];
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) r[k2] = buf[lr * S::VS + S::GS * k2 + p];
    fft_s1_inv<Q>(r);
#pragma unroll
    for (int q = 0; q < Q; ++q) cfma_conj(acc[q], mreg[q], r[q]);
    __syncthreads();  // buf (j & 1) is refilled by the prefetch issued next iteration
  }
  if (!valid) return;
  if (gridDim.z > 1) {
    float2* pr = wb + jb * D + (long long)lr * N + p;
#pragma unroll
    for (int q = 0; q < Q; ++q) pr[P * q] = acc[q];
    return;
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = cscale(acc[q], oscale);  // 1/D of the unitary FFT pair
  const long long off = b * x_bstride + (long long)row * N + p;
  if (coef == nullptr) {
#pragma unroll
    for (int q = 0; q < Q; ++q) out[off + P * q] = acc[q];
  } else {
    const float4 c = coef[b];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      float2 v = cscale(acc[q], c.x);
      if (u) { const float2 uu = u[off + P * q]; v.x = fmaf(c.y, uu.x, v.x); v.y = fmaf(c.y, uu.y, v.y); }
      if (d) { const float2 dd = d[off + P * q]; v.x = fmaf(c.z, dd.x, v.x); v.y = fmaf(c.z, dd.y, v.y); }
      out[off + P * q] = v;
    }
  }
}

// ------------------------------------------------------------------- pass B

#ifndef SR_COL_CB16
#define SR_COL_CB16 16  // columns per CTA of the column pass for P >= 16
#endif
template <int P, int Q>
struct ColCfg {
  static constexpr int CB = (P >= 16) ? SR_COL_CB16 : (P >= 4 ? 32 : 64);
  static constexpr int T = CB * P;
  static constexpr int VSP = FftShape<P, Q>::VS0 | 1;  // odd stride: conflict-free over columns
};

// NXC > 0: row length known at compile time (square images) -> immediate address offsets
template <int P, int Q, int NXC>
__global__ void __launch_bounds__(ColCfg<P, Q>::T)
k_colpass(float2* __restrict__ ws, const uint8_t* __restrict__ maskT, long long mask_bstride,
          float mscale, int mode, int nx_rt, int ncoils, SampleIO sio) {
  using S = FftShape<P, Q>;
  constexpr int N = S::N, CB = ColCfg<P, Q>::CB, T = ColCfg<P, Q>::T, VSP = ColCfg<P, Q>::VSP;
  constexpr bool FULL = NXC > 0 && (NXC % CB) == 0;  // every column block is complete
  const int nx = NXC > 0 ? NXC : nx_rt;
  extern __shared__ float2 smem[];
  float2* t1 = smem;
  float2* t2 = smem + N;
  float2* buf = smem + 2 * N;
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * CB;
  const int j = blockIdx.y, b = blockIdx.z;
  const long long D = (long long)nx * N;
  float2* img = ws + ((long long)b * ncoils + j) * D;
  const int ncols = FULL ? CB : min(CB, nx - c0);
  init_tw_s1<P, Q>(t1, tid, T);
  init_tw_s2<P, Q>(t2, tid, T);
  __syncthreads();
  const int c = tid % CB, p = tid / CB;
  const bool cvalid = FULL || c < ncols;
  const bool inv_only = (mode == COL_INV || mode == COL_INV_S);
  const bool fwd_only = (mode == COL_FWD || mode == COL_FWD_G);

  if (mode == COL_INV) {
    // spectrum in perm order along y -> smem
    for (int e = tid; e < CB * N; e += T) {
      const int cc = e % CB, pos = e / CB;
      if (cc < ncols) buf[cc * VSP + S::pad(pos)] = img[(long long)pos * nx + c0 + cc];
    }
    __syncthreads();
  } else if (mode == COL_INV_S) {
    // adjoint sample scatter straight into the zeroed strip (no workspace memset / scatter pass)
    for (int e = tid; e < CB * VSP; e += T) buf[e] = make_float2(0.f, 0.f);
    __syncthreads();
    const long long s0 = sio.soff[b];
    const int* bp = sio.bptr + (long long)b * (sio.nblk + 1) + blockIdx.x;
    const long long yo = ((long long)b * ncoils + j) * sio.ystride;
    for (int t = bp[0] + tid; t < bp[1]; t += T) {
      const int i = sio.bidx[t];
      const int sp = sio.spos[s0 + i];
      const int py = sp / nx, cx = sp - py * nx - c0;
      buf[cx * VSP + S::pad(py)] = cscale(cmulc(sio.ph[s0 + i], sio.yin[yo + i]), sio.scale);
    }
    __syncthreads();
  } else {
    // forward step 1 straight from global (coalesced over columns)
    float2 r[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q)
      r[q] = cvalid ? img[(long long)(p + P * q) * nx + c0 + c] : make_float2(0.f, 0.f);
    fft_s1_fwd<P, Q>(r, p, t1);
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) buf[c * VSP + S::GS * k2 + p] = r[k2];
    __syncthreads();
  }

  // step 2 (forward and/or inverse) per (column, k2) group
  const uint8_t* mcol = (mode == COL_NORMAL) ? maskT + b * mask_bstride : nullptr;
  for (int it = tid; it < CB * Q; it += T) {
    const int cc = it % CB, k2 = it / CB;
    if (cc >= ncols) continue;
    float2 g[P];
    float2* gp = buf + cc * VSP + S::GS * k2;
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) g[k1] = gp[k1];
    if (!inv_only) fft_s2_fwd<P>(g);
    if (mode == COL_NORMAL) {
      const uint8_t* mk = mcol + (long long)(c0 + cc) * N + P * k2;
      if ((P % 4) == 0) {
#pragma unroll
        for (int w4 = 0; w4 < P / 4; ++w4) {
          const uint32_t m4 = __ldg(reinterpret_cast<const uint32_t*>(mk) + w4);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const bool keep = (m4 >> (8 * i)) & 0xffu;
            g[4 * w4 + i] = keep ? g[4 * w4 + i] : make_float2(0.f, 0.f);
          }
        }
        if (mscale != 1.f) {
#pragma unroll
          for (int k1 = 0; k1 < P; ++k1) g[k1] = cscale(g[k1], mscale);
        }
      } else {
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) g[k1] = cscale(g[k1], mk[k1] ? mscale : 0.f);
      }
    }
    if (!fwd_only) fft_s2_inv<P, Q>(g, k2, t2);
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) gp[k1] = g[k1];
  }
  __syncthreads();

  if (mode == COL_FWD) {
    for (int e = tid; e < CB * N; e += T) {
      const int cc = e % CB, pos = e / CB;
      if (cc < ncols) img[(long long)pos * nx + c0 + cc] = buf[cc * VSP + S::pad(pos)];
    }
    return;
  }
  if (mode == COL_FWD_G) {
    // forward sample gather straight from the strip (no workspace write / gather pass);
    // residual y - ymeas and its squared norm per block (deterministic tree reduction)
    const long long s0 = sio.soff[b];
    const int* bp = sio.bptr + (long long)b * (sio.nblk + 1) + blockIdx.x;
    const long long yo = ((long long)b * ncoils + j) * sio.ystride;
    double acc = 0.0;
    for (int t = bp[0] + tid; t < bp[1]; t += T) {
      const int i = sio.bidx[t];
      const int sp = sio.spos[s0 + i];
      const int py = sp / nx, cx = sp - py * nx - c0;
      float2 v = cscale(cmul(sio.ph[s0 + i], buf[cx * VSP + S::pad(py)]), sio.scale);
      if (sio.ymeas) {
        v = csub(v, sio.ymeas[yo + i]);
        acc += (double)v.x * v.x + (double)v.y * v.y;
      }
      sio.y[yo + i] = v;
    }
    if (sio.partial) {
      __syncthreads();  // strip no longer read: reuse it for the reduction
      double* red = reinterpret_cast<double*>(buf);
      constexpr int T2 = pow2_floor(T);  // fold the tail above the largest power of two first
      red[tid] = acc;
      __syncthreads();
      if (tid >= T2) red[tid - T2] += red[tid];
      __syncthreads();
      for (int st = T2 / 2; st > 0; st >>= 1) {
        if (tid < st) red[tid] += red[tid + st];
        __syncthreads();
      }
      if (tid == 0) sio.partial[((long long)b * ncoils + j) * sio.pblocks + blockIdx.x] = red[0];
    }
    return;
  }
  // inverse step 1' -> natural order along y, straight to global
  float2 r[Q];
#pragma unroll
  for (int k2 = 0; k2 < Q; ++k2) r[k2] = buf[c * VSP + S::GS * k2 + p];
  fft_s1_inv<Q>(r);
  if (cvalid) {
#pragma unroll
    for (int q = 0; q < Q; ++q) img[(long long)(p + P * q) * nx + c0 + c] = r[q];
  }
}

// Column pass of the normal operator, several coils per CTA: the mask words of the
// CTA's (column, k2) groups are loaded once, and coil j+1's column strip is loaded into
// registers while coil j is transformed (the load latency is hidden behind steps 2/3).
// Requires CB * Q <= T (one step-2 group per thread) and full column blocks.
template <int P, int Q, int NXC, bool PF>
__global__ void __launch_bounds__(ColCfg<P, Q>::T, PF ? 2 : 3)
k_colnormal(float2* __restrict__ ws, const uint8_t* __restrict__ maskT, long long mask_bstride,
            int ncoils, int jc) {
  using S = FftShape<P, Q>;
  constexpr int N = S::N, CB = ColCfg<P, Q>::CB, T = ColCfg<P, Q>::T, VSP = ColCfg<P, Q>::VSP;
  constexpr int NX = NXC;
  static_assert(NX % CB == 0 && CB * Q <= T && (P % 4) == 0, "k_colnormal shape");
  constexpr long long D = (long long)NX * N;
  extern __shared__ float2 smem[];
  float2* t1 = smem;
  float2* t2 = smem + N;
  float2* buf = smem + 2 * N;
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * CB;
  const int j0 = blockIdx.y * jc, j1 = min(ncoils, j0 + jc);
  const int b = blockIdx.z;
  init_tw_s1<P, Q>(t1, tid, T);
  init_tw_s2<P, Q>(t2, tid, T);
  const int c = tid % CB, p = tid / CB;
  // step-2 task of this thread: column cc, group k2
  const int cc = tid % CB, k2 = tid / CB;
  const bool s2 = tid < CB * Q;
  uint32_t mw[P / 4];
  {
    const uint32_t* mk = reinterpret_cast<const uint32_t*>(maskT + b * mask_bstride +
                                                           (long long)(c0 + cc) * N + P * k2);
#pragma unroll
    for (int w4 = 0; w4 < P / 4; ++w4) mw[w4] = s2 ? __ldg(mk + w4) : 0u;
  }
  float2* img0 = ws + ((long long)b * ncoils) * D + (long long)p * NX + c0 + c;
  float2 rn[PF ? Q : 1];
  if constexpr (PF) {
#pragma unroll
    for (int q = 0; q < Q; ++q) rn[q] = img0[j0 * D + (long long)(P * q) * NX];
  }
  __syncthreads();
  for (int j = j0; j < j1; ++j) {
    float2* img = img0 + j * D;
    float2 r[Q];
    if constexpr (PF) {
#pragma unroll
      for (int q = 0; q < Q; ++q) r[q] = rn[q];
    } else {
#pragma unroll
      for (int q = 0; q < Q; ++q) r[q] = img[(long long)(P * q) * NX];
    }
    fft_s1_fwd<P, Q>(r, p, t1);
#pragma unroll
    for (int kk = 0; kk < Q; ++kk) buf[c * VSP + S::GS * kk + p] = r[kk];
    if (PF && j + 1 < j1) {
#pragma unroll
      for (int q = 0; q < Q; ++q) rn[q] = img[D + (long long)(P * q) * NX];
    }
    __syncthreads();
    if (s2) {
      float2 g[P];
      float2* gp = buf + cc * VSP + S::GS * k2;
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) g[k1] = gp[k1];
      fft_s2_fwd<P>(g);
#pragma unroll
      for (int w4 = 0; w4 < P / 4; ++w4) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (!((mw[w4] >> (8 * i)) & 0xffu)) g[4 * w4 + i] = make_float2(0.f, 0.f);
      }
      fft_s2_inv<P, Q>(g, k2, t2);
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) gp[k1] = g[k1];
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < Q; ++kk) r[kk] = buf[c * VSP + S::GS * kk + p];
    fft_s1_inv<Q>(r);
#pragma unroll
    for (int q = 0; q < Q; ++q) img[(long long)(P * q) * NX] = r[q];
    __syncthreads();  // buf is rewritten by the next coil's step 1
  }
}

// ---------------------------------------------------------------- dispatch
// rowfwd output through TMA bulk stores: measured faster only for 20-element groups with
// Q >= 12 (320^2: 0.705 -> 0.680 ms; 256x160 / 384^2 / 640^2 slower) -> mode 2 (auto) picks
// those; 0 / 1 force the copy-out pass / the bulk stores (sr_cart_tune_rows)
template <int P, int Q>
int row_bulk() {
  if (P * Q < sr_g_row_bulk_min_n) return 0;
  if (sr_g_row_bulk == 2) return (P == 20 && Q >= 12) ? 1 : 0;
  return sr_g_row_bulk;
}

// coil groups for a row pass of `blocks` CTAs: small batches (config 0: one 256^2 slice = 32 row
// blocks) spread their coils over CTAs so the pass covers the SMs
inline int row_coil_groups(int blocks, int ncoils) {
  const int target = 2 * 148;
  if (blocks >= target) return 1;
  const int g = (target + blocks - 1) / blocks;
  return g < ncoils ? g : ncoils;
}

template <int P, int Q>
int launch_rowfwd(const float2* x, const float2* anchor, const float2* maps, float2* ws,
                  int batch, int ncoils, int ny, long long xbs, long long mbs, cudaStream_t st) {
  using R = RowCfg<P, Q>;
  static bool configured = false;
  static int carve = -2;
  if (!configured) {
    if (cudaFuncSetAttribute(k_rowfwd<P, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)R::SMEM_FWD) != cudaSuccess)
      return SR_ECUDA;
    configured = true;
  }
  const int blocks = (ny + R::ROWS - 1) / R::ROWS;
  const int groups = row_coil_groups(blocks * batch, ncoils);
  const int cpg = (ncoils + groups - 1) / groups;
  dim3 grid(blocks, batch, (ncoils + cpg - 1) / cpg);
  k_rowfwd<P, Q><<<grid, R::T, R::SMEM_FWD, st>>>(x, anchor, maps, ws, ncoils, ny, xbs, mbs,
                                                   row_bulk<P, Q>(), cpg);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

// coil-group partial sums (k_rowinv with gridDim.z > 1) -> out, fixed group order, + epilogue
__global__ void k_rowinv_sum(const float2* __restrict__ ws, float2* __restrict__ out, int ncoils, int cpg,
                             int ngroups, long long D, long long x_bstride, const float4* __restrict__ coef,
                             const float2* __restrict__ u, const float2* __restrict__ d, float oscale) {
  const int b = blockIdx.y;
  const float2* wb = ws + (long long)b * ncoils * D;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < D; e += (long long)gridDim.x * blockDim.x) {
    float2 a = wb[e];
    for (int g = 1; g < ngroups; ++g) a = cadd(a, wb[(long long)g * cpg * D + e]);
    a = cscale(a, oscale);
    const long long o = b * x_bstride + e;
    if (coef) {
      const float4 c = coef[b];
      a = cscale(a, c.x);
      if (u) { const float2 uu = u[o]; a.x = fmaf(c.y, uu.x, a.x); a.y = fmaf(c.y, uu.y, a.y); }
      if (d) { const float2 dd = d[o]; a.x = fmaf(c.z, dd.x, a.x); a.y = fmaf(c.z, dd.y, a.y); }
    }
    out[o] = a;
  }
}

template <int P, int Q>
int launch_rowinv(const float2* ws, const float2* maps, float2* out, int batch, int ncoils,
                  int ny, long long xbs, long long mbs, const float4* coef, const float2* u,
                  const float2* d, float oscale, cudaStream_t st) {
  using R = RowCfg<P, Q>;
  static bool configured = false;
  static int carve = -2;
  if (!configured) {
    if (cudaFuncSetAttribute(k_rowinv<P, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)R::SMEM_INV) != cudaSuccess)
      return SR_ECUDA;
    configured = true;
  }
  const int blocks = (ny + R::ROWS - 1) / R::ROWS;
  const int groups = row_coil_groups(blocks * batch, ncoils);
  const int cpg = (ncoils + groups - 1) / groups, ng = (ncoils + cpg - 1) / cpg;
  dim3 grid(blocks, batch, ng);
  k_rowinv<P, Q><<<grid, R::T, R::SMEM_INV, st>>>(const_cast<float2*>(ws), maps, out, ncoils, ny, xbs, mbs, coef,
                                                   u, d, oscale, cpg);
  SR_CHECK_LAUNCH();
  if (ng > 1) {
    const long long D = (long long)ny * P * Q;
    dim3 g2((unsigned)((D + 255) / 256 < 1024 ? (D + 255) / 256 : 1024), batch);
    k_rowinv_sum<<<g2, 256, 0, st>>>(ws, out, ncoils, cpg, ng, D, xbs, coef, u, d, oscale);
    SR_CHECK_LAUNCH();
  }
  return SR_OK;
}

template <int P, int Q, int NXC>
int launch_colpass_t(float2* ws, const uint8_t* maskT, long long mbs, float mscale, int mode,
                     int batch, int ncoils, int nx, cudaStream_t st, const SampleIO* sio) {
  using C = ColCfg<P, Q>;
  const size_t smem = sizeof(float2) * (2 * P * Q + C::CB * C::VSP);
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(k_colpass<P, Q, NXC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return SR_ECUDA;
    configured = true;
  }
  dim3 grid((nx + C::CB - 1) / C::CB, ncoils, batch);
  k_colpass<P, Q, NXC><<<grid, C::T, smem, st>>>(ws, maskT, mbs, mscale, mode, nx, ncoils,
                                                 sio ? *sio : SampleIO{});
  SR_CHECK_LAUNCH();
  return SR_OK;
}

template <int P, int Q, int NX, bool PF>
int launch_colnormal_t(float2* ws, const uint8_t* maskT, long long mbs, int batch, int ncoils, cudaStream_t st) {
  using C = ColCfg<P, Q>;
  const size_t smem = sizeof(float2) * (2 * P * Q + C::CB * C::VSP);
  static bool configured = false;
  static int carve = -2;
  if (!configured) {
    if (cudaFuncSetAttribute(k_colnormal<P, Q, NX, PF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return SR_ECUDA;
    configured = true;
  }
  if (apply_carveout(k_colnormal<P, Q, NX, PF>, carve)) return SR_ECUDA;
  int jc = sr_g_col_jc < ncoils ? sr_g_col_jc : ncoils;
  if ((NX / C::CB) * ((ncoils + jc - 1) / jc) * batch < 2 * 148) jc = 1;  // small batches: a coil per CTA
  dim3 grid(NX / C::CB, (ncoils + jc - 1) / jc, batch);
  k_colnormal<P, Q, NX, PF><<<grid, C::T, smem, st>>>(ws, maskT, mbs, ncoils, jc);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

template <int P, int Q, int NX>
int launch_colnormal(float2* ws, const uint8_t* maskT, long long mbs, int batch, int ncoils, cudaStream_t st) {
  if (sr_g_col_pf) return launch_colnormal_t<P, Q, NX, true>(ws, maskT, mbs, batch, ncoils, st);
  return launch_colnormal_t<P, Q, NX, false>(ws, maskT, mbs, batch, ncoils, st);
}

// non-square grids with a coil-looped column pass: (column length ny = P Q, row length nx)
// -- config 2's 256 x 160 readout-decoupled slices
#define SR_COLNORMAL_RECT(X) X(16, 16, 160)

template <int P, int Q>
int launch_colpass(float2* ws, const uint8_t* maskT, long long mbs, float mscale, int mode,
                   int batch, int ncoils, int nx, cudaStream_t st, const SampleIO* sio) {
  using C = ColCfg<P, Q>;
  if constexpr (P > 1 && (P % 4) == 0 && ((P * Q) % C::CB) == 0 && C::CB * Q <= C::T) {
    if (mode == COL_NORMAL && mscale == 1.f && sr_g_col_jc > 0) {
      if (nx == P * Q) return launch_colnormal<P, Q, P * Q>(ws, maskT, mbs, batch, ncoils, st);
#define X(P_, Q_, NX_)                                                                    \
      if constexpr (P == P_ && Q == Q_)                                                   \
        if (nx == NX_) return launch_colnormal<P_, Q_, NX_>(ws, maskT, mbs, batch, ncoils, st);
      SR_COLNORMAL_RECT(X)
#undef X
    }
  }
  if (nx == P * Q && P > 1)
    return launch_colpass_t<P, Q, P * Q>(ws, maskT, mbs, mscale, mode, batch, ncoils, nx, st, sio);
  // compile-time row length for the listed non-square grids too (immediate address offsets)
#define X(P_, Q_, NX_)                                                                                 \
  if constexpr (P == P_ && Q == Q_)                                                                    \
    if (nx == NX_) return launch_colpass_t<P_, Q_, NX_>(ws, maskT, mbs, mscale, mode, batch, ncoils, nx, st, sio);
  SR_COLNORMAL_RECT(X)
#undef X
  return launch_colpass_t<P, Q, 0>(ws, maskT, mbs, mscale, mode, batch, ncoils, nx, st, sio);
}

}  // namespace

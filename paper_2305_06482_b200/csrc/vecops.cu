// K7: solver vector kernels -- per-slice linear combinations and deterministic
// fixed-order reductions (no atomics, so results are bit-reproducible).
//
// Reference loops these serve:
//   fista            /root/reference/pkg/src/sketchrecon/solvers.py:290-297
//   _cg_loop         /root/reference/pkg/src/sketchrecon/solvers.py:206-229
//   max_eig_power    /root/reference/pkg/src/sketchrecon/linops.py:766-782
// All scalars stay on the device (per-slice arrays) so an inner loop never
// synchronises with the host.
#include "common.cuh"

namespace {

constexpr int RED_THREADS = 256;
// Partial sums per slice: a function of the vector length only (>= 2048 elements per block, 16..592
// blocks), so a reduction is deterministic and independent of the batch, and a single long vector
// (config 4: 84 MB images, 2.4 GB sample arrays) is read by the whole GPU -- 64 blocks per slice read
// such a vector at ~1 TB/s.  Callers size their partial buffers with sr_reduce_nparts() (the maximum).
constexpr int RED_BLOCKS_MAX = 592;
static inline int red_blocks(long long n) {
  const long long nb = n / 2048;
  return (int)(nb < 16 ? 16 : (nb > RED_BLOCKS_MAX ? RED_BLOCKS_MAX : nb));
}

enum { RED_NORM2 = 0, RED_DOT = 1, RED_ABS = 2, RED_DIFF2 = 3 };

// result[b] = (re, im) of the reduction of slice b.
__global__ void __launch_bounds__(RED_THREADS)
k_reduce_partial(int mode, const float2* __restrict__ a, const float2* __restrict__ bv,
                 long long n, long long bstride, double2* __restrict__ partial) {
  const int b = blockIdx.y;
  const float2* ab = a + b * bstride;
  const float2* bb = bv ? bv + b * bstride : nullptr;
  // contiguous chunk per block
  const long long chunk = (n + gridDim.x - 1) / gridDim.x;
  const long long lo = blockIdx.x * chunk;
  const long long hi = min(n, lo + chunk);
  double sr = 0.0, si = 0.0;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const float2 x = ab[i];
    if (mode == RED_NORM2) {
      sr += (double)x.x * x.x + (double)x.y * x.y;
    } else if (mode == RED_DOT) {  // sum conj(a) * b
      const float2 y = bb[i];
      sr += (double)x.x * y.x + (double)x.y * y.y;
      si += (double)x.x * y.y - (double)x.y * y.x;
    } else if (mode == RED_ABS) {
      sr += sqrt((double)x.x * x.x + (double)x.y * x.y);
    } else {  // RED_DIFF2
      const float2 y = bb[i];
      const double dx = (double)x.x - y.x, dy = (double)x.y - y.y;
      sr += dx * dx + dy * dy;
    }
  }
  __shared__ double rr[RED_THREADS], ri[RED_THREADS];
  rr[threadIdx.x] = sr;
  ri[threadIdx.x] = si;
  __syncthreads();
  for (int s = RED_THREADS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      rr[threadIdx.x] += rr[threadIdx.x + s];
      ri[threadIdx.x] += ri[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[(long long)b * gridDim.x + blockIdx.x] = make_double2(rr[0], ri[0]);
}

__global__ void k_reduce_final(const double2* __restrict__ partial, int nparts, int batch,
                               double2* __restrict__ result) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  double sr = 0.0, si = 0.0;
  for (int k = 0; k < nparts; ++k) {
    sr += partial[(long long)b * nparts + k].x;
    si += partial[(long long)b * nparts + k].y;
  }
  result[b] = make_double2(sr, si);
}

// out = c.x * X + c.y * Y + c.z * Z  (per-slice real coefficients; Y/Z nullable)
__global__ void k_lincomb(float2* __restrict__ out, const float2* __restrict__ X,
                          const float2* __restrict__ Y, const float2* __restrict__ Z,
                          const float4* __restrict__ coef, float4 hcoef, long long n,
                          long long bstride) {
  const int b = blockIdx.y;
  const float4 c = coef ? coef[b] : hcoef;
  const long long o = b * bstride;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float2 x = X[o + i];
    float2 v = make_float2(c.x * x.x, c.x * x.y);
    if (Y) { const float2 y = Y[o + i]; v.x = fmaf(c.y, y.x, v.x); v.y = fmaf(c.y, y.y, v.y); }
    if (Z) { const float2 z = Z[o + i]; v.x = fmaf(c.z, z.x, v.x); v.y = fmaf(c.z, z.y, v.y); }
    out[o + i] = v;
  }
}

// Scalar bookkeeping kernels (one thread per slice) -------------------------
enum {
  SC_POWER = 0,     // in0 = (|w|^2, .), in1 = <v, w>: lam = Re in1; coef = (1/|w|, 0, 0); flag |w| == 0
  SC_CG_ALPHA = 1,  // in0 = rs (re), in1 = <p, Mp>: alpha = rs / denom; coefX = (1, alpha, 0), coefR = (1, -alpha, 0)
  SC_CG_BETA = 2,   // in0 = rs_new, state.rs_old: beta = rs_new / rs_old; coef = (1, beta, 0)
};

__global__ void k_scalar(int op, const double2* __restrict__ in0, const double2* __restrict__ in1,
                         double* __restrict__ state, float4* __restrict__ coefA,
                         float4* __restrict__ coefB, int* __restrict__ flags, int batch) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  if (op == SC_POWER) {
    const double nw = sqrt(in0[b].x);
    if (nw == 0.0) {
      flags[b] = 1;
      state[b] = 0.0;
      coefA[b] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else if (!flags[b]) {
      state[b] = in1[b].x;  // lam = Re <v, w>
      coefA[b] = make_float4((float)(1.0 / nw), 0.f, 0.f, 0.f);
    } else {
      coefA[b] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  } else if (op == SC_CG_ALPHA) {
    // state layout per slice: [rs, active]
    const double rs = state[2 * b];
    const double denom = in1[b].x;
    const bool active = state[2 * b + 1] != 0.0 && denom > 0.0;
    if (!active) state[2 * b + 1] = 0.0;
    const double alpha = active ? rs / denom : 0.0;
    coefA[b] = make_float4(1.f, (float)alpha, 0.f, 0.f);
    coefB[b] = make_float4(1.f, (float)(-alpha), 0.f, 0.f);
  } else if (op == SC_CG_BETA) {
    const double rs_new = in0[b].x;
    const double rs = state[2 * b];
    const bool active = state[2 * b + 1] != 0.0;
    const double beta = (active && rs != 0.0) ? rs_new / rs : 0.0;
    if (active) state[2 * b] = rs_new;
    // p = r + beta p (inactive slices keep p: coef (0, 1))
    coefA[b] = active ? make_float4(1.f, (float)beta, 0.f, 0.f) : make_float4(0.f, 1.f, 0.f, 0.f);
  }
}

// ---------------------------------------------------------------- fused CG (K7)
// One conjugate-gradient iteration of _cg_loop (solvers.py:206-229) for B independent slices,
// after the matvec mp = M p, in three launches (k_reduce_partial <p, mp>, k_cg_xr, k_cg_p)
// instead of two reductions, two scalar kernels and three linear combinations.  Per-slice
// state (double): [rs(0), rs(1), active, iterations]; rs ping-pongs on the iteration parity
// so no block overwrites a value another block of the same launch still reads.  Every block
// of a slice reduces the slice's partials itself in the same fixed order, so the decisions and
// coefficients are identical in all blocks and the results are bit-reproducible.
__device__ __forceinline__ double2 sum_parts(const double2* __restrict__ part, int nparts) {
  __shared__ double2 s_sum;
  if (threadIdx.x == 0) {
    double sr = 0.0, si = 0.0;
    for (int k = 0; k < nparts; ++k) {
      sr += part[k].x;
      si += part[k].y;
    }
    s_sum = make_double2(sr, si);
  }
  __syncthreads();
  return s_sum;
}

// alpha = rs / <p, mp> (if active, <p, mp> > 0 and sqrt(rs) > tol); x += alpha p; r -= alpha mp;
// per-block partials of |r|^2
__global__ void __launch_bounds__(RED_THREADS)
k_cg_xr(float2* __restrict__ x, float2* __restrict__ r, const float2* __restrict__ p,
        const float2* __restrict__ mp, const double2* __restrict__ pdot, double* __restrict__ state,
        double2* __restrict__ prs, long long n, long long bstride, int parity, double tol_abs) {
  const int b = blockIdx.y;
  double* stb = state + 4 * (long long)b;
  const double2 dn = sum_parts(pdot + (long long)b * gridDim.x, gridDim.x);
  const double rs = stb[parity];
  const bool go = stb[2] != 0.0 && sqrt(rs) > tol_abs;
  const bool upd = go && dn.x > 0.0;
  const float alpha = upd ? (float)(rs / dn.x) : 0.f;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (go) stb[3] += 1.0;       // iterations entered (a denominator break still counts, as in the reference)
    if (!upd) stb[2] = 0.0;      // the reference breaks: this slice keeps x and r from here on
  }
  const long long chunk = (n + gridDim.x - 1) / gridDim.x;
  const long long lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  const long long o = b * bstride;
  double sr = 0.0;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    float2 rv = r[o + i];
    if (upd) {
      const float2 pv = p[o + i], mv = mp[o + i];
      float2 xv = x[o + i];
      xv.x = fmaf(alpha, pv.x, xv.x);
      xv.y = fmaf(alpha, pv.y, xv.y);
      x[o + i] = xv;
      rv.x = fmaf(-alpha, mv.x, rv.x);
      rv.y = fmaf(-alpha, mv.y, rv.y);
      r[o + i] = rv;
    }
    sr += (double)rv.x * rv.x + (double)rv.y * rv.y;
  }
  __shared__ double rr[RED_THREADS];
  rr[threadIdx.x] = sr;
  __syncthreads();
  for (int s = RED_THREADS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) rr[threadIdx.x] += rr[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) prs[(long long)b * gridDim.x + blockIdx.x] = make_double2(rr[0], 0.0);
}

// rs_new = |r|^2; beta = rs_new / rs; p = r + beta p (active slices); rs -> the other parity slot;
// hist[it] = sqrt(rs_new) if hist is given (the residual history of _cg_loop)
__global__ void __launch_bounds__(RED_THREADS)
k_cg_p(float2* __restrict__ p, const float2* __restrict__ r, const double2* __restrict__ prs,
       double* __restrict__ state, double* __restrict__ hist, int hist_len, long long n, long long bstride,
       int parity) {
  const int b = blockIdx.y;
  double* stb = state + 4 * (long long)b;
  const double rs_new = sum_parts(prs + (long long)b * gridDim.x, gridDim.x).x;
  const double rs = stb[parity];
  const bool act = stb[2] != 0.0;
  const float beta = (act && rs != 0.0) ? (float)(rs_new / rs) : 0.f;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    stb[parity ^ 1] = act ? rs_new : rs;
    if (act && hist) {
      const int it = (int)stb[3];
      if (it >= 1 && it <= hist_len) hist[(long long)b * (hist_len + 1) + it] = sqrt(rs_new);
    }
  }
  if (!act) return;
  const long long chunk = (n + gridDim.x - 1) / gridDim.x;
  const long long lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  const long long o = b * bstride;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const float2 rv = r[o + i];
    float2 pv = p[o + i];
    pv.x = fmaf(beta, pv.x, rv.x);
    pv.y = fmaf(beta, pv.y, rv.y);
    p[o + i] = pv;
  }
}

}  // namespace

extern "C" {

int sr_reduce_nparts(void) { return RED_BLOCKS_MAX; }

// Fused CG vector step (see k_cg_xr / k_cg_p): after mp = M p.  pdot, prs: (batch, sr_reduce_nparts())
// double2 scratch; state: (batch, 4) double [rs0, rs1, active, iterations] initialised by the
// caller (rs0 = |r0|^2, active = 1, iterations = 0); parity = iteration index & 1; hist: NULL or
// (batch, hist_len + 1) doubles receiving sqrt(rs) after iteration it at [it].
int sr_cg_step(sr_c64* x, sr_c64* r, sr_c64* p, const sr_c64* mp, double* pdot, double* prs, double* state,
               double* hist, int hist_len, long long n, long long bstride, int batch, int parity,
               double tol_abs, void* stream) {
  if (n < 0 || batch < 1 || !x || !r || !p || !mp || !pdot || !prs || !state || (parity & ~1)) return SR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int nblk = red_blocks(n);
  dim3 grid(nblk, batch);
  k_reduce_partial<<<grid, RED_THREADS, 0, st>>>(RED_DOT, (const float2*)p, (const float2*)mp, n, bstride,
                                                 (double2*)pdot);
  SR_CHECK_LAUNCH();
  k_cg_xr<<<grid, RED_THREADS, 0, st>>>((float2*)x, (float2*)r, (const float2*)p, (const float2*)mp,
                                        (const double2*)pdot, state, (double2*)prs, n, bstride, parity, tol_abs);
  SR_CHECK_LAUNCH();
  k_cg_p<<<grid, RED_THREADS, 0, st>>>((float2*)p, (const float2*)r, (const double2*)prs, state, hist, hist_len,
                                       n, bstride, parity);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

// partial: (batch, sr_reduce_nparts()) double2 workspace; result: (batch,) double2
int sr_reduce(int mode, const sr_c64* a, const sr_c64* b, long long n, long long bstride,
              int batch, double* partial, double* result, void* stream) {
  if (n < 0 || batch < 1 || mode < 0 || mode > 3) return SR_EINVAL;
  if ((mode == RED_DOT || mode == RED_DIFF2) && b == nullptr) return SR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int nblk = red_blocks(n);
  dim3 grid(nblk, batch);
  k_reduce_partial<<<grid, RED_THREADS, 0, st>>>(mode, (const float2*)a, (const float2*)b, n,
                                                 bstride, (double2*)partial);
  SR_CHECK_LAUNCH();
  k_reduce_final<<<(batch + 127) / 128, 128, 0, st>>>((const double2*)partial, nblk, batch,
                                                      (double2*)result);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

// coef: device (batch, 4) floats or NULL -> host coefficients (cx, cy, cz) for every slice
int sr_lincomb(sr_c64* out, const sr_c64* X, const sr_c64* Y, const sr_c64* Z,
               const float* coef, float cx, float cy, float cz, long long n,
               long long bstride, int batch, void* stream) {
  if (n < 0 || batch < 1) return SR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 4) blocks = 148 * 4;
  if (blocks < 1) blocks = 1;
  dim3 grid((unsigned)blocks, batch);
  k_lincomb<<<grid, 256, 0, st>>>((float2*)out, (const float2*)X, (const float2*)Y,
                                  (const float2*)Z, (const float4*)coef,
                                  make_float4(cx, cy, cz, 0.f), n, bstride);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

int sr_scalar_op(int op, const double* in0, const double* in1, double* state, float* coefA,
                 float* coefB, int* flags, int batch, void* stream) {
  if (batch < 1 || op < 0 || op > 2) return SR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  k_scalar<<<(batch + 127) / 128, 128, 0, st>>>(op, (const double2*)in0, (const double2*)in1,
                                                state, (float4*)coefA, (float4*)coefB, flags,
                                                batch);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

}  // extern "C"

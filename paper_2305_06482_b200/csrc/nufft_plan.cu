// NUFFT plan construction on the device (host prep on the GPU).
//
// Reference: _GriddedNUFFTKernel._build_interpolator (linops.py:464-492) derives, per axis,
//   u = k * g / n,  base = ceil(u - w/2),  taps base + 0..w-1,  weight KB(u - col)
// in float64 and keeps a tap iff 1 - (2 d / w)^2 > 0 (linops.py:404-410).  The device plan
// stores the fp64-derived int32 tap base and a float32 offset t = u - base per axis; where a
// float32 offset would make a different support decision than the reference's float64 one
// (samples lying on a grid line up to 1e-16) it is moved by float32 ulps until every tap agrees
// -- the same rule as the host plan's support_safe_frac (nufft.py), so both plans are
// bit-identical (tests/test_gpu_parity.py::test_device_plan_equals_host_plan).
//
// The plan's sample order sorts by bin (binsize^d grid cells holding the first tap) and, inside
// a bin, by first-tap cell; the sort key is produced here, the stable sort itself is a library
// radix sort (torch.sort for the Python GriddedKernel; CUB DeviceRadixSort inside the opaque
// sr_nufft_plan of the C ABI, which also builds the grid, Beatty betas, apodisation and chunk
// list so that a non-Python caller needs nothing but this library).
#include "common.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cmath>
#include <vector>

namespace {

struct PlanDims {
  int n[3], g[3], nbins[3];
};

__global__ void k_plan_geom(const double* __restrict__ pts, long long N, int nd, PlanDims pd, int w, int B,
                            int* __restrict__ base3, float* __restrict__ frac3, long long* __restrict__ key,
                            int* __restrict__ err) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int pad = 3 - nd;
  long long binid = 0, local = 0;
  for (int a = 0; a < nd; ++a) {
    const int n = pd.n[a], g = pd.g[a];
    // Trajectory.validate_for (linops.py:130-140): coordinates in [-n/2, n/2)
    const double pv = pts[i * nd + a];
    if (!(pv >= -0.5 * n) || !(pv < 0.5 * n)) atomicExch(err, 1);
    const double u = pv * ((double)g / (double)n);
    const double b = ceil(u - (double)w / 2.0);
    const double d = u - b;
    float t = __double2float_rn(d);
    // only offsets within a few float32 ulps of a support edge (t - k = +-w/2) can disagree
    if (fabs(d * 2.0 - rint(d * 2.0)) < 1e-5) {
      bool ok = false;
      for (int it = 0; it < 8 && !ok; ++it) {
        bool moved = false;
        for (int k = 0; k < w; ++k) {
          const double q = 2.0 * (u - (b + (double)k)) / (double)w;
          const bool ref = (1.0 - q * q) > 0.0;
          const bool dev = fabsf(__fdiv_rn(2.0f * (t - (float)k), (float)w)) < 1.0f;
          if (ref != dev) {
            float toward = ref ? ((float)k - t) : (t - (float)k);
            toward = (toward > 0.f) ? 1.f : (toward < 0.f ? -1.f : 1.f);
            t = nextafterf(t, toward > 0.f ? INFINITY : -INFINITY);
            moved = true;
          }
        }
        ok = !moved;
      }
      if (!ok) atomicExch(err, 1);
    }
    const long long bi = (long long)b;
    base3[(long long)(pad + a) * N + i] = (int)bi;
    frac3[(long long)(pad + a) * N + i] = t;
    long long bp = bi % g;
    if (bp < 0) bp += g;
    binid = binid * pd.nbins[a] + bp / B;
    local = local * B + bp % B;
  }
  for (int a = 0; a < pad; ++a) {
    base3[(long long)a * N + i] = 0;
    frac3[(long long)a * N + i] = 0.f;
  }
  long long bnd = 1;
  for (int a = 0; a < nd; ++a) bnd *= B;
  key[i] = binid * bnd + local;
}

__global__ void k_plan_permute(const int* __restrict__ base_in, const float* __restrict__ frac_in,
                               const long long* __restrict__ order, long long N, int* __restrict__ base_out,
                               float* __restrict__ frac_out, int* __restrict__ orig) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const long long s = order[i];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    base_out[a * N + i] = base_in[a * N + s];
    frac_out[a * N + i] = frac_in[a * N + s];
  }
  orig[i] = (int)s;
}

// --- opaque plan (sr_nufft_plan_create): sort by key, chunk list ------------------------------
constexpr int PLAN_CHUNK = 256;  // samples per chunk (BIN_CHUNK of nufft.cu)

__global__ void k_plan_iota(int* v, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int)i;
}

// bin start index of every position (for the max-scan) of the sorted keys
__global__ void k_plan_binstart(const long long* __restrict__ skey, long long n, long long bnd, int* __restrict__ bs) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bs[i] = (i == 0 || skey[i] / bnd != skey[i - 1] / bnd) ? (int)i : 0;
}

__global__ void k_plan_chunkflag(const int* __restrict__ binstart, long long n, int* __restrict__ flag) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  flag[i] = ((i - binstart[i]) % PLAN_CHUNK) == 0 ? 1 : 0;
}

__global__ void k_plan_chunks(const long long* __restrict__ skey, const int* __restrict__ flag,
                              const int* __restrict__ cpos, long long n, long long bnd, int nd, int B,
                              int nb0, int nb1, int nb2, int* __restrict__ chunks) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !flag[i]) return;
  const long long bid = skey[i] / bnd;
  int cnt = 1;
  while (cnt < PLAN_CHUNK && i + cnt < n && skey[i + cnt] / bnd == bid) ++cnt;
  long long r = bid;
  int c[3] = {0, 0, 0};
  const int nb[3] = {nb0, nb1, nb2};
  for (int a = 2; a >= 3 - nd; --a) {  // active axes padded to 3 (leading zeros for 2-D)
    c[a] = (int)(r % nb[a]) * B;
    r /= nb[a];
  }
  int* row = chunks + 5LL * cpos[i];
  row[0] = c[0];
  row[1] = c[1];
  row[2] = c[2];
  row[3] = (int)i;
  row[4] = cnt;
}

__global__ void k_plan_permute32(const int* __restrict__ base_in, const float* __restrict__ frac_in,
                                 const int* __restrict__ order, long long N, int* __restrict__ base_out,
                                 float* __restrict__ frac_out, int* __restrict__ orig) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int s = order[i];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    base_out[a * N + i] = base_in[a * N + s];
    frac_out[a * N + i] = frac_in[a * N + s];
  }
  orig[i] = s;
}

// w_sorted[i] = (w[orig[i]])^2 (normal op: density weight applied on both sides)
__global__ void k_plan_weights(const float* __restrict__ sqrtw, const int* __restrict__ orig, long long n,
                               float* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float v = sqrtw[orig[i]];
  out[i] = v * v;
}

}  // namespace

extern "C" {

int sr_nufft_plan_geom(const double* pts, long long nsamples, int ndim, const int* dims, const int* gdims,
                       int width, int binsize, int* base, float* frac, long long* key, int* err, void* stream) {
  if (nsamples < 0 || (ndim != 2 && ndim != 3) || width < 1 || width > 8 || binsize < 1 || !dims || !gdims)
    return SR_EINVAL;
  if (nsamples == 0) return SR_OK;
  if (!pts || !base || !frac || !key || !err) return SR_EINVAL;
  PlanDims pd{};
  for (int a = 0; a < ndim; ++a) {
    if (dims[a] < 1 || gdims[a] < 1) return SR_EINVAL;
    pd.n[a] = dims[a];
    pd.g[a] = gdims[a];
    pd.nbins[a] = (gdims[a] + binsize - 1) / binsize;
  }
  const int T = 256;
  k_plan_geom<<<(unsigned)((nsamples + T - 1) / T), T, 0, (cudaStream_t)stream>>>(pts, nsamples, ndim, pd, width,
                                                                                  binsize, base, frac, key, err);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

int sr_nufft_plan_permute(const int* base_in, const float* frac_in, const long long* order, long long nsamples,
                          int* base_out, float* frac_out, int* orig, void* stream) {
  if (nsamples < 0) return SR_EINVAL;
  if (nsamples == 0) return SR_OK;
  if (!base_in || !frac_in || !order || !base_out || !frac_out || !orig) return SR_EINVAL;
  const int T = 256;
  k_plan_permute<<<(unsigned)((nsamples + T - 1) / T), T, 0, (cudaStream_t)stream>>>(base_in, frac_in, order,
                                                                                     nsamples, base_out, frac_out,
                                                                                     orig);
  SR_CHECK_LAUNCH();
  return SR_OK;
}


// -------------------------------------------------------------------------- opaque plan
struct sr_nufft_plan {
  int ndim, width, binsize;
  int dims3[3], gdims3[3];  // leading 1s for 2-D
  float betas3[3];
  long long n, nchunks;
  int *base, *frac_i, *orig, *chunks;  // frac stored as float (frac_i reinterpreted)
  float* ia[3];
  float* wbuf;  // per-sample weights in sorted order (normal op)
};

int sr_nufft_normal(const sr_c64* x, const sr_c64* anchor, const sr_c64* maps, int ncoils, const int* dims,
                    const int* gdims, const float* betas, int width, const float* ia0, const float* ia1,
                    const float* ia2, const int* base, const float* frac, const float* wgt, long long nsamples,
                    sr_c64* out, sr_c64* grids, const float* coef, const sr_c64* u, const sr_c64* d,
                    const int* chunks, int nchunks, int binsize, void* stream);
int sr_fft_size_supported(int n);

static void plan_free(sr_nufft_plan* p) {
  if (!p) return;
  cudaFree(p->base);
  cudaFree(p->frac_i);
  cudaFree(p->orig);
  cudaFree(p->chunks);
  cudaFree(p->wbuf);
  for (int a = 0; a < 3; ++a) cudaFree(p->ia[a]);
  delete p;
}

// Builds the whole gridding plan on the device from a HOST float64 trajectory (N, ndim):
// oversampled grid (2 ceil(n os / 2), linops.py:438), Beatty beta (linops.py:440-445), inverse
// apodisation (linops.py:413-421, 447-452), tap geometry with the reference's float64 support
// decisions, stable radix sort by (bin, first-tap cell), chunk list.  Identical to the Python plan
// (GriddedKernel(plan="device"/"host")).  binsize 0 = 8 (3-D) / 16 (2-D).
int sr_nufft_plan_create(const double* pts, long long nsamples, int ndim, const int* dims, double oversamp,
                         int width, int binsize, sr_nufft_plan** out, void* stream) {
  if (!out || nsamples < 0 || (ndim != 2 && ndim != 3) || !dims || width < 1 || width > 8 || binsize < 0 ||
      !(oversamp >= 1.0) || (nsamples > 0 && !pts) || nsamples > 0x7fffffffLL)
    return SR_EINVAL;
  *out = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  sr_nufft_plan* p = new sr_nufft_plan{};
  p->ndim = ndim;
  p->width = width;
  p->binsize = binsize ? binsize : (ndim == 3 ? 8 : 16);
  p->n = nsamples;
  const int pad = 3 - ndim;
  int gd[3];
  for (int a = 0; a < 3; ++a) {
    p->dims3[a] = 1;
    p->gdims3[a] = 1;
    p->betas3[a] = 0.f;
  }
  for (int a = 0; a < ndim; ++a) {
    const int n = dims[a];
    if (n < 1) { plan_free(p); return SR_EINVAL; }
    const int g = (int)(std::ceil((double)n * oversamp / 2.0) * 2.0);
    if (!sr_fft_size_supported(g)) { plan_free(p); return SR_EUNSUPPORTED; }
    gd[a] = g;
    const double sc = (double)g / (double)n;
    const double wsc = (double)width / sc;
    const double beta = M_PI * std::sqrt(wsc * wsc * (sc - 0.5) * (sc - 0.5) - 0.8);
    p->dims3[pad + a] = n;
    p->gdims3[pad + a] = g;
    p->betas3[pad + a] = (float)beta;
    std::vector<float> ia((size_t)n);
    for (int i = 0; i < n; ++i) {
      const double r = (double)(i - n / 2) / (double)g;
      const double t = M_PI * width * r;
      const double z2 = beta * beta - t * t;
      const double z = std::sqrt(std::fabs(z2));
      double ap;
      if (z2 > 0) {
        ap = std::sinh(z) / z;
      } else {
        const double xx = z / M_PI;  // numpy sinc(x) = sin(pi x) / (pi x)
        ap = (xx == 0.0) ? 1.0 : std::sin(M_PI * xx) / (M_PI * xx);
      }
      ia[(size_t)i] = (float)(1.0 / (width * ap));
    }
    if (cudaMalloc(&p->ia[pad + a], sizeof(float) * n) != cudaSuccess ||
        cudaMemcpyAsync(p->ia[pad + a], ia.data(), sizeof(float) * n, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      plan_free(p);
      return SR_ECUDA;
    }
  }
  for (int a = 0; a < pad; ++a) {
    const float one = 1.f;
    if (cudaMalloc(&p->ia[a], sizeof(float)) != cudaSuccess ||
        cudaMemcpy(p->ia[a], &one, sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess) {
      plan_free(p);
      return SR_ECUDA;
    }
  }
  const long long N = nsamples;
  const size_t n3 = 3 * (size_t)(N > 0 ? N : 1);
  if (cudaMalloc(&p->base, sizeof(int) * n3) != cudaSuccess || cudaMalloc(&p->frac_i, sizeof(float) * n3) != cudaSuccess ||
      cudaMalloc(&p->orig, sizeof(int) * (N > 0 ? N : 1)) != cudaSuccess ||
      cudaMalloc(&p->wbuf, sizeof(float) * (N > 0 ? N : 1)) != cudaSuccess) {
    plan_free(p);
    return SR_ECUDA;
  }
  if (N == 0) {
    p->nchunks = 0;
    if (cudaMalloc(&p->chunks, 5 * sizeof(int)) != cudaSuccess) { plan_free(p); return SR_ECUDA; }
    *out = p;
    return SR_OK;
  }
  // scratch
  double* pts_d = nullptr;
  int *base_u = nullptr, *err = nullptr, *iota = nullptr, *order = nullptr, *bs = nullptr, *flag = nullptr,
      *cpos = nullptr;
  float* frac_u = nullptr;
  long long *key = nullptr, *skey = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int rc = SR_OK;
  const int T = 256;
  const unsigned nbk = (unsigned)((N + T - 1) / T);
  long long bnd = 1;
  for (int a = 0; a < ndim; ++a) bnd *= p->binsize;
  int nbins[3] = {1, 1, 1};
  for (int a = 0; a < ndim; ++a) nbins[pad + a] = (gd[a] + p->binsize - 1) / p->binsize;
  long long maxkey = bnd;
  for (int a = 0; a < 3; ++a) maxkey *= nbins[a];
  int end_bit = 1;
  while (end_bit < 63 && (1LL << end_bit) < maxkey) ++end_bit;
  do {
    if (cudaMalloc(&pts_d, sizeof(double) * N * ndim) != cudaSuccess ||
        cudaMalloc(&base_u, sizeof(int) * 3 * N) != cudaSuccess || cudaMalloc(&frac_u, sizeof(float) * 3 * N) != cudaSuccess ||
        cudaMalloc(&key, sizeof(long long) * N) != cudaSuccess || cudaMalloc(&skey, sizeof(long long) * N) != cudaSuccess ||
        cudaMalloc(&err, sizeof(int)) != cudaSuccess || cudaMalloc(&iota, sizeof(int) * N) != cudaSuccess ||
        cudaMalloc(&order, sizeof(int) * N) != cudaSuccess || cudaMalloc(&bs, sizeof(int) * N) != cudaSuccess ||
        cudaMalloc(&flag, sizeof(int) * N) != cudaSuccess || cudaMalloc(&cpos, sizeof(int) * N) != cudaSuccess) {
      rc = SR_ECUDA;
      break;
    }
    if (cudaMemcpyAsync(pts_d, pts, sizeof(double) * N * ndim, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemsetAsync(err, 0, sizeof(int), st) != cudaSuccess) {
      rc = SR_ECUDA;
      break;
    }
    rc = sr_nufft_plan_geom(pts_d, N, ndim, dims, gd, width, p->binsize, base_u, frac_u, key, err, st);
    if (rc) break;
    k_plan_iota<<<nbk, T, 0, st>>>(iota, N);
    // stable LSD radix sort of (key, sample index)
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key, skey, iota, order, (int)N, 0, end_bit, st);
    size_t scan_bytes = 0, scan2 = 0;
    cub::DeviceScan::InclusiveScan(nullptr, scan_bytes, bs, bs, cub::Max(), (int)N, st);
    cub::DeviceScan::ExclusiveSum(nullptr, scan2, flag, cpos, (int)N, st);
    if (scan_bytes > tmp_bytes) tmp_bytes = scan_bytes;
    if (scan2 > tmp_bytes) tmp_bytes = scan2;
    if (cudaMalloc(&tmp, tmp_bytes) != cudaSuccess) { rc = SR_ECUDA; break; }
    if (cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key, skey, iota, order, (int)N, 0, end_bit, st) != cudaSuccess) {
      rc = SR_ECUDA;
      break;
    }
    k_plan_permute32<<<nbk, T, 0, st>>>(base_u, frac_u, order, N, p->base, (float*)p->frac_i, p->orig);
    k_plan_binstart<<<nbk, T, 0, st>>>(skey, N, bnd, bs);
    if (cub::DeviceScan::InclusiveScan(tmp, tmp_bytes, bs, bs, cub::Max(), (int)N, st) != cudaSuccess) {
      rc = SR_ECUDA;
      break;
    }
    k_plan_chunkflag<<<nbk, T, 0, st>>>(bs, N, flag);
    if (cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flag, cpos, (int)N, st) != cudaSuccess) { rc = SR_ECUDA; break; }
    int last_pos = 0, last_flag = 0, herr = 0;
    if (cudaMemcpyAsync(&last_pos, cpos + N - 1, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(&last_flag, flag + N - 1, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      rc = SR_ECUDA;
      break;
    }
    if (herr) { rc = SR_EINVAL; break; }  // out-of-range coordinate, or float32 support decisions not aligned
    p->nchunks = (long long)last_pos + last_flag;
    if (cudaMalloc(&p->chunks, sizeof(int) * 5 * p->nchunks) != cudaSuccess) { rc = SR_ECUDA; break; }
    k_plan_chunks<<<nbk, T, 0, st>>>(skey, flag, cpos, N, bnd, ndim, p->binsize, nbins[0], nbins[1], nbins[2],
                                     p->chunks);
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) rc = SR_ECUDA;
  } while (false);
  cudaFree(pts_d);
  cudaFree(base_u);
  cudaFree(frac_u);
  cudaFree(key);
  cudaFree(skey);
  cudaFree(err);
  cudaFree(iota);
  cudaFree(order);
  cudaFree(bs);
  cudaFree(flag);
  cudaFree(cpos);
  cudaFree(tmp);
  if (rc) {
    plan_free(p);
    return rc;
  }
  *out = p;
  return SR_OK;
}

int sr_nufft_plan_destroy(sr_nufft_plan* plan) {
  if (!plan) return SR_EINVAL;
  plan_free(plan);
  return SR_OK;
}

// Plan geometry and device arrays (any output pointer may be NULL): gdims/dims/betas 3 entries
// (leading 1 / 0 for 2-D); base (3, N) int32, frac (3, N) float32, orig (N) int32, chunks
// (nchunks, 5) int32 -- the arrays sr_nufft_normal / _forward / _adjoint take.
int sr_nufft_plan_info(const sr_nufft_plan* plan, int* dims, int* gdims, float* betas, long long* nsamples,
                       long long* nchunks, const int** base, const float** frac, const int** orig,
                       const int** chunks, const float** ia0, const float** ia1, const float** ia2) {
  if (!plan) return SR_EINVAL;
  for (int a = 0; a < 3; ++a) {
    if (dims) dims[a] = plan->dims3[a];
    if (gdims) gdims[a] = plan->gdims3[a];
    if (betas) betas[a] = plan->betas3[a];
  }
  if (nsamples) *nsamples = plan->n;
  if (nchunks) *nchunks = plan->nchunks;
  if (base) *base = plan->base;
  if (frac) *frac = (const float*)plan->frac_i;
  if (orig) *orig = plan->orig;
  if (chunks) *chunks = plan->chunks;
  if (ia0) *ia0 = plan->ia[0];
  if (ia1) *ia1 = plan->ia[1];
  if (ia2) *ia2 = plan->ia[2];
  return SR_OK;
}

// Device-to-device copy on a stream (lets a caller copy the plan arrays into its own buffers).
int sr_memcpy_d2d(void* dst, const void* src, long long bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return SR_EINVAL;
  if (bytes == 0) return SR_OK;
  return cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream) == cudaSuccess
             ? SR_OK
             : SR_ECUDA;
}

// Sketched / full SENSE normal operator through a plan: sqrtw = sqrt of the density weights in
// TRAJECTORY order (device, NULL = 1), grids = 2 * ncoils * prod(gdims) complex64 workspace.
int sr_nufft_plan_normal(sr_nufft_plan* plan, const sr_c64* x, const sr_c64* anchor, const sr_c64* maps, int ncoils,
                         const float* sqrtw, sr_c64* out, sr_c64* grids, const float* coef, const sr_c64* u,
                         const sr_c64* d, void* stream) {
  if (!plan) return SR_EINVAL;
  const float* w = nullptr;
  if (sqrtw && plan->n > 0) {
    k_plan_weights<<<(unsigned)((plan->n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(sqrtw, plan->orig, plan->n,
                                                                                          plan->wbuf);
    SR_CHECK_LAUNCH();
    w = plan->wbuf;
  }
  return sr_nufft_normal(x, anchor, maps, ncoils, plan->dims3, plan->gdims3, plan->betas3, plan->width, plan->ia[0],
                         plan->ia[1], plan->ia[2], plan->base, (const float*)plan->frac_i, w, plan->n, out, grids,
                         coef, u, d, plan->chunks, (int)plan->nchunks, plan->binsize, stream);
}

}  // extern "C"

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
// radix sort (torch.sort on the device), the gather below applies it.
#include "common.cuh"

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
    const double u = pts[i * nd + a] * ((double)g / (double)n);
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

}  // extern "C"

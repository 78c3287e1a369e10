// Opaque Cartesian plan of the C ABI: the index / phase tables of plan.py (cartesian_plan) and
// cartesian.py (batch assembly, per-column-block sample lists) built by the library from a HOST
// float64 trajectory, so a caller without Python / torch can run K1 / K2 through plain pointers.
//
// Reference: _CartesianMaskKernel (linops.py:332-364): flat_idx = ravel_multi_index(points + n//2)
// (linops.py:341-342), the centered FFT pair (linops.py:300-313) and numpy fancy assignment in
// apply_adjoint (linops.py:357: the last duplicate wins).  The device keeps spectra in perm order
// (fft2step.cuh): a sample's perm-order offset spos, its centering phase ph = e^{2 pi i (n//2) f/n}
// per axis (which replaces the ifftshift / fftshift pair), the transposed mask maskT
// [pos_x][pos_y], the adjoint write list (last occurrence of every bin) and the per-column-block
// sample lists of the fused K2 column pass.  Identical to CartesianKernel's tables
// (tests/test_gpu_parity.py::test_opaque_cartesian_plan_equals_python_plan).
#include "common.cuh"

#include <cmath>
#include <vector>

extern "C" {
int sr_fft_split(int n, int* P, int* Q);
int sr_cart_col_block(int ny);
long long sr_cart_ws_bytes(int batch, int ncoils, int ny, int nx, int chunk);
}

struct sr_cart_plan {
  int batch, ny, nx, shared, nblk;
  long long nmax, total, wtotal;
  int* spos;
  float2* ph;
  long long *soff, *woff;
  int* wlist;
  uint8_t* maskT;
  int *g_ptr, *g_idx, *s_ptr, *s_idx;
};

namespace {

template <typename T>
int upload(T** dst, const std::vector<T>& src, cudaStream_t st) {
  const size_t n = src.empty() ? 1 : src.size();
  if (cudaMalloc(dst, sizeof(T) * n) != cudaSuccess) return SR_ECUDA;
  if (!src.empty() && cudaMemcpyAsync(*dst, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice, st) != cudaSuccess)
    return SR_ECUDA;
  return SR_OK;
}

void cart_plan_free(sr_cart_plan* p) {
  if (!p) return;
  cudaFree(p->spos);
  cudaFree(p->ph);
  cudaFree(p->soff);
  cudaFree(p->woff);
  cudaFree(p->wlist);
  cudaFree(p->maskT);
  cudaFree(p->g_ptr);
  cudaFree(p->g_idx);
  cudaFree(p->s_ptr);
  cudaFree(p->s_idx);
  delete p;
}

// perm position of frequency k of an axis of length n = P Q: P (k mod Q) + k / Q
bool perm_table(int n, std::vector<long long>& pos) {
  pos.assign((size_t)n, 0);
  if (n == 1) return true;
  int P = 0, Q = 0;
  if (sr_fft_split(n, &P, &Q) != SR_OK) return false;
  for (int k = 0; k < n; ++k) pos[(size_t)k] = (long long)P * (k % Q) + k / Q;
  return true;
}

}  // namespace

extern "C" {

// pts: HOST float64 (total, ndim) centered integer bins (the reference's Trajectory.points of a
// cartesian-mask trajectory), slices concatenated; counts: samples per slice (batch entries), or
// one entry with shared = 1 (one mask for every slice); ndim 1 or 2 (dims[0] = ny, dims[1] = nx).
int sr_cart_plan_create(const double* pts, const long long* counts, int batch, int ndim, const int* dims,
                        int shared, sr_cart_plan** out, void* stream) {
  if (!out || !counts || !dims || batch < 1 || (ndim != 1 && ndim != 2)) return SR_EINVAL;
  *out = nullptr;
  const int ny = ndim == 2 ? dims[0] : 1, nx = ndim == 2 ? dims[1] : dims[0];
  if (ny < 1 || nx < 2) return SR_EINVAL;
  std::vector<long long> py, px;
  if (!perm_table(ny, py) || !perm_table(nx, px)) return SR_EUNSUPPORTED;
  const int cb = sr_cart_col_block(ny);
  if (cb < 1) return SR_EUNSUPPORTED;
  const int nplans = shared ? 1 : batch;
  long long ptotal = 0;
  for (int b = 0; b < nplans; ++b) {
    if (counts[b] < 0) return SR_EINVAL;
    ptotal += counts[b];
  }
  if (ptotal > 0 && !pts) return SR_EINVAL;
  // Trajectory.validate_for (linops.py:130-140): every coordinate in [-n/2, n/2) per axis
  for (long long i = 0; i < ptotal; ++i) {
    for (int a = 0; a < ndim; ++a) {
      const double n = (double)(ndim == 2 && a == 0 ? ny : nx);
      const double v = pts[i * ndim + a];
      if (!(v >= -n / 2) || !(v < n / 2)) return SR_EINVAL;
    }
  }
  const long long D = (long long)ny * nx;
  const int nblk = (nx + cb - 1) / cb;
  // per distinct plan: tables in trajectory order
  struct Tab {
    std::vector<int> spos, wl, gidx, sidx;
    std::vector<float2> ph;
    std::vector<long long> gcnt, scnt;
  };
  std::vector<Tab> tabs((size_t)nplans);
  std::vector<uint8_t> maskT((size_t)(nplans * D), 0);
  long long off = 0;
  for (int b = 0; b < nplans; ++b) {
    Tab& t = tabs[(size_t)b];
    const long long n = counts[b];
    t.spos.resize((size_t)n);
    t.ph.resize((size_t)n);
    for (long long i = 0; i < n; ++i) {
      const double* pp = pts + (off + i) * ndim;
      const long long fy = ndim == 2 ? (long long)std::rint(pp[0]) : 0;
      const long long fx = (long long)std::rint(pp[ndim - 1]);
      const long long ky = ((fy % ny) + ny) % ny, kx = ((fx % nx) + nx) % nx;
      const long long pyv = py[(size_t)ky], pxv = px[(size_t)kx];
      t.spos[(size_t)i] = (int)(pyv * nx + pxv);
      // exp(2 pi i (n//2) f / n) per axis in float64 (plan.py), rounded once to float32
      double ang = 2.0 * M_PI * ((double)((long long)(ny / 2) * ky) / ny + (double)((long long)(nx / 2) * kx) / nx);
      ang = std::fmod(ang, 2.0 * M_PI);
      t.ph[(size_t)i] = make_float2((float)std::cos(ang), (float)std::sin(ang));
      maskT[(size_t)(b * D + pxv * ny + pyv)] = 1;
    }
    // adjoint write list: last occurrence of every bin, ascending
    std::vector<uint8_t> seen((size_t)D, 0);
    std::vector<int> rev;
    for (long long i = n - 1; i >= 0; --i) {
      const int s = t.spos[(size_t)i];
      if (!seen[(size_t)s]) {
        seen[(size_t)s] = 1;
        rev.push_back((int)i);
      }
    }
    t.wl.assign(rev.rbegin(), rev.rend());
    // per-column-block lists (stable counting sort by block)
    t.gcnt.assign((size_t)nblk, 0);
    t.scnt.assign((size_t)nblk, 0);
    for (long long i = 0; i < n; ++i) ++t.gcnt[(size_t)((t.spos[(size_t)i] % nx) / cb)];
    for (int i : t.wl) ++t.scnt[(size_t)((t.spos[(size_t)i] % nx) / cb)];
    std::vector<long long> gs((size_t)nblk + 1, 0), ss((size_t)nblk + 1, 0);
    for (int k = 0; k < nblk; ++k) {
      gs[(size_t)k + 1] = gs[(size_t)k] + t.gcnt[(size_t)k];
      ss[(size_t)k + 1] = ss[(size_t)k] + t.scnt[(size_t)k];
    }
    t.gidx.resize((size_t)n);
    t.sidx.resize(t.wl.size());
    std::vector<long long> gp(gs.begin(), gs.end() - 1), sp(ss.begin(), ss.end() - 1);
    for (long long i = 0; i < n; ++i) t.gidx[(size_t)gp[(size_t)((t.spos[(size_t)i] % nx) / cb)]++] = (int)i;
    for (int i : t.wl) t.sidx[(size_t)sp[(size_t)((t.spos[(size_t)i] % nx) / cb)]++] = i;
    off += n;
  }
  // batch assembly (a shared plan is repeated for every slice, the mask stored once)
  std::vector<int> spos, wlist, gidx, sidx, gptr, sptr;
  std::vector<float2> ph;
  std::vector<long long> soff(1, 0), woff(1, 0);
  long long nmax = 0, gbase = 0, sbase = 0;
  for (int b = 0; b < batch; ++b) {
    const Tab& t = tabs[(size_t)(shared ? 0 : b)];
    spos.insert(spos.end(), t.spos.begin(), t.spos.end());
    ph.insert(ph.end(), t.ph.begin(), t.ph.end());
    wlist.insert(wlist.end(), t.wl.begin(), t.wl.end());
    soff.push_back(soff.back() + (long long)t.spos.size());
    woff.push_back(woff.back() + (long long)t.wl.size());
    nmax = std::max(nmax, (long long)t.spos.size());
    gidx.insert(gidx.end(), t.gidx.begin(), t.gidx.end());
    sidx.insert(sidx.end(), t.sidx.begin(), t.sidx.end());
    long long g = gbase, s = sbase;
    gptr.push_back((int)g);
    sptr.push_back((int)s);
    for (int k = 0; k < nblk; ++k) {
      g += t.gcnt[(size_t)k];
      s += t.scnt[(size_t)k];
      gptr.push_back((int)g);
      sptr.push_back((int)s);
    }
    gbase = g;
    sbase = s;
  }
  cudaStream_t st = (cudaStream_t)stream;
  sr_cart_plan* p = new sr_cart_plan{};
  p->batch = batch;
  p->ny = ny;
  p->nx = nx;
  p->shared = shared ? 1 : 0;
  p->nblk = nblk;
  p->nmax = nmax;
  p->total = (long long)spos.size();
  p->wtotal = (long long)wlist.size();
  int rc = SR_OK;
  if ((rc = upload(&p->spos, spos, st)) || (rc = upload(&p->ph, ph, st)) || (rc = upload(&p->soff, soff, st)) ||
      (rc = upload(&p->woff, woff, st)) || (rc = upload(&p->wlist, wlist, st)) || (rc = upload(&p->maskT, maskT, st)) ||
      (rc = upload(&p->g_ptr, gptr, st)) || (rc = upload(&p->g_idx, gidx, st)) || (rc = upload(&p->s_ptr, sptr, st)) ||
      (rc = upload(&p->s_idx, sidx, st)) || (rc = (cudaStreamSynchronize(st) == cudaSuccess ? SR_OK : SR_ECUDA))) {
    cart_plan_free(p);
    return rc;
  }
  *out = p;
  return SR_OK;
}

int sr_cart_plan_destroy(sr_cart_plan* plan) {
  if (!plan) return SR_EINVAL;
  cart_plan_free(plan);
  return SR_OK;
}

// Geometry and device tables (any pointer may be NULL).
int sr_cart_plan_info(const sr_cart_plan* plan, int* ny, int* nx, long long* nmax, long long* total,
                      long long* wtotal, int* nblk, const int** spos, const sr_c64** ph, const long long** soff,
                      const int** wlist, const long long** woff, const uint8_t** maskT, const int** g_ptr,
                      const int** g_idx, const int** s_ptr, const int** s_idx) {
  if (!plan) return SR_EINVAL;
  if (ny) *ny = plan->ny;
  if (nx) *nx = plan->nx;
  if (nmax) *nmax = plan->nmax;
  if (total) *total = plan->total;
  if (wtotal) *wtotal = plan->wtotal;
  if (nblk) *nblk = plan->nblk;
  if (spos) *spos = plan->spos;
  if (ph) *ph = (const sr_c64*)plan->ph;
  if (soff) *soff = plan->soff;
  if (wlist) *wlist = plan->wlist;
  if (woff) *woff = plan->woff;
  if (maskT) *maskT = plan->maskT;
  if (g_ptr) *g_ptr = plan->g_ptr;
  if (g_idx) *g_idx = plan->g_idx;
  if (s_ptr) *s_ptr = plan->s_ptr;
  if (s_idx) *s_idx = plan->s_idx;
  return SR_OK;
}

// Workspace bytes the plan's normal / forward / adjoint need for ncoils coils.
long long sr_cart_plan_ws_bytes(const sr_cart_plan* plan, int ncoils) {
  if (!plan || ncoils < 1) return -1;
  const long long k2 = 8LL * plan->batch * ncoils * plan->ny * plan->nx;
  const long long k1 = sr_cart_ws_bytes(plan->batch, ncoils, plan->ny, plan->nx, 0);
  return k1 > k2 ? k1 : k2;
}

// K1 / K2 through the plan (argument meaning as sr_cart_normal / _forward / _adjoint; maps
// (batch or 1, ncoils, D) with map_bstride 0 for maps shared by every slice).
int sr_cart_plan_normal(const sr_cart_plan* plan, const sr_c64* x, const sr_c64* anchor, const sr_c64* maps,
                        long long map_bstride, int ncoils, sr_c64* out, sr_c64* ws, const float* coef,
                        const sr_c64* u, const sr_c64* d, void* stream) {
  if (!plan) return SR_EINVAL;
  return sr_cart_normal(x, anchor, maps, map_bstride, plan->maskT, plan->shared ? 0 : (long long)plan->ny * plan->nx,
                        out, ws, plan->batch, ncoils, plan->ny, plan->nx, coef, u, d, 0, stream);
}

int sr_cart_plan_forward(const sr_cart_plan* plan, const sr_c64* x, const sr_c64* maps, long long map_bstride,
                         int ncoils, sr_c64* y, long long ystride, const sr_c64* ymeas, double* partial,
                         int partial_blocks, sr_c64* ws, void* stream) {
  if (!plan || ystride < plan->nmax) return SR_EINVAL;
  return sr_cart_forward(x, maps, map_bstride, plan->spos, (const sr_c64*)plan->ph, plan->soff, y, ystride, ymeas,
                         partial, partial_blocks, ws, plan->batch, ncoils, plan->ny, plan->nx, plan->g_ptr,
                         plan->g_idx, plan->nblk, stream);
}

int sr_cart_plan_adjoint(const sr_cart_plan* plan, const sr_c64* y, long long ystride, const sr_c64* maps,
                         long long map_bstride, int ncoils, sr_c64* out, sr_c64* ws, const float* coef,
                         const sr_c64* u, const sr_c64* d, void* stream) {
  if (!plan || ystride < plan->nmax) return SR_EINVAL;
  return sr_cart_adjoint(y, ystride, maps, map_bstride, plan->spos, (const sr_c64*)plan->ph, plan->soff, plan->wlist,
                         plan->woff, out, ws, plan->batch, ncoils, plan->ny, plan->nx, coef, u, d, plan->s_ptr,
                         plan->s_idx, plan->nblk, stream);
}

}  // extern "C"

/*
 * sketchrecon_b200 -- C ABI of the B200 (sm_100a) sketched SENSE normal-operator path.
 *
 * Drop-in boundary for the reference package `sketchrecon`
 * (/root/reference/pkg/src/sketchrecon).  The reference is pure Python/NumPy and
 * has no FFI of its own; its plugin seams are the duck-typed Fourier kernel
 * (`apply` / `apply_adjoint`, linops.py:332-364, forward_model.py:134,147-148)
 * and the SenseOperator / solver API (forward_model.py:119-224, solvers.py,
 * coil_sketch.py).  Each entry point below names the reference computation it
 * replaces.  The Python host package `paper_2305_06482_b200` binds these with
 * ctypes (INTEGRATION.md shows the binding).
 *
 * Conventions
 *   - complex64 = interleaved (re, im) float32 (`sr_c64`); all array pointers
 *     are DEVICE pointers owned by the caller; sizes are element counts.
 *   - images are C-order (batch, ny, nx); coil stacks (batch, C, ny, nx);
 *     a *_bstride of 0 shares one array across the batch.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Every call is
 *     asynchronous and stream-ordered; none synchronises with the host.
 *   - return 0 on success, 1 invalid argument / shape (the reference raises
 *     ValueError), 2 unsupported transform length, 3 CUDA launch error.
 *   - FFT lengths: sr_fft_size_supported(n) (2^a 3^b 5^c with a register split,
 *     e.g. 8..1024 powers of two, 10..640 x5, 200, 400, 800, 24..768 x3).
 *   - Spectrum layout: the 2-D spectrum kept in `ws` is in "perm order" along
 *     both axes: frequency k of an n = P*Q axis sits at P*(k % Q) + k / Q.
 *     `maskT`, `spos` are built by the host in that layout.
 */
#ifndef SKETCHRECON_B200_H
#define SKETCHRECON_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { float x, y; } sr_c64;

/* 1 if an axis of length n has an instantiated FFT. */
int sr_fft_size_supported(int n);
/* (P, Q) register split of an axis of length n = P*Q (perm order P*(k % Q) + k / Q). */
int sr_fft_split(int n, int* P, int* Q);

/* K1 -- fused Cartesian (sketched) SENSE normal operator, batched over slices.
 *   out_b = e( sum_j conj(c_bj) * F^H M'_b F (c_bj * (x_b - anchor_b)) )
 * replaces `a_s.adjoint(a_s.forward(v))` (forward_model.py:168-180 over
 * linops.py:344-364), the call made at coil_sketch.py:126,133,197 and
 * solvers.py:175,248,460.
 *   maps: (batch, ncoils, ny, nx), map_bstride elements between slices (0 = shared)
 *   maskT: uint8 (ny*nx per mask) sampled-bin indicator, transposed [pos_x][pos_y]
 *          in perm order; mask_bstride bytes between slices (0 = shared)
 *   ws: workspace of batch*ncoils*ny*nx complex64
 *   anchor: NULL or (batch, ny, nx): operator input is x - anchor
 *   coef: NULL -> out = acc; else device float4 per slice {s_acc, s_u, s_d, -}:
 *         out = s_acc*acc + s_u*u + s_d*d  (FISTA: z - step*(acc + d); CG: acc + lam*v)
 *   chunk: 0 = three launches (row FFT, column FFT-mask-IFFT, row IFFT + coil sum)
 *          over the whole batch; > 0: the three launches per group of `chunk` slices
 *          (the single-launch / L2-exchange schedules of round 1 were measured slower and
 *          removed)
 *   ws: sr_cart_ws_bytes(batch, ncoils, ny, nx, chunk) bytes */
int sr_cart_normal(const sr_c64* x, const sr_c64* anchor, const sr_c64* maps,
                   long long map_bstride, const uint8_t* maskT, long long mask_bstride,
                   sr_c64* out, sr_c64* ws, int batch, int ncoils, int ny, int nx,
                   const float* coef, const sr_c64* u, const sr_c64* d, int chunk,
                   void* stream);

/* Tuning of the three-launch schedule: coils per CTA of the column pass (0 = one coil per
 * CTA, the generic kernel; default 4). */
int sr_cart_tune(int col_jc);
/* Tuning: the coil-looped column pass prefetches the next coil's strip in registers (pf = 1,
 * 2 CTAs/SM, default) or not (pf = 0, 3 CTAs/SM). */
int sr_cart_tune_colpf(int pf);
/* Tuning: preferred L1 / shared-memory carveout (percent of the maximum shared memory, -1 =
 * the driver's choice, the measured best) of the K1 column pass; it bounds how many CTAs of
 * the pass share an SM. */
int sr_cart_tune_carveout(int pct);
/* Tuning: the row FFT pass stores its output with TMA bulk copies (bulk = 1), through a
 * coalesced copy-out pass (0), or picks per size (2, default: bulk for 20-element groups with
 * Q >= 12, where it measured faster); rows shorter than min_n always use the copy-out. */
int sr_cart_tune_rows(int bulk, int min_n);

/* Workspace bytes sr_cart_normal needs for these arguments. */
long long sr_cart_ws_bytes(int batch, int ncoils, int ny, int nx, int chunk);

/* K2 -- SENSE forward A x (unweighted Cartesian): per-coil centered unitary FFT
 * sampled at the trajectory bins, `SenseOperator._forward` (forward_model.py:168-172)
 * over `_CartesianMaskKernel.apply` (linops.py:344-352).
 *   spos/ph: per-sample perm-order spectrum offset and centering phase; slice b owns
 *            samples [soff[b], soff[b+1]); y is (batch, ncoils, ystride)
 *   ymeas: NULL, or measured data -> y = A x - ymeas and, if partial != NULL,
 *          partial[(b*ncoils + j)*partial_blocks + k] = sum |y|^2 pieces
 *          (the residual of composite_objective, solvers.py:188-195).
 *   bptr/bidx/nblk: optional per-column-block sample lists (bptr (batch, nblk+1) absolute
 *          offsets into bidx = sample indices within the slice grouped by perm-order x block of
 *          sr_cart_col_block(ny) columns); given, the gather runs inside the column pass
 *          (nblk partial blocks, the rest zeroed); NULL = separate gather launch. */
int sr_cart_forward(const sr_c64* x, const sr_c64* maps, long long map_bstride,
                    const int* spos, const sr_c64* ph, const long long* soff,
                    sr_c64* y, long long ystride, const sr_c64* ymeas, double* partial,
                    int partial_blocks, sr_c64* ws, int batch, int ncoils, int ny, int nx,
                    const int* bptr, const int* bidx, int nblk, void* stream);
/* Column-block width (x positions per CTA) of the column pass for a column length ny. */
int sr_cart_col_block(int ny);

/* Opaque Cartesian plan (the tables of _CartesianMaskKernel, linops.py:332-364, in the device's
 * perm-order layout: sample offsets, centering phases, transposed mask, adjoint write list with
 * the last duplicate winning as linops.py:357, per-column-block sample lists), built by the library
 * from a HOST float64 trajectory: pts (total, ndim) centered integer bins of all slices
 * concatenated, counts = samples per slice (batch entries; one entry with shared = 1 for one mask
 * used by every slice); ndim 1 or 2, dims = (ny, nx) or (nx).  Identical to CartesianKernel's
 * tables.  Returns SR_EINVAL if any coordinate lies outside [-n/2, n/2) on its axis, as
 * Trajectory.validate_for (linops.py:130-140) rejects it.  The _normal / _forward / _adjoint entries take the arguments of sr_cart_normal /
 * sr_cart_forward / sr_cart_adjoint that the plan does not hold; ws: sr_cart_plan_ws_bytes. */
typedef struct sr_cart_plan sr_cart_plan;
int sr_cart_plan_create(const double* pts, const long long* counts, int batch, int ndim, const int* dims,
                        int shared, sr_cart_plan** out, void* stream);
int sr_cart_plan_destroy(sr_cart_plan* plan);
int sr_cart_plan_info(const sr_cart_plan* plan, int* ny, int* nx, long long* nmax, long long* total,
                      long long* wtotal, int* nblk, const int** spos, const sr_c64** ph, const long long** soff,
                      const int** wlist, const long long** woff, const uint8_t** maskT, const int** g_ptr,
                      const int** g_idx, const int** s_ptr, const int** s_idx);
long long sr_cart_plan_ws_bytes(const sr_cart_plan* plan, int ncoils);
int sr_cart_plan_normal(const sr_cart_plan* plan, const sr_c64* x, const sr_c64* anchor, const sr_c64* maps,
                        long long map_bstride, int ncoils, sr_c64* out, sr_c64* ws, const float* coef,
                        const sr_c64* u, const sr_c64* d, void* stream);
int sr_cart_plan_forward(const sr_cart_plan* plan, const sr_c64* x, const sr_c64* maps, long long map_bstride,
                         int ncoils, sr_c64* y, long long ystride, const sr_c64* ymeas, double* partial,
                         int partial_blocks, sr_c64* ws, void* stream);
int sr_cart_plan_adjoint(const sr_cart_plan* plan, const sr_c64* y, long long ystride, const sr_c64* maps,
                         long long map_bstride, int ncoils, sr_c64* out, sr_c64* ws, const float* coef,
                         const sr_c64* u, const sr_c64* d, void* stream);

/* K2 -- SENSE adjoint A^H y: scatter (last duplicate wins, as numpy fancy
 * assignment at linops.py:357), centered unitary IFFT, conjugate coil sum
 * (forward_model.py:174-180).  wlist/woff: per-slice list of sample indices to
 * write (duplicates removed by the host).  coef/u/d: epilogue as sr_cart_normal.
 * bptr/bidx/nblk: optional per-column-block lists of the wlist samples (as in sr_cart_forward);
 * given, the scatter runs inside the column pass (no workspace memset / scatter launch). */
int sr_cart_adjoint(const sr_c64* y, long long ystride, const sr_c64* maps,
                    long long map_bstride, const int* spos, const sr_c64* ph,
                    const long long* soff, const int* wlist, const long long* woff,
                    sr_c64* out, sr_c64* ws, int batch, int ncoils, int ny, int nx,
                    const float* coef, const sr_c64* u, const sr_c64* d,
                    const int* bptr, const int* bidx, int nblk, void* stream);

/* K5 -- coil contraction out[b,i,:] = sum_k S[b,i,k] in[b,k,:]:
 * `sketch_maps` (sketching.py:97-103, S real Chat x C) and the map/data rotation
 * of `coil_compress_svd` (forward_model.py:268-269, S = comp complex keep x C).
 * s_bstride = 0 shares S across the batch. in and out must not alias. */
int sr_coil_contract(const sr_c64* in, sr_c64* out, const sr_c64* S, long long s_bstride,
                     int batch, int cout, int cin, long long D, long long in_bstride,
                     long long out_bstride, void* stream);
/* K5, real coefficients (the sketch matrix of sketching.py:69-94): S (batch or 1, cout, cin)
 * float32, cout <= 32, D even, in/out 16-byte aligned; two voxels per thread. */
int sr_coil_contract_real(const sr_c64* in, sr_c64* out, const float* S, long long s_bstride, int batch, int cout,
                          int cin, long long D, long long in_bstride, long long out_bstride, void* stream);

/* K6 -- one level of the 2-D periodic DB4 analysis (linops.py:619-635, 677-687)
 * on the top-left h x w corner (row stride ld, slice stride bs); optional fused
 * soft threshold (solvers.py:129-135) with per-slice thresh[] (device) or host
 * hthresh >= 0; `last` thresholds the low-pass corner too; l1part collects
 * sum |coef| (Regularizer.value, solvers.py:61-69). src and dst must differ. */
int sr_wavelet_ana2(const sr_c64* src, sr_c64* dst, int h, int w, int ld, long long bs,
                    int batch, const float* thresh, float hthresh, int last, double* l1part,
                    void* stream);
int sr_wavelet_ana2_nblocks(int h, int w);
/* K6 -- one level of 2-D synthesis (linops.py:638-651, 689-702); at the final
 * level an optional FISTA momentum epilogue z = x + beta (x - xold)
 * (solvers.py:292-293). coef and out must differ. */
int sr_wavelet_syn2(const sr_c64* coef, sr_c64* out, int h, int w, int ld, long long bs,
                    int batch, sr_c64* zout, const sr_c64* xold, float beta, void* stream);
/* K6 -- the whole 2-D L1-wavelet prox (solvers.py:71-81, linops.py:654-702) in one call: `levels`
 * thresholded analysis levels into the scratch pair buf0/buf1 (each ny x nx per slice, row
 * stride nx, slice stride bs) and the synthesis into out, with the optional FISTA momentum
 * epilogue zout = out + beta (out - xold) on level 0 (out may alias xold, not v). */
int sr_wavelet_prox2(const sr_c64* v, sr_c64* out, sr_c64* buf0, sr_c64* buf1, int ny, int nx, long long bs,
                     int batch, int levels, const float* thresh, float hthresh, sr_c64* zout, const sr_c64* xold,
                     float beta, void* stream);
int sr_wavelet_levels_max(void);
/* K6 n-D -- one axis of one DB4 level (analysis or synthesis) over the (h0, h1, h2)
 * corner of (n0, n1, n2) arrays, for 1-D and 3-D grids (linops.py:619-651, 677-702);
 * thr_enable (analysis, last axis of a level) soft-thresholds the detail sub-bands
 * (and the low-pass corner when last_level) and fills l1part (batch, nblocks);
 * zout/xold/beta: FISTA momentum epilogue on the final synthesis launch. */
int sr_wavelet_axis(const sr_c64* src, sr_c64* dst, int h0, int h1, int h2, int n1, int n2, long long bs,
                    int batch, int axis, int inverse, const float* thresh, float hthresh, int thr_enable,
                    int last_level, double* l1part, sr_c64* zout, const sr_c64* xold, float beta,
                    void* stream);
int sr_wavelet_axis_nblocks(void);

/* K7 -- deterministic per-slice reductions (fixed-order, no atomics).
 * mode 0: sum |a|^2   1: sum conj(a) b   2: sum |a|   3: sum |a - b|^2
 * partial: batch * sr_reduce_nparts() double2; result: batch double2.
 * (np.linalg.norm / np.vdot in solvers.py:192,211,219,225 and linops.py:777-780) */
int sr_reduce(int mode, const sr_c64* a, const sr_c64* b, long long n, long long bstride,
              int batch, double* partial, double* result, void* stream);
int sr_reduce_nparts(void);

/* Total variation for the PDHG sub-solver (l1-tv; coil_sketch.py:200-216, solvers.py:315-362).
 * Images (batch, dims...) complex64, dual variables (batch, ndim, D) axis-major as the
 * reference's FiniteDiffOp (linops.py:717-741).  dims: host array of ndim extents.
 *   sr_tv_dual   mode 0: p = clamp(p + sigma[b] * D z, lam) (_clamp_magnitude, solvers.py:138-142)
 *                mode 1: p = D z (forward differences, for the objective)
 *   sr_tv_primal v = x - tau[b] * D^H p
 * sigma / tau: per-slice device float arrays. */
int sr_tv_dual(sr_c64* p, const sr_c64* z, const int* dims, int ndim, int mode, const float* sigma, float lam,
               int batch, void* stream);
int sr_tv_primal(sr_c64* v, const sr_c64* x, const sr_c64* p, const int* dims, int ndim, const float* tau,
                 int batch, void* stream);

/* K7 -- out = cx*X + cy*Y + cz*Z with per-slice device coefficients (float4) or
 * host coefficients when coef == NULL (axpy / momentum of solvers.py:223-227,293). */
int sr_lincomb(sr_c64* out, const sr_c64* X, const sr_c64* Y, const sr_c64* Z,
               const float* coef, float cx, float cy, float cz, long long n,
               long long bstride, int batch, void* stream);

/* K7 -- per-slice scalar bookkeeping on the device:
 * op 0 power iteration step (linops.py:776-781), op 1 CG alpha, op 2 CG beta
 * (solvers.py:218-228). */
/* K7 fused CG vector step of _cg_loop (solvers.py:206-229) for `batch` slices after the matvec
 * mp = M p: alpha = rs / <p, mp>, x += alpha p, r -= alpha mp, rs_new = |r|^2, p = r + beta p,
 * in three launches with fixed-order reductions (bit-reproducible).  pdot, prs: (batch,
 * sr_reduce_nparts()) double2 scratch; state (batch, 4) doubles [rs0, rs1, active, iterations]
 * set by the caller before the first step (rs0 = |r0|^2, active = 1, iterations = 0);
 * parity = iteration & 1.  A slice stops updating (the reference's break) when sqrt(rs) <=
 * tol_abs or <p, mp> <= 0; `iterations` then equals the reference's iteration count.  hist:
 * NULL or (batch, hist_len + 1) doubles, hist[b][it] = sqrt(rs) after iteration it. */
int sr_cg_step(sr_c64* x, sr_c64* r, sr_c64* p, const sr_c64* mp, double* pdot, double* prs, double* state,
               double* hist, int hist_len, long long n, long long bstride, int batch, int parity,
               double tol_abs, void* stream);
int sr_scalar_op(int op, const double* in0, const double* in1, double* state, float* coefA,
                 float* coefB, int* flags, int batch, void* stream);

/* K3/K4 -- Kaiser-Bessel gridded NUFFT SENSE operator, 2-D or 3-D, one image
 * (replaces _GriddedNUFFTKernel.apply/apply_adjoint, linops.py:494-516, inside
 * SenseOperator with density weights, forward_model.py:168-180).
 *   dims/gdims: 3 image / oversampled-grid dims (leading 1 for 2-D); betas: 3 KB betas
 *   (dims, gdims, betas are HOST arrays, every other pointer is a device pointer);
 *   ia0..ia2: inverse apodisation per axis (fp32 of the fp64 reference formula);
 *   base (3, N) int32 = ceil(u - w/2) per axis (fp64 on the host), frac (3, N) fp32 = u - base;
 *   wgt: w (normal) or sqrt(w) (forward / adjoint) per sample, NULL = 1; orig: original
 *   index of each (locality-sorted) sample or NULL; grids: ncoils*G (fwd/adj) or
 *   2*ncoils*G (normal) complex64 workspace.  Epilogue coef/u/d as sr_cart_normal.
 *   chunks (nchunks x 5 int32: bin origin (3 grid indices), first sorted sample, count <= 256)
 *   selects the binned shared-memory gridding with bins of binsize^d cells; chunks = NULL
 *   uses one thread per sample with global float2 atomics.  With chunks, partial has
 *   nchunks entries (forward with ymeas), else sr_nufft_partial_blocks(N). */
int sr_nufft_normal(const sr_c64* x, const sr_c64* anchor, const sr_c64* maps, int ncoils,
                    const int* dims, const int* gdims, const float* betas, int width,
                    const float* ia0, const float* ia1, const float* ia2, const int* base,
                    const float* frac, const float* wgt, long long nsamples, sr_c64* out,
                    sr_c64* grids, const float* coef, const sr_c64* u, const sr_c64* d, const int* chunks,
                    int nchunks, int binsize, void* stream);
/* sr_nufft_normal with the zeroing of the spread grid off the critical path (binned plans only,
 * else SR_EUNSUPPORTED).  grids: 3 * ncoils * G complex64 -- the spectrum grids and two spread grids
 * used in turn.  The call spreads into spread grid dst_index (0 | 1), which it zeroes first unless
 * dst_clean != 0, and the gridding kernel zeroes the other one as it runs (that kernel leaves HBM
 * nearly idle, so the stores are free).  A caller
 * alternating dst_index may pass dst_clean = 1 from its second call on, as long as nothing else
 * wrote the workspace in between.  Same result as sr_nufft_normal. */
int sr_nufft_normal_pp(const sr_c64* x, const sr_c64* anchor, const sr_c64* maps, int ncoils,
                       const int* dims, const int* gdims, const float* betas, int width,
                       const float* ia0, const float* ia1, const float* ia2, const int* base,
                       const float* frac, const float* wgt, long long nsamples, sr_c64* out,
                       sr_c64* grids, const float* coef, const sr_c64* u, const sr_c64* d, const int* chunks,
                       int nchunks, int binsize, int dst_index, int dst_clean, void* stream);
/* sr_nufft_normal in two parts for the coil-sharded pipeline (config 4): _head runs the embed, the
 * forward passes, the gridding and the axis-0 inverse pass into `grids`; _tail finishes image
 * planes i0 in [i0a, i0b) only (remaining inverse passes, crop, conjugate coil sum, epilogue), so
 * a caller can all-reduce one slab of the coil sum while the next slab computes.  head + tail over
 * [0, dims[0]) == sr_nufft_normal.  Partial slabs need dims[0] * dims[1] >= 9472 image rows
 * (sr_nufft_normal_slabs_ok); otherwise _tail returns SR_EUNSUPPORTED for a partial slab. */
int sr_nufft_normal_head(const sr_c64* x, const sr_c64* anchor, const sr_c64* maps, int ncoils,
                         const int* dims, const int* gdims, const float* betas, int width, const float* ia0,
                         const float* ia1, const float* ia2, const int* base, const float* frac, const float* wgt,
                         long long nsamples, sr_c64* grids, const int* chunks, int nchunks, int binsize,
                         void* stream);
int sr_nufft_normal_tail(const sr_c64* maps, int ncoils, const int* dims, const int* gdims, const float* betas,
                         int width, const float* ia0, const float* ia1, const float* ia2, sr_c64* out,
                         sr_c64* grids, const float* coef, const sr_c64* u, const sr_c64* d, int i0a, int i0b,
                         void* stream);
int sr_nufft_normal_slabs_ok(const int* dims);
int sr_nufft_forward(const sr_c64* x, const sr_c64* maps, int ncoils, const int* dims, const int* gdims,
                     const float* betas, int width, const float* ia0, const float* ia1, const float* ia2,
                     const int* base, const float* frac, const float* sqrtw, const int* orig,
                     long long nsamples, sr_c64* y, const sr_c64* ymeas, double* partial, sr_c64* grids,
                     const int* chunks, int nchunks, int binsize, void* stream);
int sr_nufft_adjoint(const sr_c64* y, const sr_c64* maps, int ncoils, const int* dims, const int* gdims,
                     const float* betas, int width, const float* ia0, const float* ia1, const float* ia2,
                     const int* base, const float* frac, const float* sqrtw, const int* orig,
                     long long nsamples, sr_c64* out, sr_c64* grids, const float* coef, const sr_c64* u,
                     const sr_c64* d, const int* chunks, int nchunks, int binsize, void* stream);
int sr_nufft_partial_blocks(long long nsamples);
/* 3-D Cartesian mask kernel (_CartesianMaskKernel on a 3-D grid, linops.py:332-364, which the
 * 2-D K1/K2 kernels do not cover): the grid pipeline of the NUFFT entries with g = n and unit
 * apodisation.  dims (3, HOST ints, axes with sr_fft_size_supported lengths); ones0..2 device
 * float vectors of ones (lengths dims[a]); spos (N) int32 grid offset of each sample,
 * perm(f_0) n1 n2 + perm(f_1) n2 + f_2 (f_a mod n_a; axes 0-1 perm order, the contiguous axis 2
 * natural); mask (n0 n1 n2) uint8 sampled-bin indicator in the same
 * layout; wlist (nw) the last occurrence of every distinct bin (linops.py:357); grids ncoils * D
 * complex64 workspace; y / ymeas (ncoils, ystride); partial: sr_cart3_partial_blocks(N, ncoils)
 * doubles of |A x - y|^2 when ymeas is given.  Epilogue coef/u/d as sr_cart_normal. */
int sr_cart3_normal(const sr_c64* x, const sr_c64* anchor, const sr_c64* maps, int ncoils, const int* dims,
                    const float* ones0, const float* ones1, const float* ones2, const unsigned char* mask,
                    sr_c64* out, sr_c64* grids, const float* coef, const sr_c64* u, const sr_c64* d, void* stream);
int sr_cart3_forward(const sr_c64* x, const sr_c64* maps, int ncoils, const int* dims, const float* ones0,
                     const float* ones1, const float* ones2, const int* spos, long long nsamples, sr_c64* y,
                     long long ystride, const sr_c64* ymeas, double* partial, sr_c64* grids, void* stream);
int sr_cart3_adjoint(const sr_c64* y, long long ystride, const sr_c64* maps, int ncoils, const int* dims,
                     const float* ones0, const float* ones1, const float* ones2, const int* spos,
                     const int* wlist, long long nw, sr_c64* out, sr_c64* grids, const float* coef, const sr_c64* u,
                     const sr_c64* d, void* stream);
int sr_cart3_partial_blocks(long long nsamples, int ncoils);
/* NUFFT plan on the device (replaces the host loop of _GriddedNUFFTKernel._build_interpolator,
 * linops.py:464-492, for the tap geometry): pts (N, ndim) float64 trajectory (device);
 * dims/gdims HOST arrays of ndim entries.  Writes, in trajectory order, base (3, N) int32 =
 * ceil(k g / n - w/2) per axis (leading zero rows for 2-D), frac (3, N) float32 offsets whose
 * KB support decisions equal the reference's float64 ones, and the locality sort key
 * key (N) int64 = bin * binsize^ndim + cell within bin; *err (device int) is set to 1 if an
 * offset could not be aligned or a coordinate lies outside [-n/2, n/2) (linops.py:130-140).  sr_nufft_plan_permute gathers base/frac by a (stable) sort
 * order of key and writes orig (N) int32 = order. */
int sr_nufft_plan_geom(const double* pts, long long nsamples, int ndim, const int* dims, const int* gdims,
                       int width, int binsize, int* base, float* frac, long long* key, int* err, void* stream);
int sr_nufft_plan_permute(const int* base_in, const float* frac_in, const long long* order, long long nsamples,
                          int* base_out, float* frac_out, int* orig, void* stream);

/* Opaque NUFFT plan owned by the library (the whole _build_interpolator of linops.py:464-492 plus
 * the grid / Beatty beta / apodisation of linops.py:434-462, built on the device from a HOST
 * float64 trajectory (N, ndim); identical to GriddedKernel's plan).  binsize 0 = default.
 * sr_nufft_plan_info returns its geometry and device arrays (any pointer may be NULL);
 * sr_nufft_plan_normal applies the (sketched) SENSE normal operator with it, sqrtw = sqrt of the
 * density weights in trajectory order (device, NULL = 1), grids as sr_nufft_normal. */
typedef struct sr_nufft_plan sr_nufft_plan;
int sr_nufft_plan_create(const double* pts, long long nsamples, int ndim, const int* dims, double oversamp,
                         int width, int binsize, sr_nufft_plan** out, void* stream);
int sr_nufft_plan_destroy(sr_nufft_plan* plan);
int sr_nufft_plan_info(const sr_nufft_plan* plan, int* dims, int* gdims, float* betas, long long* nsamples,
                       long long* nchunks, const int** base, const float** frac, const int** orig,
                       const int** chunks, const float** ia0, const float** ia1, const float** ia2);
int sr_nufft_plan_normal(sr_nufft_plan* plan, const sr_c64* x, const sr_c64* anchor, const sr_c64* maps, int ncoils,
                         const float* sqrtw, sr_c64* out, sr_c64* grids, const float* coef, const sr_c64* u,
                         const sr_c64* d, void* stream);
/* Batched tall-skinny Householder QR, R only (LAPACK zgeqr2 / zlarfg conventions), complex128:
 * A (batch, N, C) row-major blocks Y^H (overwritten), R (batch, C, C); C <= 32.  The LQ step of
 * numpy's SVD of a wide C x N block (coil_compress_svd, forward_model.py:245-272). */
int sr_tsqr_r(void* A, long long N, int C, long long a_bstride, int batch, void* R, void* stream);
/* Device-to-device copy on a stream. */
int sr_memcpy_d2d(void* dst, const void* src, long long bytes, void* stream);
/* Batched unnormalised FFT along the middle axis of an [outer][n][inner] array, in
 * place: inv = 0 natural -> perm order, inv = 1 perm -> natural. */
int sr_fft_axis(sr_c64* data, long long outer, int n, long long inner, int inv, void* stream);

/* K8 -- readout decoupling of 3-D Cartesian data (BASELINE config 2): centered unitary
 * IDFT along the fully sampled readout of in (ncoils, n, inner), written slice-major to
 * out (n, ncoils, inner); pre[k], post[x] (device, length n) carry the centering phases
 * and n^-1/2 (host-computed in fp64).  Each out[x] is then the 2-D SENSE data of slice x. */
int sr_readout_idft(const sr_c64* in, sr_c64* out, const sr_c64* pre, const sr_c64* post, int ncoils, int n,
                    long long inner, void* stream);

/* Host (CPU) synthetic-input helper: variable-density Poisson-disc mask of
 * ny x nx bins (1 = sampled, row-major) with a fully sampled calib x calib
 * centre and about ny*nx/accel samples (BASELINE configs 0-2; the reference
 * only has 1-D line masks, simulate.py:209-259).  Returns the sample count. */
long long sr_host_vd_poisson(int ny, int nx, double accel, int calib, unsigned long long seed,
                             uint8_t* mask);

#ifdef __cplusplus
}
#endif
#endif /* SKETCHRECON_B200_H */

/*
 * psb200.h -- C ABI of libpsb200.so, the sm_100a implementation of the
 * ProxSkip / PDHGSkip TV hot path (arXiv 2411.00688).
 *
 * The reference (`imgskip`, pure Python) has no FFI: its drop-in surface is
 * the duck-typed Python API listed in SURVEY.md 8(b).  Each entry point below
 * names the reference function it replaces (paths relative to
 * /root/reference/pkg/src/imgskip).  The Python package
 * `paper_2411_00688_b200` binds these symbols with ctypes and re-exposes the
 * reference's names and signatures (INTEGRATION.md shows the binding).
 *
 * Conventions
 *   - every function returns PSB_OK (0) or a PSB_ERR_* status; the message is
 *     available from psb_last_error() (thread-local).
 *   - device buffers are plain device pointers; sizes are element counts;
 *     `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *   - layouts follow the reference: image (H, W) row-major; dual field
 *     (2, H, W) with channel 0 = row (vertical) differences (tensor.py:80-106,
 *     operators.py:44-57); sinogram (n_angles, n_bins) (tensor.py:109-127).
 *     A batch of problems is the same layout repeated with a per-problem
 *     stride ("pstride", in elements).
 *   - FGP dual state: each problem owns three dual "slots" of (2, H, W)
 *     (q_pstride >= 6*H*W); the warm start q_warm (tv.py:25-50) lives in
 *     slot 0 between prox calls, inner iteration `it` reads slots it%3 and
 *     (it+2)%3 and writes slot (it+1)%3, and the finalize step moves the last
 *     iterate back to slot 0.
 *   - dtype codes: PSB_F32 (production) or PSB_F64 (bit-exact debug path:
 *     every op rounded separately, matching numpy).
 */
#ifndef PSB200_H_
#define PSB200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSB_ABI_VERSION 2

#define PSB_OK 0
#define PSB_ERR_VALUE 1    /* maps to ValueError */
#define PSB_ERR_CUDA 2     /* maps to RuntimeError */
#define PSB_ERR_DIVERGED 3 /* maps to DivergenceError (errors.py:4-11) */

#define PSB_F32 0
#define PSB_F64 1

int psb_abi_version(void);
const char* psb_last_error(void);
int psb_device_sm_count(int* out);

/* ---- context + device buffers: for hosts without a CUDA
 * runtime of their own.  Every compute entry point below takes plain device
 * pointers and a stream; psb_ctx_stream() provides one, psb_buf_alloc() the
 * device memory (zero-filled, stream-ordered), psb_upload()/psb_download()
 * synchronous host copies staged through pinned memory.  A context is used
 * by one host thread at a time (the reference's runs are single-threaded,
 * SURVEY 8(b) "Threading"). */
typedef struct psb_ctx psb_ctx;
int psb_ctx_create(int device, psb_ctx** out);
int psb_ctx_destroy(psb_ctx* ctx);
void* psb_ctx_stream(psb_ctx* ctx);
int psb_ctx_sync(psb_ctx* ctx);
int psb_buf_alloc(psb_ctx* ctx, int64_t bytes, void** dptr);
int psb_buf_free(psb_ctx* ctx, void* dptr);
int psb_upload(psb_ctx* ctx, void* dptr, const void* host, int64_t bytes);
int psb_download(psb_ctx* ctx, void* host, const void* dptr, int64_t bytes);

/* ---- finite differences: operators.py:44-57 (grad_forward), :60-71 (divergence) */
int psb_grad2d(int dtype, const void* u, void* g, int64_t n, int H, int W, void* stream);
int psb_div2d(int dtype, const void* q, void* d, int64_t n, int H, int W, void* stream);

/* ---- pointwise proxes: proximal.py:10-21 (project_ball), :39-41 (project_nonneg) */
int psb_project_ball2d(int dtype, const void* q, void* out, int64_t n, int64_t HW, double radius,
                       void* stream);
int psb_project_nonneg(int dtype, const void* u, void* out, int64_t count, void* stream);

/* ---- generic elementwise building block for the drivers' vector algebra
 * (skip.py:66-74, solvers.py:139-206 with user-supplied closures):
 * out = (a*x) + (b*y), each product rounded separately; a == 1 skips the
 * first product, y == NULL drops the second term. */
int psb_lincomb(int dtype, double a, const void* x, double b, const void* y, void* out,
                int64_t count, void* stream);

/* ---- diagonal-step PDHG building blocks (solvers.py:187-234, problems.py:139-146)
 * psb_axpy_arr:   out = x + sign * (s .* y), s an array (diagonal steps)
 * psb_fidprox:    out = (v - t .* b) / (1 + t), t scalar or t_arr per element
 * psb_recip_floor: out = 1 / max(x, floor)  (diagonal_steps, solvers.py:212-224)
 * psb_absgrad2d / psb_absdiv2d: |D| u and |D|^T q, the abs maps of grad_map
 *   (operators.py:81-94) that back diagonal preconditioning */
int psb_axpy_arr(int dtype, const void* x, int sign, const void* s, const void* y, void* out,
                 int64_t count, void* stream);
int psb_fidprox(int dtype, const void* v, double t, const void* t_arr, const void* b, void* out,
                int64_t count, void* stream);
int psb_recip_floor(int dtype, const void* x, double floor_, void* out, int64_t count,
                    void* stream);
/* Iteration loops replayed from one captured CUDA graph (no per-iteration
 * host round trip): psb_mark_nonfinite sets *bad_iter = min(*bad_iter,
 * *iter_ctr) if x has a non-finite entry (solvers.py:111-113, the 0-based
 * iteration the reference's DivergenceError names); psb_counter_add adds v
 * to the device counter. */
int psb_mark_nonfinite(int dtype, const void* x, int64_t count, int32_t* bad_iter,
                       const int32_t* iter_ctr, void* stream);
int psb_counter_add(int32_t* ctr, int v, void* stream);
/* psb_prox_l2_fidelity: out = (x + t .* b) / (1 + t), t scalar or t_arr per
 * element -- prox_l2_fidelity(x, b, tau), proximal.py:44-55 */
int psb_prox_l2_fidelity(int dtype, const void* x, double t, const void* t_arr, const void* b,
                         void* out, int64_t count, void* stream);
int psb_absgrad2d(int dtype, const void* u, void* g, int H, int W, void* stream);
int psb_absdiv2d(int dtype, const void* q, void* d, int H, int W, void* stream);

/* ---- FGP TV prox, tv.py:53-89 -------------------------------------------
 * psb_fgp2d_iter: ONE inner iteration (tv.py:75-80) for every problem in
 *   `active` (device int32[n_active]; NULL = problems 0..n_active-1):
 *     y   = q_it + beta_prev * (q_it - q_{it-1})        (recomputed, not stored)
 *     q'  = P_w(y + step * grad(clamp(x + div y)))        -> slot (it+1)%3
 *   At it == 0 the warm start is re-projected onto the new ball first when the
 *   problem's reproject flag is set (tv.py:68-69).  `weights` (device double,
 *   one per ACTIVE-LIST POSITION) overrides `weight` when non-NULL; likewise
 *   `reproject` (device uint8 per active-list position) overrides
 *   `reproject_all`.
 * psb_fgp2d_finalize: u = clamp(x + div q_n) (tv.py:89) and q_n -> slot 0.
 * psb_tv_prox2d: the whole prox (re-projection, n_inner iterations with the
 *   Beck-Teboulle beta table computed in double on the host, finalize).
 *   accelerated = 0 runs the plain projected-gradient branch (tv.py:82-84). */
int psb_fgp2d_iter(int dtype, const void* x, int64_t x_pstride, void* q, int64_t q_pstride,
                   const int32_t* active, int n_active, double weight, const double* weights,
                   int reproject_all, const uint8_t* reproject, int H, int W, int it,
                   double beta_prev, double step, int nonneg, void* stream);
int psb_fgp2d_finalize(int dtype, const void* x, int64_t x_pstride, void* q, int64_t q_pstride,
                       const int32_t* active, int n_active, int H, int W, int n_inner, int nonneg,
                       void* u, int64_t u_pstride, void* stream);
/* Accelerated projected gradient on the dual ROF problem (run_aprojgd on
 * build_dual_rof(b, alpha) with huber_eps = 0, solvers.py:148-174,
 * problems.py:22-71): q = 3 (2,H,W) slots with the start point in slot 0; on
 * return slot 0 holds the final dual iterate and u = b + div q
 * (primal_from_dual, problems.py:78-84).  step = gamma (1/8 = 1/L). */
int psb_aprojgd_dual_rof(int dtype, const void* b, void* q, int H, int W, double alpha,
                         double step, int iters, void* u, void* stream);
/* Dual-ROF light-prox drivers (build_dual_rof, problems.py:22-84; SURVEY 8(f)
 * row 4): algo 0 = GD, 1 = PGD / ProjGD, 2 = FISTA / AProjGD, 3 = ProxSkip
 * (solvers.py:116-174, skip.py:46-79) on q (2,H,W) in place; h: ProxSkip
 * control variate (2,H,W) or NULL; work: 4*H*W scratch; huber_mu =
 * huber_eps / alpha; coins_host: uint8[K] (ProxSkip only).  Optional per-
 * iteration device elapsed times and iterate history as in the other run
 * drivers. */
int psb_dual_rof_run(int dtype, int algo, const void* b, void* q, void* h, void* work, int H,
                     int W, double alpha, double huber_mu, double gamma, double p,
                     const uint8_t* coins_host, int K, int32_t* bad_iter, int use_graph,
                     double* elapsed_host, void* x_hist, void* stream);
int psb_tv_prox2d(int dtype, const void* x, int64_t x_pstride, void* q, int64_t q_pstride,
                  const int32_t* active, int n_active, double weight, const double* weights,
                  int reproject_all, const uint8_t* reproject, int H, int W, int n_inner,
                  int accelerated, int nonneg, double step, void* u, int64_t u_pstride,
                  void* stream);

/* ---- periodic blur, operators.py:109-184 -----------------------------------
 * psb_blur2d: blur_forward (adjoint = 0) / blur_adjoint (adjoint = 1) of n
 *   images with the reference's 2-D tap order (bit-exact in fp64).
 *   taps2d: HOST double[ksize*ksize], row-major, odd ksize <= 15.
 * psb_blur_grad2d: the fidelity gradient g = A^T (A u - b) (problems.py:121).
 *   separable != 0: one fused kernel with the 1-D factor taps1d (HOST
 *   double[ksize], w = taps1d taps1d^T); separable == 0: the direct order via
 *   `scratch` (device, H*W elements). */
int psb_blur2d(int dtype, const void* u, void* out, int64_t n, int H, int W, const double* taps2d,
               int ksize, int adjoint, void* stream);
int psb_blur_grad2d(int dtype, const void* u, const void* b, void* g, int H, int W,
                    const double* taps2d, const double* taps1d, int ksize, int separable,
                    void* scratch, void* stream);

/* ---- reductions (fp64 accumulation, deterministic two-pass) ---------------
 * per-problem results are written to the DEVICE array out[n].
 * psb_sumsq: sum((a-b)^2) (b may be NULL) -- tensor.py:28-30, 42-51 building block
 * psb_dot:   sum(a*b)                      -- tensor.py:17-25
 * psb_tv2d:  isotropic TV, tv.py:19-22
 * psb_count_nonfinite: number of non-finite entries (solvers.py:111-113) */
int psb_sumsq(int dtype, const void* a, const void* b, int64_t n, int64_t len, double* out,
              void* stream);
int psb_dot(int dtype, const void* a, const void* b, int64_t n, int64_t len, double* out,
            void* stream);
int psb_tv2d(int dtype, const void* u, int64_t n, int H, int W, double* out, void* stream);
int psb_count_nonfinite(int dtype, const void* a, int64_t count, double* out, void* stream);
/* Batched logging reductions over an iterate history a[n][len] (device
 * IterationLog): psb_sumsq_bcast = sum((a_p - b)^2) with one
 * shared b (rel_error against the reference solution, tensor.py:42-51, and the
 * identity fidelity of objective_tv, problems.py:187-192); psb_count_below =
 * number of entries < thresh (the nonneg guard of objective_tv). */
int psb_sumsq_bcast(int dtype, const void* a, const void* b, int64_t n, int64_t len, double* out,
                    void* stream);
int psb_count_below(int dtype, const void* a, int64_t n, int64_t len, double thresh, double* out,
                    void* stream);
/* psb_count_outside_ball: number of pixels of a (2, len) dual field q with
 * sqrt(q0^2 + q1^2) > r, evaluated in fp64 -- the feasibility test of
 * dual_gap_rof (tv.py:98-100) */
int psb_count_outside_ball(int dtype, const void* q, int64_t len, double r, double* out,
                           void* stream);

/* Bernoulli coin table of many problems (skip.py:16-28): coins[k*n + i] =
 * Generator(Philox(seeds[i])).random() < p for k < K, bit-identical to numpy
 * (SeedSequence key derivation + Philox4x64-10 on the device); host in/out. */
int psb_coin_table(const int64_t* seeds_host, int64_t n, int K, double p, uint8_t* coins_host,
                   void* stream);

/* ---- ProxSkip outer step, skip.py:46-79 -------------------------------------
 * State x, h (dtype_outer) and prox input z (dtype_fgp), all (n, H, W).
 * `g_or_b`: when ident != 0 it is b and the gradient x - b of the identity
 * fidelity (problems.py:121, operators.py:297-307) is fused; otherwise it is
 * the precomputed gradient g = A^T(Ax - b).
 * psb_proxskip_pre: for every problem i: if coins[i]:
 *      z = (x - gamma g) + hcoef h            (hcoef = gamma - gamma/p)
 *   else (skipped, h unchanged):
 *      x = (x - gamma g) + gamma h
 *   coins: device uint8[n] (NULL = all fire, e.g. PGD).
 * psb_proxskip_post (coin-fired problems in `active`): fused FGP finalize
 *   u = clamp(z + div q_n), q_n -> slot 0, then
 *      xhat = (x - gamma g) + gamma h ; h += pg * (u - xhat) ; x = u   (pg = p/gamma)
 * Non-finite iterates record min(bad_iter[i], k) (device int32[n]) so the
 * host can raise DivergenceError(k) (solvers.py:111-113). */
int psb_proxskip_pre(int dtype_outer, int dtype_fgp, void* x, const void* g_or_b, int ident,
                     const void* h, void* z, int64_t n, int64_t HW, const uint8_t* coins,
                     double gamma, double hcoef, int32_t* bad_iter, int k, void* stream);
int psb_proxskip_post(int dtype_outer, int dtype_fgp, void* x, const void* g_or_b, int ident,
                      void* h, const void* z, void* q, int64_t q_pstride, const int32_t* active,
                      int n_active, int H, int W, int n_inner, int nonneg, double gamma, double pg,
                      int32_t* bad_iter, int k, void* stream);

/* psb_skip_chain: `pend` deferred skipped ProxSkip iterations of the identity
 * fidelity (skip.py:68, h unchanged), executed in registers in the reference's
 * op order -- bit-identical to `pend` separate passes.  z != NULL: write the
 * prox input z = (x_m - gamma (x_m - b)) + hcoef h and leave x in memory
 * (the post kernel recomputes x_m); z == NULL: store x_m (end-of-run flush).
 * Non-finite x_m at step s records kfirst + s in bad_iter[0]. */
int psb_skip_chain(int dtype_outer, int dtype_fgp, void* x, const void* b, const void* h, void* z,
                   int64_t count, int pend, double gamma, double hcoef, int32_t* bad_iter,
                   int kfirst, void* stream);

/* ---- fused run drivers (the native runtime) ---------------------------------
 * psb_proxskip_denoise_run: K outer ProxSkip iterations of the implicit TV
 *   denoising problem (identity fidelity; problems.py:117-132 + skip.py:46-79)
 *   for n independent problems.  coins_host: host uint8[K * n] (row k =
 *   iteration k, the per-problem Philox streams drawn by the caller,
 *   skip.py:27-28).  last_weight_host: host double[n], NaN = never called
 *   (TvProxState.last_weight = None).  On return last_weight_host is updated
 *   and prox_count_host[n] (host int64) holds the prox calls per problem.
 *   use_graph != 0 captures the launch sequence into one CUDA graph.
 *   elapsed_host (nullable, host double[K]) receives the device time in
 *   seconds from the run start to the end of each outer iteration
 *   (IterationLog.elapsed_s, solvers.py:84-86), from CUDA events.
 *   fgp_time_host (nullable, host double[K]) receives the device time of the
 *   FGP inner-iteration burst of each outer iteration (0 when no coin fired),
 *   for the benchmark's roofline accounting.
 *   x_hist (nullable, device, K*n*H*W of dtype_outer) receives the iterate
 *   after every outer iteration (device IterationLog; forces the streaming
 *   path, since the cluster path defers skipped iterations).  The PDHG and
 *   implicit-CT drivers below take the same x_hist (K*n*n).
 *   algo 0 = ProxSkip, 1 = FISTA (solvers.py:148-168; coins all set, p = 1,
 *   aux = x_prev then xbar, 2*n*H*W of dtype_outer, x_prev initialised to x0). */
int psb_proxskip_denoise_run(int dtype_outer, int dtype_fgp, void* x, const void* b, void* h,
                             void* z, void* q, int64_t n, int H, int W, const uint8_t* coins_host,
                             int K, double gamma, double p, double alpha, int n_inner,
                             int accelerated, int nonneg, double* last_weight_host,
                             int64_t* prox_count_host, int32_t* bad_iter, int use_graph,
                             double* elapsed_host, double* fgp_time_host, void* x_hist, int algo,
                             void* aux, void* stream);

/* psb_proxskip_denoise_run_streamed: psb_proxskip_denoise_run (fp32 FGP,
 *   256x256, no graph, no log) whose kernels start before their inputs have
 *   arrived.  Problems form chunks c = [bounds_host[c], bounds_host[c+1])
 *   (host int64[n_chunks + 1], 0 .. n); the run kernels wait, per problem,
 *   until ready[c] != 0 (device
 *   int32[n_chunks + 1], zeroed; the caller's copy stream writes 1 after the
 *   chunk's H2D copy with psb_stream_write_u32), and add 16 per finished
 *   problem to done[p / chunk] (device int32[n_chunks], zeroed) so the copy
 *   stream can psb_stream_wait_geq_u32 for 16 * (problems in the chunk)
 *   before the chunk's D2H copy.  ready[n_chunks] becomes 1 if a wait timed
 *   out (20 s).  The run starts COLD: x = h = 0 and a zero warm start are
 *   implied (x, h, q need not be initialised; the kernels write them).  Same
 *   results as psb_proxskip_denoise_run from zeroed buffers (bit-identical). */
int psb_proxskip_denoise_run_streamed(int dtype_outer, int dtype_fgp, void* x, const void* b,
                                      void* h, void* z, void* q, int64_t n, int H, int W,
                                      const uint8_t* coins_host, int K, double gamma, double p,
                                      double alpha, int n_inner, int accelerated, int nonneg,
                                      double* last_weight_host, int64_t* prox_count_host,
                                      int32_t* bad_iter, const int32_t* ready, int32_t* done,
                                      const int64_t* bounds_host, int n_chunks, void* stream);
/* Stream memory operations (cuStreamWriteValue32 / cuStreamWaitValue32 with
 * GEQ), used to order copies against the streamed run without a host
 * round trip; psb_stream_memops_supported reports whether the driver has them. */
int psb_stream_memops_supported(int* out);
int psb_stream_write_u32(void* stream, void* dptr, uint32_t value);
int psb_stream_wait_geq_u32(void* stream, void* dptr, uint32_t value);
/* psb_chunked_h2d / psb_chunked_d2h: the streamed batch's copies, enqueued in
 * one call each (items of item_bytes; chunk c = items [bounds[c], bounds[c+1]),
 * bounds a host int64 array of n_chunks + 1).  H2D: copy
 * chunk c from page-locked host memory, then ready[c] = 1 (fenced stream
 * write).  D2H: wait until done[c] >= unit * (items in chunk c) (stream wait),
 * then copy chunk c to page-locked host memory.  Replaces the per-chunk copy
 * loop of run_proxskip_batched's streamed path. */
int psb_chunked_h2d(void* dst, const void* src_host, int64_t item_bytes, const int64_t* bounds,
                    int n_chunks, int32_t* ready, void* stream);
int psb_chunked_d2h(void* dst_host, const void* src, int64_t item_bytes, const int64_t* bounds,
                    int n_chunks, const int32_t* done, uint32_t unit, void* stream);

/* Peer memory for the config-5 z-slab exchange (the reference has
 * no multi-GPU path -- this replaces the halo transfer of the decomposed
 * tv.py:53-89 loop).  A rank exports its halo receive rings and flags with
 * psb_ipc_get_handle (psb_ipc_handle_size() bytes), its neighbours map them
 * with psb_ipc_open_handle and deposit planes there: the edge kernel's
 * send_lo / send_hi stores (psb_fgp3d_iter_part) or psb_copy_async, each
 * followed by psb_stream_write_u32 on the receiver's flag. */
int psb_copy_async(void* dst, const void* src, int64_t bytes, void* stream);
int psb_ipc_handle_size(void);
int psb_ipc_get_handle(const void* dptr, void* handle_out, int64_t* offset);
int psb_ipc_open_handle(const void* handle, void** dptr_out);
int psb_ipc_close(void* dptr);

/* ---- parallel-beam projector, operators.py:189-292 (matrix-free) ------------
 * Geometry of RadonGeometry (operators.py:189-215) plus the sample lattice of
 * radon_system_matrix (operators.py:224-229): `tables` is a DEVICE double
 * array [offsets (n_bins) | steps (n_steps) | cos(angles) | sin(angles)]
 * computed on the host with numpy exactly as the reference does, so sample
 * positions are bit-identical.  step_spacing = 2*half_span/(n_steps-1). */
typedef struct psb_radon_geom {
  int n;
  int n_angles;
  int n_bins;
  int n_steps;
  double center;
  double half_span;
  double step_spacing;
  double bin_spacing;
  const double* tables;
} psb_radon_geom;

/* psb_radon_fwd: sino = A img (CSR SpMV of operators.py:273-277, ray-driven)
 * psb_radon_adj: img = A^T sino (operators.py:279-283, pixel-driven gather,
 *   the exact transpose of psb_radon_fwd's weights) */
int psb_radon_fwd(int dtype, const psb_radon_geom* geom, const void* img, void* sino, void* stream);
int psb_radon_adj(int dtype, const psb_radon_geom* geom, const void* sino, void* img, void* stream);

/* ---- PDHG / PDHGSkip-2 on K = [A; D] (explicit splitting, BASELINE config 3)
 * y is the reference's flat dual [y_A (n_angles*n_bins) | y_D (2*n*n)]
 * (problems.py:136-146); b the sinogram.  One step =
 *   primal (fused A^T y_A - div y_D, prox_g = max(., 0) when nonneg, the
 *   ProxSkip control variate when h != NULL, xbar = 2x' - x),
 *   dual fidelity ((y_A + tau A xbar) - tau b)/(1 + tau),
 *   dual TV P_alpha(y_D + tau grad xbar).
 * h == NULL: plain PDHG (solvers.py:187-209); else PDHGSkip-2 (skip.py:117-150)
 * with coin = this iteration's Bernoulli draw, hcoef = sigma - sigma/p,
 * ps = p/sigma.  psb_pdhg_run loops K steps (coins_host: host uint8[K]; skip=0
 * runs PDHG), optionally as one CUDA graph; sigma_arr (n*n) / tau_arr (the
 * flat dual length) are the optional diagonal (Pock-Chambolle) steps of
 * run_pdhg_preconditioned (solvers.py:212-234), PDHG only.  skip: 0 PDHG,
 * 1 PDHGSkip-2 (h = control variate), 2 PDHGSkip-1 (skip.py:82-114, omega;
 * K^T and the prox only on success draws). */
int psb_pdhg_step(int dtype, const psb_radon_geom* geom, void* x, void* y, void* h, void* xbar,
                  const void* b, int32_t* bad_iter, int k, int coin, double sigma, double tau,
                  double hcoef, double ps, double alpha, int nonneg, void* stream);
int psb_pdhg_run(int dtype, const psb_radon_geom* geom, void* x, void* y, void* h, void* xbar,
                 const void* b, const uint8_t* coins_host, int K, double sigma, double tau,
                 const void* sigma_arr, const void* tau_arr, double p, double alpha, int nonneg,
                 int skip, double omega, int32_t* bad_iter, int use_graph, double* elapsed_host,
                 void* x_hist, void* stream);

/* PDHGSkip-2 / PDHG on the implicit splitting K = A (Radon), TV in the
 * warm-started FGP prox with optional u >= 0 (problems.py:162-184,
 * skip.py:117-150).  y: sinogram (n_angles*n_bins, dtype_outer);
 * h, xbar: n*n (dtype_outer); z: n*n and q: 3*2*n*n FGP slots (dtype_fgp,
 * q_warm in slot 0); p = 1 with all coins set is PDHG.  last_weight_host /
 * prox_count_host are the TvProxState accounting (in/out). */
int psb_ct_implicit_run(int dtype_outer, int dtype_fgp, const psb_radon_geom* geom, void* x,
                        void* y, void* h, void* xbar, void* z, void* q, const void* b,
                        const uint8_t* coins_host, int K, double sigma, double tau, double p,
                        double alpha, int n_inner, int accelerated, int nonneg,
                        double* last_weight_host, int64_t* prox_count_host, int32_t* bad_iter,
                        int use_graph, double* elapsed_host, void* x_hist, void* stream);

/* ---- 3-D TV prox + ProxSkip for BASELINE config 5 -----
 * Volume (D, H, W) with dual channels (z, y, x), dual step 1/12 (pass it as
 * `step`), the 2-D reference algorithm otherwise.  Slots as in 2-D, each of
 * (3, D, H, W).  z-slab decomposition: this call owns planes [z0, z0+D) of a
 * volume of depth Dg; halo_below_* are plane z0-1 of q_it / q_{it-1} (3, H, W)
 * (NULL when z0 == 0), halo_above_* plane z0+D of q_it / q_{it-1} and of x
 * (NULL when z0+D == Dg).  zchunk <= 0 picks the z-chunk per CTA.
 * psb_proxskip_post3d: identity-fidelity ProxSkip post fused with the 3-D
 * finalize; halo_below_qn = plane z0-1 of the final dual iterate; `pend`
 * deferred skip iterations are applied to x (in registers) before x-hat. */
int psb_fgp3d_iter(int dtype, const void* x, void* q, int D, int H, int W, int z0, int Dg, int it,
                   double beta_prev, double step, double weight, int reproject, int nonneg,
                   const void* halo_below_qk, const void* halo_below_qm, const void* halo_above_qk,
                   const void* halo_above_qm, const void* halo_above_x, int zchunk, void* stream);
/* psb_fgp3d_iter_part: psb_fgp3d_iter restricted to a plane subset, for the
 * overlapped slab schedule: part 1 = interior planes [1, D-1),
 * which read no halo plane and so run while the halo exchange is in flight;
 * part 2 = the edge planes 0 and D-1, launched once the halos have arrived.
 * send_lo / send_hi (optional, (3, H, W)) receive a copy of the new q_{it+1}
 * of plane 0 / D-1 from the same store -- a local send buffer or, for the
 * peer-memory exchange, the neighbour's receive ring mapped over NVLink.
 * part 0 = all planes (psb_fgp3d_iter). */
int psb_fgp3d_iter_part(int dtype, const void* x, void* q, int D, int H, int W, int z0, int Dg,
                        int it, double beta_prev, double step, double weight, int reproject,
                        int nonneg, const void* halo_below_qk, const void* halo_below_qm,
                        const void* halo_above_qk, const void* halo_above_qm,
                        const void* halo_above_x, int zchunk, int part, void* send_lo,
                        void* send_hi, void* stream);
int psb_proxskip_post3d(int dtype_outer, int dtype_fgp, void* x, const void* b, void* h,
                        const void* z, void* q, const void* halo_below_qn, int D, int H, int W,
                        int z0, int Dg, int n_inner, int nonneg, double gamma, double pg,
                        int pend, int32_t* bad_iter, int k, void* stream);

/* psb_cluster_max_active: how many 16-CTA clusters of the cluster-resident
 * 256x256 ProxSkip kernel (csrc/fgp_cluster.cu: fp64 outer state and small
 * batches; fp32 batches run on the 8-CTA kernel, csrc/fgp_cluster8.cu) fit
 * on the device. */
int psb_cluster_max_active(int* out);

/* psb_queue_stats: work-queue statistics of the last cluster-path run
 * (psb_proxskip_denoise_run[_streamed]) -- out6 = {ns, cost units} of the
 * 16-CTA clusters, of the SM workers and of the 8-CTA clusters, summed over
 * finished problems (cost unit = one FGP inner iteration of one 256x256
 * problem; +2 per problem).  Valid once the run's stream has been synchronised. */
int psb_queue_stats(double* out6);

/* psb_proxskip_deblur_run: the same native driver for the implicit TV
 *   deblurring problem (BASELINE config 2): A = periodic blur, one problem,
 *   the gradient A^T(Ax - b) recomputed every outer iteration into `g`
 *   (device, H*W of dtype_outer) by psb_blur_grad2d (`scratch` is needed only
 *   when separable == 0). */
int psb_proxskip_deblur_run(int dtype_outer, int dtype_fgp, void* x, const void* b, void* h,
                            void* z, void* q, void* g, void* scratch, int H, int W,
                            const double* taps2d, const double* taps1d, int ksize, int separable,
                            const uint8_t* coins_host, int K, double gamma, double p, double alpha,
                            int n_inner, int accelerated, int nonneg, double* last_weight_host,
                            int64_t* prox_count_host, int32_t* bad_iter, int use_graph,
                            double* elapsed_host, double* fgp_time_host, void* x_hist, int algo,
                            void* aux, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PSB200_H_ */

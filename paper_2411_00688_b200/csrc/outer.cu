// ProxSkip outer update (skip.py:46-79), split around the FGP prox:
//   pre  : skipped problems take x <- xhat = (x - gamma g) + gamma h,
//          coin-fired problems get the prox input z = (x - gamma g) + hcoef h
//   post : fused FGP finalize u = clamp(z + div q_n) (tv.py:89) + control
//          variate h <- h + (p/gamma)(u - xhat), x <- u
// For the identity fidelity g = x - b is fused (problems.py:121 with
// operators.py:297-307).  Outer state may be fp64 while the FGP runs in fp32
// (config 2 needs fp64 x/h/gradient).
#include <climits>

#include "common.cuh"

namespace psb {

namespace {

template <class TO, bool IDENT>
__device__ __forceinline__ TO grad_at(TO xo, const TO* gb, int64_t o) {
  using A = Ar<TO>;
  return IDENT ? A::sub(xo, gb[o]) : gb[o];
}

template <class TO, class TF, bool IDENT>
__global__ void proxskip_pre_kernel(TO* __restrict__ x, const TO* __restrict__ gb,
                                    const TO* __restrict__ h, TF* __restrict__ z, int64_t HW,
                                    const uint8_t* __restrict__ coins, TO gamma, TO hcoef,
                                    int32_t* __restrict__ bad, int k) {
  using A = Ar<TO>;
  pdl_enter();
  const int64_t p = blockIdx.y;
  const bool theta = coins ? coins[p] != 0 : true;
  const int64_t base = p * HW;
  bool ok = true;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < HW;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = base + i;
    const TO xo = x[o];
    const TO t = A::sub(xo, A::mul(gamma, grad_at<TO, IDENT>(xo, gb, o)));
    if (theta) {
      z[o] = (TF)A::add(t, A::mul(hcoef, h[o]));
    } else {
      const TO xn = A::add(t, A::mul(gamma, h[o]));
      x[o] = xn;
      ok &= finite(xn);
    }
  }
  if (!ok && bad) atomicMin(bad + p, k);
}

template <class TO, class TF, bool IDENT>
__global__ void proxskip_post_kernel(TO* __restrict__ x, const TO* __restrict__ gb,
                                     TO* __restrict__ h, const TF* __restrict__ z, TF* q,
                                     int64_t qps, const int32_t* __restrict__ active, int H, int W,
                                     int n_inner, int nonneg, TO gamma, TO pg,
                                     int32_t* __restrict__ bad, int k) {
  using A = Ar<TO>;
  using F = Ar<TF>;
  pdl_enter();
  const int p = active ? active[blockIdx.y] : (int)blockIdx.y;
  const int64_t HW = (int64_t)H * W;
  const int slot = n_inner % 3;
  TF* qb = q + (int64_t)p * qps;
  const TF* qn = qb + (int64_t)slot * 2 * HW;
  const int64_t base = (int64_t)p * HW;
  bool ok = true;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < HW;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / W), c = (int)(i % W);
    const TF yy = qn[i], yx = qn[HW + i];
    TF d = TF(0);
    if (r < H - 1) d = F::add(d, yy);
    if (r > 0) d = F::sub(d, qn[i - W]);
    if (c < W - 1) d = F::add(d, yx);
    if (c > 0) d = F::sub(d, qn[HW + i - 1]);
    TF uf = F::add(z[base + i], d);
    if (nonneg) uf = uf > TF(0) ? uf : TF(0);
    if (slot != 0) {
      qb[i] = yy;
      qb[HW + i] = yx;
    }
    const int64_t o = base + i;
    const TO xn = (TO)uf;
    if (h) {  // ProxSkip control variate (skip.py:74); FISTA passes h = NULL
      const TO xo = x[o], ho = h[o];
      const TO xhat = A::add(A::sub(xo, A::mul(gamma, grad_at<TO, IDENT>(xo, gb, o))), A::mul(gamma, ho));
      h[o] = A::add(ho, A::mul(pg, A::sub(xn, xhat)));
    }
    x[o] = xn;
    ok &= finite(xn);
  }
  if (!ok && bad) atomicMin(bad + p, k);
}

template <class TO, class TF>
void launch_pre(void* x, const void* gb, int ident, const void* h, void* z, int64_t n, int64_t HW,
                const uint8_t* coins, double gamma, double hcoef, int32_t* bad, int k,
                cudaStream_t st) {
  dim3 block(256);
  const int64_t want = (HW + 255) / 256;
  dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(want, std::max<int64_t>(1, 4LL * sm_count() * 8 / std::max<int64_t>(n, 1)))), (unsigned)n);
  if (ident)
    (void)launch_chain(proxskip_pre_kernel<TO, TF, true>, grid, block, 0, st, (TO*)x,
                       (const TO*)gb, (const TO*)h, (TF*)z, HW, coins, (TO)gamma, (TO)hcoef, bad, k);
  else
    (void)launch_chain(proxskip_pre_kernel<TO, TF, false>, grid, block, 0, st, (TO*)x,
                       (const TO*)gb, (const TO*)h, (TF*)z, HW, coins, (TO)gamma, (TO)hcoef, bad, k);
}

template <class TO, class TF>
void launch_post(void* x, const void* gb, int ident, void* h, const void* z, void* q, int64_t qps,
                 const int32_t* active, int n_active, int H, int W, int n_inner, int nonneg,
                 double gamma, double pg, int32_t* bad, int k, cudaStream_t st) {
  const int64_t HW = (int64_t)H * W;
  dim3 block(256);
  const int64_t want = (HW + 255) / 256;
  dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(want, std::max<int64_t>(1, 4LL * sm_count() * 8 / n_active))), (unsigned)n_active);
  if (ident)
    (void)launch_chain(proxskip_post_kernel<TO, TF, true>, grid, block, 0, st, (TO*)x,
                       (const TO*)gb, (TO*)h, (const TF*)z, (TF*)q, qps, active, H, W, n_inner,
                       nonneg, (TO)gamma, (TO)pg, bad, k);
  else
    (void)launch_chain(proxskip_post_kernel<TO, TF, false>, grid, block, 0, st, (TO*)x,
                       (const TO*)gb, (TO*)h, (const TF*)z, (TF*)q, qps, active, H, W, n_inner,
                       nonneg, (TO)gamma, (TO)pg, bad, k);
}

// Deferred skip iterations of the identity-fidelity ProxSkip (skip.py:68 with
// h unchanged, repeated `pend` times in registers, bit-identical to `pend`
// separate passes).  z != NULL: write the prox input z = (x_m - g(x_m - b)) +
// hc h without storing x_m (the post kernel recomputes it); z == NULL: store
// x_m (flush).
template <class TO, class TF>
__global__ void skip_chain_kernel(TO* __restrict__ x, const TO* __restrict__ b,
                                  const TO* __restrict__ h, TF* __restrict__ z, int64_t count,
                                  int pend, TO gamma, TO hcoef, int32_t* bad, int kfirst) {
  using A = Ar<TO>;
  int kbad = 0x7fffffff;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const TO bo = b[i], ho = h[i];
    const TO xo = skip_chain_px(x[i], bo, ho, gamma, pend, kfirst, &kbad);
    if (z)
      z[i] = (TF)A::add(A::sub(xo, A::mul(gamma, A::sub(xo, bo))), A::mul(hcoef, ho));
    else
      x[i] = xo;
  }
  if (kbad != 0x7fffffff && bad) atomicMin(bad, kbad);
}

}  // namespace

int skip_chain(int dto, int dtf, void* x, const void* b, const void* h, void* z, int64_t count,
               int pend, double gamma, double hcoef, int32_t* bad, int kfirst, cudaStream_t st) {
  PSB_REQUIRE(pend >= 0, "skip chain: negative count");
  if (count == 0 || (pend == 0 && z == nullptr)) return PSB_OK;
  dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, 16LL * sm_count())));
  if (dto == PSB_F32 && dtf == PSB_F32)
    skip_chain_kernel<float, float><<<grid, 256, 0, st>>>((float*)x, (const float*)b, (const float*)h,
                                                         (float*)z, count, pend, (float)gamma,
                                                         (float)hcoef, bad, kfirst);
  else if (dto == PSB_F64 && dtf == PSB_F32)
    skip_chain_kernel<double, float><<<grid, 256, 0, st>>>((double*)x, (const double*)b,
                                                          (const double*)h, (float*)z, count, pend,
                                                          gamma, hcoef, bad, kfirst);
  else if (dto == PSB_F64 && dtf == PSB_F64)
    skip_chain_kernel<double, double><<<grid, 256, 0, st>>>((double*)x, (const double*)b,
                                                           (const double*)h, (double*)z, count,
                                                           pend, gamma, hcoef, bad, kfirst);
  else
    return fail(PSB_ERR_VALUE, "skip chain: unsupported dtype pair");
  PSB_LAUNCHED("skip_chain");
  return PSB_OK;
}

// ---- FISTA on the implicit splitting (solvers.py:148-168) -------------------
// xbar = x + beta (x - x_prev), x_prev <- x; then the prox input
// z = xbar - gamma g(xbar) (identity: g = xbar - b; blur: g from
// blur_grad2d(xbar)), the FGP prox, and the post kernel with h = NULL (x = u).
template <class TO>
__global__ void fista_extrap_kernel(TO* __restrict__ x, TO* __restrict__ xprev,
                                    TO* __restrict__ xbar, int64_t count, TO beta) {
  using A = Ar<TO>;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const TO xo = x[i];
    xbar[i] = A::add(xo, A::mul(beta, A::sub(xo, xprev[i])));
    xprev[i] = xo;
  }
}

template <class TO, class TF, bool IDENT>
__global__ void fista_pre_kernel(const TO* __restrict__ xbar, const TO* __restrict__ gb,
                                 TF* __restrict__ z, int64_t count, TO gamma) {
  using A = Ar<TO>;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const TO xb = xbar[i];
    const TO g = IDENT ? A::sub(xb, gb[i]) : gb[i];
    z[i] = (TF)A::add(xb, A::mul(-gamma, g));
  }
}

int fista_extrap(int dto, void* x, void* xprev, void* xbar, int64_t count, double beta,
                 cudaStream_t st) {
  const dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, 16LL * sm_count())));
  if (dto == PSB_F32)
    fista_extrap_kernel<float><<<grid, 256, 0, st>>>((float*)x, (float*)xprev, (float*)xbar, count,
                                                     (float)beta);
  else
    fista_extrap_kernel<double><<<grid, 256, 0, st>>>((double*)x, (double*)xprev, (double*)xbar,
                                                      count, beta);
  PSB_LAUNCHED("fista_extrap");
  return PSB_OK;
}

int fista_pre(int dto, int dtf, const void* xbar, const void* gb, int ident, void* z, int64_t count,
              double gamma, cudaStream_t st) {
  const dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, 16LL * sm_count())));
  auto go = [&](auto to, auto tf) {
    using TO = decltype(to);
    using TF = decltype(tf);
    if (ident)
      fista_pre_kernel<TO, TF, true><<<grid, 256, 0, st>>>((const TO*)xbar, (const TO*)gb, (TF*)z,
                                                           count, (TO)gamma);
    else
      fista_pre_kernel<TO, TF, false><<<grid, 256, 0, st>>>((const TO*)xbar, (const TO*)gb, (TF*)z,
                                                            count, (TO)gamma);
  };
  if (dto == PSB_F32 && dtf == PSB_F32)
    go(float{}, float{});
  else if (dto == PSB_F64 && dtf == PSB_F32)
    go(double{}, float{});
  else if (dto == PSB_F64 && dtf == PSB_F64)
    go(double{}, double{});
  else
    return fail(PSB_ERR_VALUE, "fista: unsupported dtype pair");
  PSB_LAUNCHED("fista_pre");
  return PSB_OK;
}

int proxskip_pre(int dto, int dtf, void* x, const void* gb, int ident, const void* h, void* z,
                 int64_t n, int64_t HW, const uint8_t* coins, double gamma, double hcoef,
                 int32_t* bad, int k, cudaStream_t st) {
  PSB_REQUIRE(n >= 0 && n <= 65535, "proxskip: batch size out of range");
  PSB_REQUIRE(gamma > 0, "run_proxskip: gamma must be positive");
  if (n == 0 || HW == 0) return PSB_OK;
  if (dto == PSB_F32 && dtf == PSB_F32)
    launch_pre<float, float>(x, gb, ident, h, z, n, HW, coins, gamma, hcoef, bad, k, st);
  else if (dto == PSB_F64 && dtf == PSB_F32)
    launch_pre<double, float>(x, gb, ident, h, z, n, HW, coins, gamma, hcoef, bad, k, st);
  else if (dto == PSB_F64 && dtf == PSB_F64)
    launch_pre<double, double>(x, gb, ident, h, z, n, HW, coins, gamma, hcoef, bad, k, st);
  else
    return fail(PSB_ERR_VALUE, "proxskip: unsupported dtype pair (outer must be >= fgp)");
  PSB_LAUNCHED("proxskip_pre");
  return PSB_OK;
}

int proxskip_post(int dto, int dtf, void* x, const void* gb, int ident, void* h, const void* z,
                  void* q, int64_t qps, const int32_t* active, int n_active, int H, int W,
                  int n_inner, int nonneg, double gamma, double pg, int32_t* bad, int k,
                  cudaStream_t st) {
  PSB_REQUIRE(n_active >= 0 && n_active <= 65535, "proxskip: batch size out of range");
  if (n_active == 0) return PSB_OK;
  if (dto == PSB_F32 && dtf == PSB_F32)
    launch_post<float, float>(x, gb, ident, h, z, q, qps, active, n_active, H, W, n_inner, nonneg,
                              gamma, pg, bad, k, st);
  else if (dto == PSB_F64 && dtf == PSB_F32)
    launch_post<double, float>(x, gb, ident, h, z, q, qps, active, n_active, H, W, n_inner, nonneg,
                               gamma, pg, bad, k, st);
  else if (dto == PSB_F64 && dtf == PSB_F64)
    launch_post<double, double>(x, gb, ident, h, z, q, qps, active, n_active, H, W, n_inner,
                                nonneg, gamma, pg, bad, k, st);
  else
    return fail(PSB_ERR_VALUE, "proxskip: unsupported dtype pair (outer must be >= fgp)");
  PSB_LAUNCHED("proxskip_post");
  return PSB_OK;
}

}  // namespace psb

extern "C" {

int psb_proxskip_pre(int dtype_outer, int dtype_fgp, void* x, const void* g_or_b, int ident,
                     const void* h, void* z, int64_t n, int64_t HW, const uint8_t* coins,
                     double gamma, double hcoef, int32_t* bad_iter, int k, void* stream) {
  return psb::proxskip_pre(dtype_outer, dtype_fgp, x, g_or_b, ident, h, z, n, HW, coins, gamma,
                           hcoef, bad_iter, k, psb::as_stream(stream));
}

int psb_proxskip_post(int dtype_outer, int dtype_fgp, void* x, const void* g_or_b, int ident,
                      void* h, const void* z, void* q, int64_t q_pstride, const int32_t* active,
                      int n_active, int H, int W, int n_inner, int nonneg, double gamma, double pg,
                      int32_t* bad_iter, int k, void* stream) {
  return psb::proxskip_post(dtype_outer, dtype_fgp, x, g_or_b, ident, h, z, q, q_pstride, active,
                            n_active, H, W, n_inner, nonneg, gamma, pg, bad_iter, k,
                            psb::as_stream(stream));
}

int psb_skip_chain(int dtype_outer, int dtype_fgp, void* x, const void* b, const void* h, void* z,
                   int64_t count, int pend, double gamma, double hcoef, int32_t* bad_iter,
                   int kfirst, void* stream) {
  return psb::skip_chain(dtype_outer, dtype_fgp, x, b, h, z, count, pend, gamma, hcoef, bad_iter,
                         kfirst, psb::as_stream(stream));
}

}  // extern "C"

// Stand-alone operators of the reference's L2 layer, used by the Python
// LinearMap / prox shims (grad_map, divergence, project_ball, project_nonneg)
// and by the PDHG drivers.  Batched over n images with stride H*W.
#include "common.cuh"

namespace psb {

namespace {

// operators.py:44-57
template <class T>
__global__ void grad2d_kernel(const T* __restrict__ u, T* __restrict__ g, int64_t n, int H, int W) {
  using A = Ar<T>;
  const int64_t HW = (int64_t)H * W;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n * HW;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = idx / HW, i = idx % HW;
    const int r = (int)(i / W), c = (int)(i % W);
    const T* up = u + p * HW;
    T* gp = g + p * 2 * HW;
    const T v = up[i];
    gp[i] = r < H - 1 ? A::sub(up[i + W], v) : T(0);
    gp[HW + i] = c < W - 1 ? A::sub(up[i + 1], v) : T(0);
  }
}

// operators.py:60-71
template <class T>
__global__ void div2d_kernel(const T* __restrict__ q, T* __restrict__ d, int64_t n, int H, int W) {
  using A = Ar<T>;
  const int64_t HW = (int64_t)H * W;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n * HW;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = idx / HW, i = idx % HW;
    const int r = (int)(i / W), c = (int)(i % W);
    const T* qy = q + p * 2 * HW;
    const T* qx = qy + HW;
    T s = T(0);
    if (r < H - 1) s = A::add(s, qy[i]);
    if (r > 0) s = A::sub(s, qy[i - W]);
    if (c < W - 1) s = A::add(s, qx[i]);
    if (c > 0) s = A::sub(s, qx[i - 1]);
    d[p * HW + i] = s;
  }
}

// proximal.py:10-21 -- always the exactly-rounded formula here (this kernel is
// not on the FGP hot loop; the fused kernels use Ar<float>::ball_scale).
template <class T>
__global__ void ball2d_kernel(const T* __restrict__ q, T* __restrict__ out, int64_t n, int64_t HW,
                              T r) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n * HW;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = idx / HW, i = idx % HW;
    const T a = q[p * 2 * HW + i], b = q[p * 2 * HW + HW + i];
    T s;
    if constexpr (sizeof(T) == 8) {
      s = Ar<double>::ball_scale(a, b, r);
    } else {
      const float m = __fsqrt_rn(__fadd_rn(__fmul_rn(a, a), __fmul_rn(b, b)));
      s = __fdiv_rn(r, fmaxf(r, m));
    }
    out[p * 2 * HW + i] = a * s;
    out[p * 2 * HW + HW + i] = b * s;
  }
}

template <class T>
__global__ void nonneg_kernel(const T* __restrict__ u, T* __restrict__ out, int64_t count) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < count;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const T v = u[idx];
    out[idx] = v > T(0) ? v : (v == v ? T(0) : v);  // np.maximum propagates NaN
  }
}

// out = (a*x) + (b*y), each product rounded separately; a == 1 skips the
// first multiply and y == NULL drops the second term, so the drivers can
// spell the reference's expressions exactly (e.g. x - gamma*g as
// lincomb(1, x, -gamma, g); -gamma*g == -(gamma*g) in IEEE arithmetic).
template <class T>
__global__ void lincomb_kernel(T a, const T* __restrict__ x, T b, const T* __restrict__ y,
                               T* __restrict__ out, int64_t count) {
  using A = Ar<T>;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < count;
       idx += (int64_t)gridDim.x * blockDim.x) {
    T t = a == T(1) ? x[idx] : A::mul(a, x[idx]);
    if (y) t = A::add(t, A::mul(b, y[idx]));
    out[idx] = t;
  }
}

// out = x + sgn * (s .* y) with an ARRAY coefficient s (diagonal PDHG steps,
// solvers.py:200-204): x - sigma*K^T y (sgn = -1), y + tau*K xbar (sgn = +1).
template <class T>
__global__ void axpy_arr_kernel(const T* __restrict__ x, int sgn, const T* __restrict__ sc,
                                const T* __restrict__ y, T* __restrict__ out, int64_t count) {
  using A = Ar<T>;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T t = A::mul(sc[i], y[i]);
    out[i] = sgn < 0 ? A::sub(x[i], t) : A::add(x[i], t);
  }
}

// conjugate prox of 0.5||. - b||^2: (v - t b) / (1 + t), t scalar (t_arr == NULL)
// or per element (problems.py:143-144, 178)
template <class T>
__global__ void fidprox_kernel(const T* __restrict__ v, T t, const T* __restrict__ t_arr,
                               const T* __restrict__ b, T* __restrict__ out, int64_t count) {
  using A = Ar<T>;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T ti = t_arr ? t_arr[i] : t;
    out[i] = A::div(A::sub(v[i], A::mul(ti, b[i])), A::add(T(1), ti));
  }
}

// graph-replayed iteration loops: non-finite check against an iteration
// counter kept in device memory (solvers.py:111-113, first bad k)
template <class T>
__global__ void mark_nonfinite_kernel(const T* __restrict__ x, int64_t count,
                                      int32_t* __restrict__ bad, const int32_t* __restrict__ ctr) {
  bool hit = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    hit |= !isfinite((double)x[i]);
  if (__syncthreads_or(hit) && threadIdx.x == 0) atomicMin(bad, *ctr);
}

__global__ void counter_add_kernel(int32_t* ctr, int v) { *ctr += v; }

// prox of 0.5||z - b||^2 with step t at x: (x + t b) / (1 + t)  (proximal.py:44-55)
template <class T>
__global__ void prox_l2_fid_kernel(const T* __restrict__ x, T t, const T* __restrict__ t_arr,
                                   const T* __restrict__ b, T* __restrict__ out, int64_t count) {
  using A = Ar<T>;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T ti = t_arr ? t_arr[i] : t;
    out[i] = A::div(A::add(x[i], A::mul(ti, b[i])), A::add(T(1), ti));
  }
}

// 1 / max(x, floor)  (diagonal_steps, solvers.py:212-224)
template <class T>
__global__ void recip_floor_kernel(const T* __restrict__ x, T fl, T* __restrict__ out,
                                   int64_t count) {
  using A = Ar<T>;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T v = x[i];
    out[i] = A::div(T(1), v > fl ? v : (v == v ? fl : v));
  }
}

// |D| u and |D|^T q (operators.py:81-94): the entrywise-absolute gradient maps
template <class T>
__global__ void absgrad2d_kernel(const T* __restrict__ u, T* __restrict__ g, int H, int W) {
  using A = Ar<T>;
  const int64_t HW = (int64_t)H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < HW;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / W), c = (int)(i % W);
    g[i] = r < H - 1 ? A::add(u[i + W], u[i]) : T(0);
    g[HW + i] = c < W - 1 ? A::add(u[i + 1], u[i]) : T(0);
  }
}

template <class T>
__global__ void absdiv2d_kernel(const T* __restrict__ q, T* __restrict__ d, int H, int W) {
  using A = Ar<T>;
  const int64_t HW = (int64_t)H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < HW;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / W), c = (int)(i % W);
    T s = T(0);
    if (r < H - 1) s = A::add(s, q[i]);
    if (r > 0) s = A::add(s, q[i - W]);
    if (c < W - 1) s = A::add(s, q[HW + i]);
    if (c > 0) s = A::add(s, q[HW + i - 1]);
    d[i] = s;
  }
}

inline dim3 grid_for(int64_t count) {
  return dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, 32LL * sm_count())));
}

}  // namespace

}  // namespace psb

extern "C" {

int psb_grad2d(int dtype, const void* u, void* g, int64_t n, int H, int W, void* stream) {
  PSB_REQUIRE(H >= 2 && W >= 2, "grad_forward: need a 2-D grid with both sides >= 2");
  const int64_t cnt = n * H * (int64_t)W;
  if (cnt == 0) return PSB_OK;
  auto st = psb::as_stream(stream);
  if (dtype == PSB_F32)
    psb::grad2d_kernel<float><<<psb::grid_for(cnt), 256, 0, st>>>((const float*)u, (float*)g, n, H, W);
  else if (dtype == PSB_F64)
    psb::grad2d_kernel<double><<<psb::grid_for(cnt), 256, 0, st>>>((const double*)u, (double*)g, n, H, W);
  else
    return psb::fail(PSB_ERR_VALUE, "grad2d: unknown dtype");
  PSB_LAUNCHED("grad2d");
  return PSB_OK;
}

int psb_div2d(int dtype, const void* q, void* d, int64_t n, int H, int W, void* stream) {
  PSB_REQUIRE(H >= 2 && W >= 2, "divergence: expected (2, H, W) with H, W >= 2");
  const int64_t cnt = n * H * (int64_t)W;
  if (cnt == 0) return PSB_OK;
  auto st = psb::as_stream(stream);
  if (dtype == PSB_F32)
    psb::div2d_kernel<float><<<psb::grid_for(cnt), 256, 0, st>>>((const float*)q, (float*)d, n, H, W);
  else if (dtype == PSB_F64)
    psb::div2d_kernel<double><<<psb::grid_for(cnt), 256, 0, st>>>((const double*)q, (double*)d, n, H, W);
  else
    return psb::fail(PSB_ERR_VALUE, "div2d: unknown dtype");
  PSB_LAUNCHED("div2d");
  return PSB_OK;
}

int psb_project_ball2d(int dtype, const void* q, void* out, int64_t n, int64_t HW, double radius,
                       void* stream) {
  PSB_REQUIRE(radius > 0, "project_ball: alpha must be positive");
  const int64_t cnt = n * HW;
  if (cnt == 0) return PSB_OK;
  auto st = psb::as_stream(stream);
  if (dtype == PSB_F32)
    psb::ball2d_kernel<float><<<psb::grid_for(cnt), 256, 0, st>>>((const float*)q, (float*)out, n, HW, (float)radius);
  else if (dtype == PSB_F64)
    psb::ball2d_kernel<double><<<psb::grid_for(cnt), 256, 0, st>>>((const double*)q, (double*)out, n, HW, radius);
  else
    return psb::fail(PSB_ERR_VALUE, "project_ball: unknown dtype");
  PSB_LAUNCHED("project_ball2d");
  return PSB_OK;
}

int psb_lincomb(int dtype, double a, const void* x, double b, const void* y, void* out,
                int64_t count, void* stream) {
  if (count == 0) return PSB_OK;
  auto st = psb::as_stream(stream);
  if (dtype == PSB_F32)
    psb::lincomb_kernel<float><<<psb::grid_for(count), 256, 0, st>>>((float)a, (const float*)x, (float)b, (const float*)y, (float*)out, count);
  else if (dtype == PSB_F64)
    psb::lincomb_kernel<double><<<psb::grid_for(count), 256, 0, st>>>(a, (const double*)x, b, (const double*)y, (double*)out, count);
  else
    return psb::fail(PSB_ERR_VALUE, "lincomb: unknown dtype");
  PSB_LAUNCHED("lincomb");
  return PSB_OK;
}

#define PSB_DISPATCH(name, ...)                                                     \
  do {                                                                              \
    if (dtype == PSB_F32) {                                                         \
      using T = float;                                                              \
      __VA_ARGS__;                                                                  \
    } else if (dtype == PSB_F64) {                                                  \
      using T = double;                                                             \
      __VA_ARGS__;                                                                  \
    } else {                                                                        \
      return psb::fail(PSB_ERR_VALUE, name ": unknown dtype");                      \
    }                                                                               \
    PSB_LAUNCHED(name);                                                             \
    return PSB_OK;                                                                  \
  } while (0)

int psb_axpy_arr(int dtype, const void* x, int sign, const void* s, const void* y, void* out,
                 int64_t count, void* stream) {
  if (count == 0) return PSB_OK;
  auto st = psb::as_stream(stream);
  PSB_DISPATCH("axpy_arr", psb::axpy_arr_kernel<T><<<psb::grid_for(count), 256, 0, st>>>(
                               (const T*)x, sign, (const T*)s, (const T*)y, (T*)out, count));
}

int psb_fidprox(int dtype, const void* v, double t, const void* t_arr, const void* b, void* out,
                int64_t count, void* stream) {
  if (count == 0) return PSB_OK;
  auto st = psb::as_stream(stream);
  PSB_DISPATCH("fidprox", psb::fidprox_kernel<T><<<psb::grid_for(count), 256, 0, st>>>(
                              (const T*)v, (T)t, (const T*)t_arr, (const T*)b, (T*)out, count));
}

int psb_mark_nonfinite(int dtype, const void* x, int64_t count, int32_t* bad_iter,
                       const int32_t* iter_ctr, void* stream) {
  if (count == 0) return PSB_OK;
  auto st = psb::as_stream(stream);
  PSB_DISPATCH("mark_nonfinite", psb::mark_nonfinite_kernel<T><<<psb::grid_for(count), 256, 0, st>>>(
                                     (const T*)x, count, bad_iter, iter_ctr));
}

int psb_counter_add(int32_t* ctr, int v, void* stream) {
  psb::counter_add_kernel<<<1, 1, 0, psb::as_stream(stream)>>>(ctr, v);
  PSB_CUDA(cudaGetLastError());
  return PSB_OK;
}

int psb_prox_l2_fidelity(int dtype, const void* x, double t, const void* t_arr, const void* b,
                         void* out, int64_t count, void* stream) {
  if (count == 0) return PSB_OK;
  auto st = psb::as_stream(stream);
  PSB_DISPATCH("prox_l2_fidelity",
               psb::prox_l2_fid_kernel<T><<<psb::grid_for(count), 256, 0, st>>>(
                   (const T*)x, (T)t, (const T*)t_arr, (const T*)b, (T*)out, count));
}

int psb_recip_floor(int dtype, const void* x, double floor_, void* out, int64_t count,
                    void* stream) {
  if (count == 0) return PSB_OK;
  auto st = psb::as_stream(stream);
  PSB_DISPATCH("recip_floor", psb::recip_floor_kernel<T><<<psb::grid_for(count), 256, 0, st>>>(
                                  (const T*)x, (T)floor_, (T*)out, count));
}

int psb_absgrad2d(int dtype, const void* u, void* g, int H, int W, void* stream) {
  PSB_REQUIRE(H >= 2 && W >= 2, "grad_map: need a 2-D grid with both sides >= 2");
  auto st = psb::as_stream(stream);
  const int64_t cnt = (int64_t)H * W;
  PSB_DISPATCH("absgrad2d", psb::absgrad2d_kernel<T><<<psb::grid_for(cnt), 256, 0, st>>>(
                                (const T*)u, (T*)g, H, W));
}

int psb_absdiv2d(int dtype, const void* q, void* d, int H, int W, void* stream) {
  PSB_REQUIRE(H >= 2 && W >= 2, "grad_map: need a 2-D grid with both sides >= 2");
  auto st = psb::as_stream(stream);
  const int64_t cnt = (int64_t)H * W;
  PSB_DISPATCH("absdiv2d", psb::absdiv2d_kernel<T><<<psb::grid_for(cnt), 256, 0, st>>>(
                               (const T*)q, (T*)d, H, W));
}

int psb_project_nonneg(int dtype, const void* u, void* out, int64_t count, void* stream) {
  if (count == 0) return PSB_OK;
  auto st = psb::as_stream(stream);
  if (dtype == PSB_F32)
    psb::nonneg_kernel<float><<<psb::grid_for(count), 256, 0, st>>>((const float*)u, (float*)out, count);
  else if (dtype == PSB_F64)
    psb::nonneg_kernel<double><<<psb::grid_for(count), 256, 0, st>>>((const double*)u, (double*)out, count);
  else
    return psb::fail(PSB_ERR_VALUE, "project_nonneg: unknown dtype");
  PSB_LAUNCHED("project_nonneg");
  return PSB_OK;
}

}  // extern "C"

// Native drivers for the dual-ROF light-prox problems:
// build_dual_rof(b, alpha, huber_eps) (problems.py:22-84) solved by GD,
// PGD (= ProjGD), FISTA / AProjGD and ProxSkip (solvers.py:116-174,
// skip.py:46-79) -- the harness's denoise-dual / denoise-huber experiments.
//
// One launch per outer iteration, one thread per pixel (both dual channels):
// u = b + div q at the pixel and at its right / lower neighbours (recomputed
// from q, no second pass), g = -grad u (+ mu q) (problems.py:46-50), then the
// algorithm's update with the reference's operation order.  The
// iterate ping-pongs between slots; FISTA forms its extrapolation
// xbar = x + beta (x - x_prev) on the fly at every point it reads.
// Non-finite iterates are reported through an atomicMin of the iteration
// (solvers.py:111-113); the run can be captured as one CUDA graph.
#include <vector>

#include "common.cuh"

namespace psb {

namespace {

enum DualAlgo { ALGO_GD = 0, ALGO_PGD = 1, ALGO_FISTA = 2, ALGO_PROXSKIP = 3 };

template <class T>
struct DualArgs {
  const T* b;
  const T* x;      // current iterate (2, H, W)
  const T* xp;     // FISTA: previous iterate (2, H, W)
  T* out;          // next iterate
  T* h;            // ProxSkip control variate (in place)
  int H, W;
  T alpha, mu, gamma, beta, hc, pg;
  int algo, coin, k;
  int32_t* bad;
};

// iterate the gradient is evaluated at: x, or FISTA's x + beta (x - x_prev)
template <class T>
__device__ __forceinline__ T at(const DualArgs<T>& a, int64_t o) {
  using A = Ar<T>;
  if (a.algo != ALGO_FISTA) return a.x[o];
  const T v = a.x[o];
  return A::add(v, A::mul(a.beta, A::sub(v, a.xp[o])));
}

// u = b + div q at (i, j) in operators.py:66-70 order: ((0 + q0) - q0_up) + q1 - q1_left
template <class T>
__device__ __forceinline__ T u_at(const DualArgs<T>& a, int i, int j) {
  using A = Ar<T>;
  const int64_t HW = (int64_t)a.H * a.W, o = (int64_t)i * a.W + j;
  T d = T(0);
  if (i < a.H - 1) d = A::add(d, at(a, o));
  if (i > 0) d = A::sub(d, at(a, o - a.W));
  if (j < a.W - 1) d = A::add(d, at(a, HW + o));
  if (j > 0) d = A::sub(d, at(a, HW + o - 1));
  return A::add(d, a.b[o]);  // divergence(q) + b
}

template <class T>
__global__ void dual_rof_step_kernel(DualArgs<T> a) {
  using A = Ar<T>;
  const int64_t HW = (int64_t)a.H * a.W;
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o >= HW) return;
  const int i = (int)(o / a.W), j = (int)(o % a.W);
  const T u = u_at(a, i, j);
  const T gy = i < a.H - 1 ? A::sub(u_at(a, i + 1, j), u) : T(0);
  const T gx = j < a.W - 1 ? A::sub(u_at(a, i, j + 1), u) : T(0);
  const T q0 = at(a, o), q1 = at(a, HW + o);
  // g = -grad(div q + b), then + mu q for the Huber dual (problems.py:46-50)
  T g0 = A::mul(T(-1), gy), g1 = A::mul(T(-1), gx);
  if (a.mu != T(0)) {
    g0 = A::add(g0, A::mul(a.mu, q0));
    g1 = A::add(g1, A::mul(a.mu, q1));
  }
  // x - gamma g
  const T t0 = A::add(q0, A::mul(-a.gamma, g0)), t1 = A::add(q1, A::mul(-a.gamma, g1));
  T n0, n1;
  if (a.algo == ALGO_GD) {
    n0 = t0;
    n1 = t1;
  } else if (a.algo != ALGO_PROXSKIP) {
    const T s = A::ball_scale(t0, t1, a.alpha);  // project_ball (proximal.py:10-21)
    n0 = A::mul(t0, s);
    n1 = A::mul(t1, s);
  } else {
    const T h0 = a.h[o], h1 = a.h[HW + o];
    const T xh0 = A::add(t0, A::mul(a.gamma, h0)), xh1 = A::add(t1, A::mul(a.gamma, h1));
    if (a.coin) {
      const T z0 = A::add(t0, A::mul(a.hc, h0)), z1 = A::add(t1, A::mul(a.hc, h1));
      const T s = A::ball_scale(z0, z1, a.alpha);
      n0 = A::mul(z0, s);
      n1 = A::mul(z1, s);
    } else {
      n0 = xh0;
      n1 = xh1;
    }
    a.h[o] = A::add(h0, A::mul(a.pg, A::sub(n0, xh0)));
    a.h[HW + o] = A::add(h1, A::mul(a.pg, A::sub(n1, xh1)));
  }
  a.out[o] = n0;
  a.out[HW + o] = n1;
  if (a.bad && !(finite(n0) && finite(n1))) atomicMin(a.bad, a.k);
}

template <class T>
int run_t(int algo, const T* b, T* q, T* h, T* work, int H, int W, double alpha, double mu,
          double gamma, double p, const uint8_t* coins, int K, int32_t* bad, int use_graph,
          double* elapsed, void* x_hist, cudaStream_t user) {
  const int64_t HW = (int64_t)H * W;
  T* slot[3] = {q, work, work + 2 * HW};  // FISTA rotates three, the others ping-pong two
  const int nslot = algo == ALGO_FISTA ? 3 : 2;
  std::vector<double> beta(std::max(K, 1), 0.0);
  {
    double t = 1.0;  // solvers.py:156-160: beta_k = (t_k - 1) / t_{k+1}, t_0 = 1
    for (int k = 0; k < K; ++k) {
      const double t1 = (1.0 + std::sqrt(1.0 + 4.0 * t * t)) / 2.0;
      beta[k] = (t - 1.0) / t1;
      t = t1;
    }
  }
  const double hc = gamma - gamma / p, pg = p / gamma;  // skip.py:59-74
  CapturedRun cap;
  if (int rc0 = cap.begin(user, use_graph != 0)) return rc0;
  cudaStream_t st = cap.st;
  IterClock clk;
  clk.begin(elapsed, K, st, use_graph != 0);
  int rc = PSB_OK;
  int cur = 0, prev = 0;  // slot indices of x_k and x_{k-1}
  const unsigned grid = (unsigned)((HW + 255) / 256);
  for (int k = 0; k < K && rc == PSB_OK; ++k) {
    if (k > 0 && (rc = cap.tick(k - 1, K)) != PSB_OK) break;
    const int nxt = algo == ALGO_FISTA ? (cur + 1 + (cur + 1 == prev ? 1 : 0)) % nslot
                                       : (cur + 1) % nslot;
    DualArgs<T> a{b, slot[cur], slot[prev], slot[nxt], h, H, W, (T)alpha, (T)mu, (T)gamma,
                  (T)beta[k], (T)hc, (T)pg, algo, coins ? coins[k] : 1, k, bad};
    dual_rof_step_kernel<T><<<grid, 256, 0, st>>>(a);
    if (cudaGetLastError() != cudaSuccess) rc = fail(PSB_ERR_CUDA, "dual rof step launch failed");
    prev = cur;
    cur = nxt;
    clk.mark(k, st);
    if (x_hist && rc == PSB_OK &&
        cudaMemcpyAsync(static_cast<T*>(x_hist) + (int64_t)k * 2 * HW, slot[cur],
                        sizeof(T) * 2 * HW, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      rc = fail(PSB_ERR_CUDA, "x history copy failed");
  }
  // the final iterate goes back into q
  if (rc == PSB_OK && cur != 0 &&
      cudaMemcpyAsync(q, slot[cur], sizeof(T) * 2 * HW, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    rc = fail(PSB_ERR_CUDA, "dual rof result copy failed");
  rc = cap.end(rc);
  if (use_graph) cudaStreamSynchronize(user);
  clk.finish(elapsed, user, rc == PSB_OK);
  return rc;
}

}  // namespace

}  // namespace psb

extern "C" int psb_dual_rof_run(int dtype, int algo, const void* b, void* q, void* h, void* work,
                                int H, int W, double alpha, double huber_mu, double gamma,
                                double p, const uint8_t* coins_host, int K, int32_t* bad_iter,
                                int use_graph, double* elapsed_host, void* x_hist, void* stream) {
  PSB_REQUIRE(H >= 2 && W >= 2, "grad_forward: need a 2-D grid with both sides >= 2");
  PSB_REQUIRE(alpha > 0, "DualRofProblem: alpha must be positive");
  PSB_REQUIRE(huber_mu >= 0, "DualRofProblem: huber_eps must be nonnegative");
  PSB_REQUIRE(gamma > 0, "step must be positive");
  PSB_REQUIRE(algo >= 0 && algo <= 3, "dual rof: unknown algorithm");
  PSB_REQUIRE(algo != 3 || (p > 0 && p <= 1 && h != nullptr && coins_host != nullptr),
              "dual rof ProxSkip: needs 0 < p <= 1, the control variate and the coins");
  if (K <= 0) return PSB_OK;
  cudaStream_t st = psb::as_stream(stream);
  if (dtype == PSB_F64)
    return psb::run_t<double>(algo, (const double*)b, (double*)q, (double*)h, (double*)work, H, W,
                              alpha, huber_mu, gamma, p, coins_host, K, bad_iter, use_graph,
                              elapsed_host, x_hist, st);
  if (dtype == PSB_F32)
    return psb::run_t<float>(algo, (const float*)b, (float*)q, (float*)h, (float*)work, H, W,
                             alpha, huber_mu, gamma, p, coins_host, K, bad_iter, use_graph,
                             elapsed_host, x_hist, st);
  return psb::fail(PSB_ERR_VALUE, "dual rof: unknown dtype");
}

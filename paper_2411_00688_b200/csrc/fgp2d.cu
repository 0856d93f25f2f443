// FGP / accelerated dual projected gradient for the 2-D TV prox (tv.py:53-89).
//
// One launch = one inner iteration for a batch of problems.  Each warp owns a
// band of 32*V columns and marches down a strip of rows, keeping the previous
// row's dual y and primal u in registers (2.5-D register blocking): per pixel
// the kernel reads x (1), q_k (2), q_{k-1} (2) and writes q_{k+1} (2) -- the
// 28 B/pixel-iteration algorithmic minimum of SURVEY 8(d) for fp32 -- and
// recomputes y_k = q_k + beta (q_k - q_{k-1}) instead of storing it.  Column
// neighbours come from warp shuffles; the two band-edge columns come from one
// predicated scalar load per row by lanes 0 and 31.  Strip-edge rows are
// re-read (L2 hits).

#include "common.cuh"


namespace psb {

namespace {

template <class T, int V>
struct FgpArgs {
  const T* x;
  int64_t xps;
  T* q;
  int64_t qps;
  const int32_t* active;
  const double* wts;
  double w_all;
  const uint8_t* rep;
  int rep_all;
  int H, W, it;
  T beta;
  T step;
  int nonneg;
  int rs;      // rows per strip
  int nbands;  // column bands of 32*V
  int nitems;  // nbands * nstrips
};

// Load y = q_k + beta (q_k - q_m) at V consecutive pixels (both channels),
// re-projecting q_k first when `rp` (only at it == 0, where beta == 0).
template <class T, int V>
__device__ __forceinline__ void load_y(const T* qk, const T* qm, int64_t off, int64_t HW, bool mom,
                                       bool rp, T beta, T w, T (&yy)[V], T (&yx)[V]) {
  using A = Ar<T>;
  ldv<T, V>(yy, qk + off);
  ldv<T, V>(yx, qk + HW + off);
  if (rp) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      T s = A::ball_scale(yy[v], yx[v], w);
      yy[v] = A::mul(yy[v], s);
      yx[v] = A::mul(yx[v], s);
    }
  }
  if (mom) {
    T my[V], mx[V];
    ldv<T, V>(my, qm + off);
    ldv<T, V>(mx, qm + HW + off);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      yy[v] = A::add(yy[v], A::mul(beta, A::sub(yy[v], my[v])));
      yx[v] = A::add(yx[v], A::mul(beta, A::sub(yx[v], mx[v])));
    }
  }
}

// divergence at one pixel in the reference's accumulation order
// (operators.py:66-70): ((0 + [i<H-1] yy) - [i>0] yy_up) + [c<W-1] yx - [c>0] yx_left
template <class T>
__device__ __forceinline__ T div_at(int i, int c, int H, int W, T yy, T yy_up, T yx, T yx_left) {
  using A = Ar<T>;
  T d = T(0);
  if (i < H - 1) d = A::add(d, yy);
  if (i > 0) d = A::sub(d, yy_up);
  if (c < W - 1) d = A::add(d, yx);
  if (c > 0) d = A::sub(d, yx_left);
  return d;
}

template <class T>
__device__ __forceinline__ T clampu(T v, int nonneg) {
  return nonneg ? (v > T(0) ? v : T(0)) : v;  // np.maximum(v, 0); NaN -> 0 differs only for NaN
}

// Loads of the item: read-only path (one inner iteration per launch), or
// L2-coherent (CG: a persistent kernel that rewrites the same arrays between
// inner iterations must not hit stale L1 / texture lines).
template <bool CG, class T, int V>
__device__ __forceinline__ void ldq(T (&d)[V], const T* p) {
  if constexpr (CG && sizeof(T) * V == 16) {
    const float4 r = __ldcg(reinterpret_cast<const float4*>(p));
    const T* s = reinterpret_cast<const T*>(&r);
#pragma unroll
    for (int i = 0; i < V; ++i) d[i] = s[i];
  } else if constexpr (CG) {
#pragma unroll
    for (int i = 0; i < V; ++i) d[i] = __ldcg(p + i);
  } else {
    ldv<T, V>(d, p);
  }
}
template <bool CG, class T>
__device__ __forceinline__ T ld1(const T* p) {
  if constexpr (CG) return __ldcg(p);
  else return __ldg(p);
}

// One work item = one (band, strip) of one problem (active-list entry `entry`).
template <class T, int V, bool CG = false>
__device__ __forceinline__ void fgp2d_item(const FgpArgs<T, V>& a, int item, int entry) {
  using A = Ar<T>;
  const int lane = threadIdx.x & 31;
  const int band = item % a.nbands;
  const int strip = item / a.nbands;
  const int p = a.active ? a.active[entry] : entry;
  const int H = a.H, W = a.W;
  const int64_t HW = (int64_t)H * W;

  const T* __restrict__ xp = a.x + (int64_t)p * a.xps;
  T* qbase = a.q + (int64_t)p * a.qps;
  const T* qk = qbase + (int64_t)(a.it % 3) * 2 * HW;
  const T* qm = qbase + (int64_t)((a.it + 2) % 3) * 2 * HW;
  T* qo = qbase + (int64_t)((a.it + 1) % 3) * 2 * HW;
  const T w = (T)(a.wts ? a.wts[entry] : a.w_all);
  const bool rp = a.it == 0 && (a.rep ? a.rep[entry] != 0 : a.rep_all != 0);
  const bool mom = a.beta != T(0);
  const T beta = a.beta, step = a.step;

  const int c0 = band * 32 * V;
  const int cl = c0 + lane * V;
  const bool lin = cl < W;  // V divides W, so the whole vector is in range
  // band-edge halo column: lane 0 -> c0-1 (needs y_x), lane 31 -> c0+32V (needs y, x)
  const int hc = lane == 0 ? c0 - 1 : c0 + 32 * V;
  const bool hval = (lane == 0 && c0 > 0) || (lane == 31 && hc < W);

  const int r0 = strip * a.rs;
  const int r1 = min(H, r0 + a.rs);

  T yyu[V], yy[V], yx[V], u[V];
  T hyyu = T(0), hyy = T(0), hyx = T(0), hu = T(0);

#pragma unroll
  for (int v = 0; v < V; ++v) yyu[v] = yy[v] = yx[v] = u[v] = T(0);

  // Raw loads of one row (issued early, consumed one row later) and their
  // completion into y = q_k + beta (q_k - q_{k-1}) (re-projection at it == 0)
  // and u := x (prim_row adds the divergence).
  struct Raw {
    T ky[V], kx[V], my[V], mx[V], xv[V];
    T hky, hkx, hmy, hmx, hx;
  };
  auto issue_row = [&](int r, Raw& R) {
    const int64_t ro = (int64_t)r * W;
    if (lin) {
      ldq<CG, T, V>(R.ky, qk + ro + cl);
      ldq<CG, T, V>(R.kx, qk + HW + ro + cl);
      if (mom) {
        ldq<CG, T, V>(R.my, qm + ro + cl);
        ldq<CG, T, V>(R.mx, qm + HW + ro + cl);
      }
      ldq<CG, T, V>(R.xv, xp + ro + cl);
    }
    if (hval) {
      R.hky = ld1<CG>(qk + ro + hc);
      R.hkx = ld1<CG>(qk + HW + ro + hc);
      if (mom) {
        R.hmy = ld1<CG>(qm + ro + hc);
        R.hmx = ld1<CG>(qm + HW + ro + hc);
      }
      R.hx = ld1<CG>(xp + ro + hc);
    }
  };
  auto finish_row = [&](const Raw& R, T(&ty)[V], T(&tx)[V], T(&tu)[V], T& ty1, T& tx1, T& tu1) {
    auto y_of = [&](T k0, T k1, T m0, T m1, T& o0, T& o1) {
      if (rp) {
        const T sc = A::ball_scale(k0, k1, w);
        k0 = A::mul(k0, sc);
        k1 = A::mul(k1, sc);
      }
      if (mom) {
        k0 = A::add(k0, A::mul(beta, A::sub(k0, m0)));
        k1 = A::add(k1, A::mul(beta, A::sub(k1, m1)));
      }
      o0 = k0;
      o1 = k1;
    };
    if (lin) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        y_of(R.ky[v], R.kx[v], mom ? R.my[v] : T(0), mom ? R.mx[v] : T(0), ty[v], tx[v]);
        tu[v] = R.xv[v];
      }
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) ty[v] = tx[v] = tu[v] = T(0);
    }
    if (hval) {
      y_of(R.hky, R.hkx, mom ? R.hmy : T(0), mom ? R.hmx : T(0), ty1, tx1);
      tu1 = R.hx;
    }
  };

  // u(i) = clamp(x(i) + div y) for the lane's V columns and (lane 31) the halo
  auto prim_row = [&](int r, const T(&ty)[V], const T(&tyu)[V], const T(&tx)[V], T(&tu)[V],
                      T ty1, T tyu1, T tx1, T& tu1) {
    T left = __shfl_up_sync(0xffffffffu, tx[V - 1], 1);
    if (lane == 0) left = tx1;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const T xl = v > 0 ? tx[v - 1] : left;
      tu[v] = clampu(A::add(tu[v], div_at<T>(r, cl + v, H, W, ty[v], tyu[v], tx[v], xl)), a.nonneg);
    }
    if (lane == 31) tu1 = clampu(A::add(tu1, div_at<T>(r, hc, H, W, ty1, tyu1, tx1, tx[V - 1])), a.nonneg);
  };

  // prologue: issue rows r0-1, r0, r0+1 together (one memory round trip),
  // then y_y(r0-1), y(r0), u(r0)
  Raw Rup, Rc, Rn;
  if (r0 > 0) issue_row(r0 - 1, Rup);
  issue_row(r0, Rc);
  if (r0 + 1 < H) issue_row(r0 + 1, Rn);
  if (r0 > 0) {
    T tx[V], tu[V], tx1 = T(0), tu1 = T(0);
    finish_row(Rup, yyu, tx, tu, hyyu, tx1, tu1);
  }
  {
    T hx1 = T(0);
    finish_row(Rc, yy, yx, u, hyy, hyx, hx1);
    hu = hx1;
    prim_row(r0, yy, yyu, yx, u, hyy, hyyu, hyx, hu);
  }

  for (int i = r0; i < r1; ++i) {
    const bool nxt = i + 1 < H;
    T nyy[V], nyx[V], nu[V];
    T nhyy = T(0), nhyx = T(0), nhu = T(0);
#pragma unroll
    for (int v = 0; v < V; ++v) nyy[v] = nyx[v] = nu[v] = T(0);
    if (nxt) {
      finish_row(Rn, nyy, nyx, nu, nhyy, nhyx, nhu);
      // row i+2 is needed only if row i+1 is still in this strip
      if (i + 2 < H && i + 1 < r1) issue_row(i + 2, Rn);
      prim_row(i + 1, nyy, yy, nyx, nu, nhyy, hyy, nhyx, nhu);
    }
    T right = __shfl_down_sync(0xffffffffu, u[0], 1);
    if (lane == 31) right = hu;
    T oy[V], ox[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int c = cl + v;
      const T ur = v < V - 1 ? u[v + 1] : right;
      const T gy = nxt ? A::sub(nu[v], u[v]) : T(0);
      const T gx = c < W - 1 ? A::sub(ur, u[v]) : T(0);
      const T ay = A::add(yy[v], A::mul(step, gy));
      const T ax = A::add(yx[v], A::mul(step, gx));
      const T s = A::ball_scale(ay, ax, w);
      oy[v] = A::mul(ay, s);
      ox[v] = A::mul(ax, s);
    }
    if (lin) {
      const int64_t o = (int64_t)i * W + cl;
      stv<T, V>(qo + o, oy);
      stv<T, V>(qo + HW + o, ox);
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      yyu[v] = yy[v];
      yy[v] = nyy[v];
      yx[v] = nyx[v];
      u[v] = nu[v];
    }
    hyyu = hyy;
    hyy = nhyy;
    hyx = nhyx;
    hu = nhu;
  }
}

template <class T, int V>
__global__ void __launch_bounds__(128) fgp2d_iter_kernel(FgpArgs<T, V> a) {
  pdl_enter();
  const int item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (item >= a.nitems) return;  // whole warp exits together
  fgp2d_item(a, item, blockIdx.y);
}

// u = clamp(x + div q_n) and q_n -> slot 0 (tv.py:86-89)
template <class T>
__global__ void fgp2d_finalize_kernel(const T* __restrict__ x, int64_t xps, T* q, int64_t qps,
                                      const int32_t* __restrict__ active, int H, int W, int n_inner,
                                      int nonneg, T* __restrict__ u, int64_t ups) {
  using A = Ar<T>;
  pdl_enter();
  const int p = active ? active[blockIdx.y] : (int)blockIdx.y;
  const int64_t HW = (int64_t)H * W;
  const int slot = n_inner % 3;
  T* qb = q + (int64_t)p * qps;
  const T* qn = qb + (int64_t)slot * 2 * HW;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < HW;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx / W), c = (int)(idx % W);
    const T yy = qn[idx], yx = qn[HW + idx];
    const T yyu = i > 0 ? qn[idx - W] : T(0);
    const T yxl = c > 0 ? qn[HW + idx - 1] : T(0);
    const T d = div_at<T>(i, c, H, W, yy, yyu, yx, yxl);
    u[(int64_t)p * ups + idx] = clampu(A::add(x[(int64_t)p * xps + idx], d), nonneg);
    if (slot != 0) {
      qb[idx] = yy;
      qb[HW + idx] = yx;
    }
  }
}

// ---- temporally blocked FGP (TBI inner iterations per launch) ------------
//
// A single 512 x 512 problem (configs 2 and 3i) runs one streaming launch per
// inner iteration at ~6 us each: latency-bound, the grid is small.  Here a
// 512-thread CTA loads a 64 x 64 window (a 44 x 44 output tile plus a
// 10-pixel halo) of z, q_k and q_{k-1} into REGISTERS -- thread (warp row wr,
// warp column wc, lane) owns column 32 wc + lane, rows 8 wr .. 8 wr + 7, as
// in the cluster kernel -- and runs TBI = 10 inner iterations on it: the
// stencil has radius 1, so the exact region shrinks by one pixel per
// iteration and the 44 x 44 interior is exact after 10 (12 x 12 = 144 CTAs
// at 512^2: one wave on 148 SMs).  Column neighbours come from shuffles (plus
// shared memory between the two warp columns), row neighbours from registers
// (plus shared memory between warp rows); two CTA barriers per iteration;
// global image boundaries by per-pixel rules on the global index.  10x fewer
// launches and ~(20 + 16) / 10 B of L2/HBM traffic per pixel-iteration, for
// (64/44)^2 = 2.1x redundant halo arithmetic.  The per-pixel formulas are
// fgp2d_item's; the compiled instruction sequences differ (FMA contraction
// of the momentum / projection), so the results agree with the streaming
// kernel to ~1e-6 absolute (tests/test_gpu_tb.py), both well inside the
// oracle tolerance.
constexpr int TBI = 10;                   // inner iterations per launch (halo width)
constexpr int TBS = 64;                   // window side
constexpr int TBT = TBS - 2 * TBI;        // output tile side (44: 12 x 12 = 144 CTAs at 512^2, one wave)
constexpr int TBR = 8;                    // rows per thread
constexpr int TB_THREADS = 512;           // 2 warp columns x 8 warp rows

struct TbArgs {
  const float* x;       // prox input z, problem p at x + p * xps
  int64_t xps;
  const float* qk_in;   // q_k (2 channels) of problem p at + p * in_ps; channel stride HW
  const float* qm_in;   // q_{k-1}, ignored when beta[0] == 0
  int64_t in_ps;
  float* qk_out;        // q_{k+nit} (+ p * out_ps)
  float* qm_out;        // q_{k+nit-1}, nullptr: not needed (last launch)
  int64_t out_ps;
  const int32_t* active;
  const double* wts;
  float w_all;
  const uint8_t* rep;   // re-project q_k after loading (first launch only)
  int rep_all;
  int H, W, nit;
  float beta[TBI];      // beta of each iteration of this launch
  float step;
  int nonneg;
  int tiles_x;
  int in_by_entry, out_by_entry;  // q_in / q_out indexed by active entry (scratch) or problem
};

__global__ void __launch_bounds__(TB_THREADS, 1) fgp2d_tb_kernel(TbArgs a) {
  using A = Ar<float>;
  __shared__ float s_yy[8][TBS];        // last-row y_y of each warp row
  __shared__ float s_u[8][TBS];         // first-row u of each warp row
  __shared__ float s_yx[8][TBR];        // lane-31 column y_x of warp column 0, per warp row
  __shared__ float s_ul[8][TBR];        // lane-0 column u of warp column 1, per warp row
  pdl_enter();  // launched as a chain: the next launch's CTAs wait here, not in the launch queue
  const int entry = blockIdx.y;
  const int p = a.active ? a.active[entry] : entry;
  const int H = a.H, W = a.W;
  const int64_t HW = (int64_t)H * W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wc = warp & 1, wr = warp >> 1;
  const int c = wc * 32 + lane, r0 = wr * TBR;
  const int ty = blockIdx.x / a.tiles_x, tx = blockIdx.x % a.tiles_x;
  const int gj = tx * TBT - TBI + c;              // global column of this thread
  const int gi0 = ty * TBT - TBI + r0;            // global row of this thread's row 0
  const bool cin = gj >= 0 && gj < W;
  const float w = a.wts ? (float)a.wts[entry] : a.w_all;
  const bool rp = a.rep ? a.rep[entry] != 0 : a.rep_all != 0;
  const bool mom0 = a.beta[0] != 0.f;
  const int pin = a.in_by_entry ? entry : p, pout = a.out_by_entry ? entry : p;
  const float* xp = a.x + (int64_t)p * a.xps;
  const float* kp = a.qk_in + (int64_t)pin * a.in_ps;
  const float* mp = a.qm_in + (int64_t)pin * a.in_ps;
  float z[TBR], ky[TBR], kx[TBR], my[TBR], mx[TBR];
  bool in[TBR];
#pragma unroll
  for (int t = 0; t < TBR; ++t) {
    const int gi = gi0 + t;
    in[t] = cin && gi >= 0 && gi < H;
    z[t] = ky[t] = kx[t] = my[t] = mx[t] = 0.f;
    if (in[t]) {
      const int64_t o = (int64_t)gi * W + gj;
      z[t] = __ldcg(xp + o);
      ky[t] = __ldcg(kp + o);
      kx[t] = __ldcg(kp + HW + o);
      if (rp) {
        const float sc = A::ball_scale(ky[t], kx[t], w);
        ky[t] = A::mul(ky[t], sc);
        kx[t] = A::mul(kx[t], sc);
      }
      if (mom0) {
        my[t] = __ldcg(mp + o);
        mx[t] = __ldcg(mp + HW + o);
      }
    }
  }
  const bool col_first = gj == 0, col_last = gj == W - 1;
  // One inner iteration; reads (QK, QM), writes the new iterate into QM.
  auto iter = [&](float(&QKy)[TBR], float(&QKx)[TBR], float(&QMy)[TBR], float(&QMx)[TBR],
                  float beta) {
    float yy[TBR], yx[TBR], u[TBR];
#pragma unroll
    for (int t = 0; t < TBR; ++t) {
      yy[t] = QKy[t];
      yx[t] = QKx[t];
      if (beta != 0.f) {
        yy[t] = A::add(yy[t], A::mul(beta, A::sub(yy[t], QMy[t])));
        yx[t] = A::add(yx[t], A::mul(beta, A::sub(yx[t], QMx[t])));
      }
    }
    s_yy[wr][c] = yy[TBR - 1];
    if (wc == 0 && lane == 31)
#pragma unroll
      for (int t = 0; t < TBR; ++t) s_yx[wr][t] = yx[t];
    __syncthreads();
    const float yy_top = wr > 0 ? s_yy[wr - 1][c] : 0.f;  // (window edge: inexact margin)
#pragma unroll
    for (int t = 0; t < TBR; ++t) {
      float left = __shfl_up_sync(0xffffffffu, yx[t], 1);
      if (lane == 0) left = wc == 1 ? s_yx[wr][t] : 0.f;
      const int gi = gi0 + t;
      // div_at's order: ((0 + [i<H-1] yy) - [i>0] yy_up) + [j<W-1] yx - [j>0] yx_left
      float d = 0.f;
      if (gi < H - 1) d = A::add(d, yy[t]);
      if (gi > 0) d = A::sub(d, t > 0 ? yy[t - 1] : yy_top);
      if (!col_last) d = A::add(d, yx[t]);
      if (!col_first) d = A::sub(d, left);
      u[t] = in[t] ? clampu(A::add(z[t], d), a.nonneg) : 0.f;
    }
    s_u[wr][c] = u[0];
    if (wc == 1 && lane == 0)
#pragma unroll
      for (int t = 0; t < TBR; ++t) s_ul[wr][t] = u[t];
    __syncthreads();
    const float u_bot = wr < 7 ? s_u[wr + 1][c] : 0.f;
#pragma unroll
    for (int t = 0; t < TBR; ++t) {
      float right = __shfl_down_sync(0xffffffffu, u[t], 1);
      if (lane == 31) right = wc == 0 ? s_ul[wr][t] : 0.f;
      const int gi = gi0 + t;
      const float ub = t < TBR - 1 ? u[t + 1] : u_bot;
      const float gy = gi < H - 1 ? A::sub(ub, u[t]) : 0.f;
      const float gx = !col_last ? A::sub(right, u[t]) : 0.f;
      const float ay = A::add(yy[t], A::mul(a.step, gy));
      const float ax = A::add(yx[t], A::mul(a.step, gx));
      const float sc = A::ball_scale(ay, ax, w);
      QMy[t] = in[t] ? A::mul(ay, sc) : 0.f;
      QMx[t] = in[t] ? A::mul(ax, sc) : 0.f;
    }
    __syncthreads();  // s_yy / s_yx / s_u / s_ul reused by the next iteration
  };
  int t = 0;
  for (; t + 1 < a.nit; t += 2) {
    iter(ky, kx, my, mx, a.beta[t]);      // new iterate in m*
    iter(my, mx, ky, kx, a.beta[t + 1]);  // new iterate in k*
  }
  const bool odd = t < a.nit;
  if (odd) iter(ky, kx, my, mx, a.beta[t]);
  // newest iterate: m* if nit is odd, else k*; the previous one in the other
  float* ko = a.qk_out + (int64_t)pout * a.out_ps;
  float* mo = a.qm_out ? a.qm_out + (int64_t)pout * a.out_ps : nullptr;
  const bool cout = c >= TBI && c < TBS - TBI && cin;
#pragma unroll
  for (int tt = 0; tt < TBR; ++tt) {
    const int r = r0 + tt;
    if (!cout || r < TBI || r >= TBS - TBI || !in[tt]) continue;
    const int64_t o = (int64_t)(gi0 + tt) * W + gj;
    ko[o] = odd ? my[tt] : ky[tt];
    ko[HW + o] = odd ? mx[tt] : kx[tt];
    if (mo) {
      mo[o] = odd ? ky[tt] : my[tt];
      mo[HW + o] = odd ? kx[tt] : mx[tt];
    }
  }
}

// ---- SM-resident ProxSkip worker (config 4, the SMs the clusters leave) ----
//
// The clusters of the run kernels do not tile the whole device (8-CTA
// clusters: 15 x 8 = 120 of 148 SMs; 16-CTA clusters: 7 x 16 = 112 -- a
// cluster needs its SMs in one GPC); the remaining SMs run this kernel concurrently,
// one 512-thread CTA per SM, each working through its own list of whole
// problems: for every coin-fired iteration of a problem the CTA runs the skip
// chain + prox input, the n_inner FGP iterations (the streaming item above
// with L2-coherent loads and a CTA barrier between iterations: the problem's
// ~2 MB working set stays L2-resident), finalize + control variate, then the
// trailing skips.  Same arithmetic as the streaming driver (proxskip_pre /
// fgp2d_iter / fgp2d_finalize / proxskip_post).  Clusters and workers claim
// problems from one device work queue (common.cuh); the kernels are
// bit-identical, so which one runs a problem never changes a result.
struct SmRunArgs {
  float* x;
  const float* b;
  float* h;
  float* q;
  int64_t qps;
  float* z;                // prox-input scratch, (N, H, W)
  WorkQueue wq;            // problems claimed dynamically (common.cuh)
  const int32_t* ev_off;
  const int32_t* ev_k;
  const uint8_t* rep;
  int K;
  int n_inner;
  int accelerated;
  int nonneg;
  float weight, gamma, hc, pg, step;
  int32_t* bad;
  const float* betas;
  ChunkSync cs;
};

constexpr int SM_THREADS = 512;
constexpr int SM_SIDE = 256;

__device__ __forceinline__ float sm_skip(float xo, float bo, float ho, float g) {
  using A = Ar<float>;
  return A::add(A::sub(xo, A::mul(g, A::sub(xo, bo))), A::mul(g, ho));  // skip.py:68
}

// rsqrt without the denormal rescaling (as the cluster kernel)
__device__ __forceinline__ float sm_rsq(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// One FGP inner iteration of a 256 x 256 problem by one 512-thread CTA: warp w
// marches rows 16w .. 16w+15, lane l owns columns 4l .. 4l+3 (half A) and
// 128+4l .. 128+4l+3 (half B) -- one fully coalesced float4 per half, array
// and row -- so a row's column neighbours need two shuffles each way and the
// previous row stays in registers.  Zero padding (q_y = 0 on the last row,
// q_x = 0 on the last column: the FGP keeps both, see the cluster kernel)
// replaces the boundary tests; the arithmetic is the cluster kernel's
// operation for operation (packed f32x2, same FMA forms).
template <bool mom, bool rp>
__device__ __forceinline__ void sm_fgp_iter(const float* __restrict__ z, const float* qk,
                                            const float* qm, float* qo, float beta, float step,
                                            float w, int nonneg) {
  constexpr int W = SM_SIDE, H = SM_SIDE;
  constexpr int HW = H * W;
  constexpr int RS = H / (SM_THREADS / 32);  // rows per warp strip
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = warp * RS, r1 = r0 + RS;
  const int c0 = lane * 4;  // half A; half B at c0 + W/2
  const float2 b2 = make_float2(beta, beta), m1 = make_float2(-1.f, -1.f);
  const float wr = w * kBallShrink;  // (common.cuh)
  const float2 st2 = make_float2(step, step), w2 = make_float2(wr, wr);
  struct Raw {
    float4 ky[2], kx[2], my[2], mx[2], zz[2];
  };
  auto ld4 = [](const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); };
  auto load = [&](int r, Raw& R, bool with_z) {
    const int o = r * W + c0;
    constexpr int B = W / 2;
    R.ky[0] = ld4(qk + o);
    R.ky[1] = ld4(qk + o + B);
    R.kx[0] = ld4(qk + HW + o);
    R.kx[1] = ld4(qk + HW + o + B);
    if constexpr (mom) {
      R.my[0] = ld4(qm + o);
      R.my[1] = ld4(qm + o + B);
      R.mx[0] = ld4(qm + HW + o);
      R.mx[1] = ld4(qm + HW + o + B);
    }
    if (with_z) {
      R.zz[0] = ld4(z + o);
      R.zz[1] = ld4(z + o + B);
    }
  };
  // float4 pair halves as float2 (columns (0,1), (2,3) of each float4)
  auto lo = [](const float4& v) { return make_float2(v.x, v.y); };
  auto hi = [](const float4& v) { return make_float2(v.z, v.w); };
  // y = q_k + beta (q_k - q_{k-1}) (re-projected q_k at the first iteration)
  auto y_of = [&](const Raw& R, float2 (&yy)[4], float2 (&yx)[4]) {
#pragma unroll
    for (int P = 0; P < 4; ++P) {
      float2 ky = (P & 1) ? hi(R.ky[P >> 1]) : lo(R.ky[P >> 1]);
      float2 kx = (P & 1) ? hi(R.kx[P >> 1]) : lo(R.kx[P >> 1]);
      if constexpr (rp) {
        const float sx = fminf(1.f, wr * sm_rsq(fmaf(ky.x, ky.x, kx.x * kx.x)));
        const float sy = fminf(1.f, wr * sm_rsq(fmaf(ky.y, ky.y, kx.y * kx.y)));
        ky = make_float2(ky.x * sx, ky.y * sy);
        kx = make_float2(kx.x * sx, kx.y * sy);
      }
      if constexpr (mom) {
        const float2 my = (P & 1) ? hi(R.my[P >> 1]) : lo(R.my[P >> 1]);
        const float2 mx = (P & 1) ? hi(R.mx[P >> 1]) : lo(R.mx[P >> 1]);
        yy[P] = __ffma2_rn(b2, __ffma2_rn(my, m1, ky), ky);
        yx[P] = __ffma2_rn(b2, __ffma2_rn(mx, m1, kx), kx);
      } else {
        yy[P] = ky;
        yx[P] = kx;
      }
    }
  };
  // u = clamp(z + ((yy - yy_up) + yx) - yx_left)
  auto u_of = [&](const float2 (&yy)[4], const float2 (&yx)[4], const float2 (&yyu)[4],
                  const Raw& R, float2 (&u)[4]) {
    // column left of half A: lane l-1's half A (0 left of column 0); of half
    // B: lane l-1's half B, lane 0 takes lane 31's half A (column 127)
    float left_a = __shfl_up_sync(0xffffffffu, yx[1].y, 1);
    if (lane == 0) left_a = 0.f;
    const float left_b = __shfl_sync(0xffffffffu, lane == 31 ? yx[1].y : yx[3].y, (lane + 31) & 31);
#pragma unroll
    for (int P = 0; P < 4; ++P) {
      const float2 l2 = make_float2(P == 0 ? left_a : P == 2 ? left_b : yx[P - 1].y, yx[P].x);
      const float2 d1 = __fadd2_rn(__ffma2_rn(yyu[P], m1, yy[P]), yx[P]);
      const float2 d2 = __ffma2_rn(l2, m1, d1);
      const float2 zz = (P & 1) ? hi(R.zz[P >> 1]) : lo(R.zz[P >> 1]);
      const float2 v = __fadd2_rn(zz, d2);
      u[P] = nonneg ? make_float2(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f)) : v;
    }
  };
  // row i: y(i+1), u(i+1) from the prefetched row, then q_{k+1}(i); the two
  // register sets alternate between "this row" and "next row" (no copies)
  Raw Rn;
  auto row = [&](int i, const float2 (&yy)[4], const float2 (&yx)[4], const float2 (&u)[4],
                 float2 (&nyy)[4], float2 (&nyx)[4], float2 (&nu)[4]) {
    if (i + 1 < H) {
      y_of(Rn, nyy, nyx);
      u_of(nyy, nyx, yy, Rn, nu);
      if (i + 2 < H && i + 1 < r1) load(i + 2, Rn, true);
    } else {
#pragma unroll
      for (int P = 0; P < 4; ++P) nu[P] = u[P];  // last row: gy = 0
    }
    // column right of half A: lane l+1's half A, lane 31 takes lane 0's half
    // B (column 128); of half B: lane l+1's half B, lane 31 keeps its own
    // (column W-1: gx = 0)
    const float right_a = __shfl_sync(0xffffffffu, lane == 0 ? u[2].x : u[0].x, (lane + 1) & 31);
    float right_b = __shfl_down_sync(0xffffffffu, u[2].x, 1);
    if (lane == 31) right_b = u[3].y;
    float4 oy[2], ox[2];
#pragma unroll
    for (int P = 0; P < 4; ++P) {
      const float2 rt = make_float2(u[P].y, P == 1 ? right_a : P == 3 ? right_b : u[P + 1].x);
      const float2 gy = __ffma2_rn(u[P], m1, nu[P]);
      const float2 gx = __ffma2_rn(u[P], m1, rt);
      const float2 ay = __ffma2_rn(st2, gy, yy[P]);
      const float2 ax = __ffma2_rn(st2, gx, yx[P]);
      const float2 m2 = __ffma2_rn(ay, ay, __fmul2_rn(ax, ax));
      float2 sc = __fmul2_rn(w2, make_float2(sm_rsq(m2.x), sm_rsq(m2.y)));
      sc.x = fminf(1.f, sc.x);
      sc.y = fminf(1.f, sc.y);
      const float2 ny = __fmul2_rn(ay, sc), nx = __fmul2_rn(ax, sc);
      float* py = (P & 1) ? &oy[P >> 1].z : &oy[P >> 1].x;
      float* px = (P & 1) ? &ox[P >> 1].z : &ox[P >> 1].x;
      py[0] = ny.x;
      py[1] = ny.y;
      px[0] = nx.x;
      px[1] = nx.y;
    }
    const int o = i * W + c0;
    __stcg(reinterpret_cast<float4*>(qo + o), oy[0]);
    __stcg(reinterpret_cast<float4*>(qo + o + W / 2), oy[1]);
    __stcg(reinterpret_cast<float4*>(qo + HW + o), ox[0]);
    __stcg(reinterpret_cast<float4*>(qo + HW + o + W / 2), ox[1]);
  };
  float2 ya[4], xa[4], ua[4], yb[4], xb[4], ub[4];
  {
    float2 yyu[4];
#pragma unroll
    for (int P = 0; P < 4; ++P) yyu[P] = make_float2(0.f, 0.f);
    if (r0 > 0) {
      Raw Ru;
      load(r0 - 1, Ru, false);
      float2 tx[4];
      y_of(Ru, yyu, tx);
    }
    Raw Rc;
    load(r0, Rc, true);
    load(r0 + 1, Rn, true);  // r0 + 1 < H for every strip (RS >= 2)
    y_of(Rc, ya, xa);
    u_of(ya, xa, yyu, Rc, ua);
  }
  static_assert(RS % 2 == 0, "rows are processed in pairs");
  for (int i = r0; i < r1; i += 2) {
    row(i, ya, xa, ua, yb, xb, ub);
    row(i + 1, yb, xb, ub, ya, xa, ua);
  }
}

__global__ void __launch_bounds__(SM_THREADS, 1) fgp_sm_run_kernel(SmRunArgs a) {
  using A = Ar<float>;
  constexpr int H = SM_SIDE, W = SM_SIDE;
  constexpr int64_t HW = (int64_t)H * W;
  constexpr int NV = (int)(HW / 4);
  const int tid = threadIdx.x;
  const float g = a.gamma;
  __shared__ int s_pos;
  for (;;) {
    if (tid == 0) s_pos = wq_claim_worker(a.wq);
    __syncthreads();
    const int pos = s_pos;
    if (pos < 0) break;
    const int p = a.wq.order[pos];
    float* xp = a.x + (int64_t)p * HW;
    const float* bp = a.b + (int64_t)p * HW;
    float* hp = a.h + (int64_t)p * HW;
    float* zp = a.z + (int64_t)p * HW;
    float* q0 = a.q + (int64_t)p * a.qps;
    const int e0 = a.ev_off[p], e1 = a.ev_off[p + 1];
    if (a.cs.ready) {  // this problem's input chunk has arrived
      if (tid == 0) chunk_wait(a.cs, p);
      __syncthreads();
    }
    if (a.cs.ready) {  // a streamed run starts cold: x = h = 0, q_warm = 0 (not initialised)
      const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int v = tid; v < NV; v += SM_THREADS) {
        __stcg(reinterpret_cast<float4*>(xp) + v, zero);
        __stcg(reinterpret_cast<float4*>(hp) + v, zero);
        __stcg(reinterpret_cast<float4*>(q0) + v, zero);
        __stcg(reinterpret_cast<float4*>(q0 + HW) + v, zero);
      }
      __syncthreads();
    }
    const uint64_t t_claim = gtimer_ns();
    int kbad = 0x7fffffff;
    int kprev = -1;
    for (int e = e0; e < e1; ++e) {
      const int kk = a.ev_k[e];
      const int m = kk - kprev - 1, kf = kprev + 1;
      // skips kprev+1 .. kk-1 (x materialised), prox input z (skip.py:66-70)
      for (int v = tid; v < NV; v += SM_THREADS) {
        float4 xv = __ldcg(reinterpret_cast<const float4*>(xp) + v);
        const float4 bv = __ldcg(reinterpret_cast<const float4*>(bp) + v);
        const float4 hv = __ldcg(reinterpret_cast<const float4*>(hp) + v);
        float* xs = &xv.x;
        const float* bs = &bv.x;
        const float* hs = &hv.x;
        float4 zv;
        float* zs = &zv.x;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float xo = skip_chain_px(xs[c], bs[c], hs[c], g, m, kf, &kbad);
          xs[c] = xo;
          zs[c] = A::add(A::sub(xo, A::mul(g, A::sub(xo, bs[c]))), A::mul(a.hc, hs[c]));
        }
        if (m > 0) __stcg(reinterpret_cast<float4*>(xp) + v, xv);
        __stcg(reinterpret_cast<float4*>(zp) + v, zv);
      }
      __syncthreads();
      // FGP on z with the warm start in slot 0 (re-projected at the run's
      // first call if the weight changed, tv.py:68-69)
      const bool rp0 = e == e0 && a.rep[p];
      for (int it = 0; it < a.n_inner; ++it) {
        const float beta = (a.accelerated && it > 0) ? a.betas[it - 1] : 0.f;
        const float* qk = q0 + (int64_t)(it % 3) * 2 * HW;
        const float* qm = q0 + (int64_t)((it + 2) % 3) * 2 * HW;
        float* qo = q0 + (int64_t)((it + 1) % 3) * 2 * HW;
        if (beta != 0.f)
          sm_fgp_iter<true, false>(zp, qk, qm, qo, beta, a.step, a.weight, a.nonneg);
        else if (it == 0 && rp0)
          sm_fgp_iter<false, true>(zp, qk, qm, qo, beta, a.step, a.weight, a.nonneg);
        else
          sm_fgp_iter<false, false>(zp, qk, qm, qo, beta, a.step, a.weight, a.nonneg);
        __syncthreads();
      }
      // finalize u = clamp(z + div q_n) (tv.py:89), ProxSkip post (skip.py:68-75),
      // q_n -> warm-start slot 0
      const int slot = a.n_inner % 3;
      const float* qn = q0 + (int64_t)slot * 2 * HW;
      bool ok = true;
      for (int v = tid; v < NV; v += SM_THREADS) {  // 4 columns of one row
        const int idx = 4 * v, i = idx / W, c = idx % W;
        const float4 yy4 = __ldcg(reinterpret_cast<const float4*>(qn + idx));
        const float4 yx4 = __ldcg(reinterpret_cast<const float4*>(qn + HW + idx));
        const float4 yu4 = i > 0 ? __ldcg(reinterpret_cast<const float4*>(qn + idx - W))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
        const float yxl = c > 0 ? __ldcg(qn + HW + idx - 1) : 0.f;
        const float4 z4 = __ldcg(reinterpret_cast<const float4*>(zp) + v);
        const float4 x4 = __ldcg(reinterpret_cast<const float4*>(xp) + v);
        const float4 b4 = __ldcg(reinterpret_cast<const float4*>(bp) + v);
        const float4 h4 = __ldcg(reinterpret_cast<const float4*>(hp) + v);
        const float yys[4] = {yy4.x, yy4.y, yy4.z, yy4.w}, yxs[4] = {yx4.x, yx4.y, yx4.z, yx4.w};
        const float yus[4] = {yu4.x, yu4.y, yu4.z, yu4.w}, zs[4] = {z4.x, z4.y, z4.z, z4.w};
        const float xs[4] = {x4.x, x4.y, x4.z, x4.w}, bs[4] = {b4.x, b4.y, b4.z, b4.w};
        const float hs[4] = {h4.x, h4.y, h4.z, h4.w};
        float un[4], hn[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float d = div_at<float>(i, c + k, H, W, yys[k], yus[k], yxs[k], k > 0 ? yxs[k - 1] : yxl);
          un[k] = clampu(A::add(zs[k], d), a.nonneg);
          const float xhat = sm_skip(xs[k], bs[k], hs[k], g);
          hn[k] = A::add(hs[k], A::mul(a.pg, A::sub(un[k], xhat)));
          ok &= finite(un[k]);
        }
        __stcg(reinterpret_cast<float4*>(hp) + v, make_float4(hn[0], hn[1], hn[2], hn[3]));
        __stcg(reinterpret_cast<float4*>(xp) + v, make_float4(un[0], un[1], un[2], un[3]));
        if (slot != 0) {
          __stcg(reinterpret_cast<float4*>(q0 + idx), yy4);
          __stcg(reinterpret_cast<float4*>(q0 + HW + idx), yx4);
        }
      }
      if (!ok) kbad = min(kbad, kk);
      kprev = kk;
      __syncthreads();
    }
    // trailing skips kprev+1 .. K-1
    const int m = a.K - 1 - kprev;
    if (m > 0) {
      for (int v = tid; v < NV; v += SM_THREADS) {
        float4 xv = __ldcg(reinterpret_cast<const float4*>(xp) + v);
        const float4 bv = __ldcg(reinterpret_cast<const float4*>(bp) + v);
        const float4 hv = __ldcg(reinterpret_cast<const float4*>(hp) + v);
        float* xs = &xv.x;
        const float* bs = &bv.x;
        const float* hs = &hv.x;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          xs[c] = skip_chain_px(xs[c], bs[c], hs[c], g, m, kprev + 1, &kbad);
        }
        __stcg(reinterpret_cast<float4*>(xp) + v, xv);
      }
    }
    if (kbad != 0x7fffffff && a.bad) atomicMin(a.bad + p, kbad);
    chunk_done(a.cs, p, 16, tid == 0);
    if (tid == 0) wq_record(a.wq, 1, pos, t_claim);
    __syncthreads();
  }
  // launched as a programmatic dependent of the cluster run: finish only after
  // it (the stream's later work is then ordered after both kernels)
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

template <class T, int V>
int launch_iter(const void* x, int64_t xps, void* q, int64_t qps, const int32_t* active, int n_active,
                double weight, const double* wts, int rep_all, const uint8_t* rep, int H, int W,
                int it, double beta, double step, int nonneg, cudaStream_t st) {
  FgpArgs<T, V> a;
  a.x = static_cast<const T*>(x);
  a.xps = xps;
  a.q = static_cast<T*>(q);
  a.qps = qps;
  a.active = active;
  a.wts = wts;
  a.w_all = weight;
  a.rep = rep;
  a.rep_all = rep_all;
  a.H = H;
  a.W = W;
  a.it = it;
  a.beta = (T)beta;
  a.step = (T)step;
  a.nonneg = nonneg;
  a.nbands = (W + 32 * V - 1) / (32 * V);
  // Strip height: long strips amortise the two re-read halo rows; short ones
  // expose enough warps when the batch is small (single 256^2 / 512^2 solves).
  const int64_t warps_per_row = (int64_t)a.nbands * n_active;
  const int64_t target = 4LL * sm_count() * 16;  // ~16 warps per SM, 4 waves
  int rs = 32;
  while (rs > 1 && warps_per_row * ((H + rs - 1) / rs) < target) rs >>= 1;
  a.rs = rs;
  a.nitems = a.nbands * ((H + rs - 1) / rs);
  dim3 block(128);
  dim3 grid((a.nitems + 3) / 4, n_active);
  PSB_CUDA(launch_chain(fgp2d_iter_kernel<T, V>, grid, block, 0, st, a));
  return PSB_OK;
}

template <class T>
int dispatch_iter(const void* x, int64_t xps, void* q, int64_t qps, const int32_t* active,
                  int n_active, double weight, const double* wts, int rep_all, const uint8_t* rep,
                  int H, int W, int it, double beta, double step, int nonneg, cudaStream_t st) {
  constexpr int VMAX = 16 / sizeof(T);
  const bool aligned = (W % VMAX == 0) && (xps % VMAX == 0) && (qps % VMAX == 0) &&
                       (reinterpret_cast<uintptr_t>(x) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(q) % 16 == 0);
  if (aligned)
    return launch_iter<T, VMAX>(x, xps, q, qps, active, n_active, weight, wts, rep_all, rep, H, W,
                                it, beta, step, nonneg, st);
  return launch_iter<T, 1>(x, xps, q, qps, active, n_active, weight, wts, rep_all, rep, H, W, it,
                           beta, step, nonneg, st);
}

}  // namespace

int fgp2d_iter(int dtype, const void* x, int64_t xps, void* q, int64_t qps, const int32_t* active,
               int n_active, double weight, const double* wts, int rep_all, const uint8_t* rep,
               int H, int W, int it, double beta, double step, int nonneg, cudaStream_t st);

// All n_inner FGP iterations for a batch (one launch per inner iteration;
// inside a captured CUDA graph the launches are back to back).
// Temporally blocked run (fp32): ceil(n_inner / TBI) launches; the first
// reads the warm start (slot 0), intermediate (q_k, q_{k-1}) pairs ping-pong
// through a stream-ordered scratch (a launch never reads what another CTA of
// the same launch writes), the last writes q_n to slot n_inner % 3 -- where
// the finalize / post kernels expect it.
static int fgp2d_run_tb(const float* x, int64_t xps, float* q, int64_t qps, const int32_t* active,
                        int n_active, double weight, const double* wts, int rep_all,
                        const uint8_t* rep, int H, int W, int n_inner, int accelerated,
                        int nonneg, double step, const double* betas_host, cudaStream_t st) {
  const int64_t HW = (int64_t)H * W;
  const int64_t sps = 4 * HW;  // scratch per entry and buffer: (q_k, q_{k-1}) x 2 channels
  float* scratch = nullptr;
  PSB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch),
                           sizeof(float) * 2 * sps * (size_t)n_active, st));
  TbArgs a{};
  a.x = x;
  a.xps = xps;
  a.active = active;
  a.wts = wts;
  a.w_all = (float)weight;
  a.H = H;
  a.W = W;
  a.step = (float)step;
  a.nonneg = nonneg;
  a.tiles_x = (W + TBT - 1) / TBT;
  const int tiles = a.tiles_x * ((H + TBT - 1) / TBT);
  const int L = (n_inner + TBI - 1) / TBI;
  int rc = PSB_OK;
  for (int l = 0; l < L && rc == PSB_OK; ++l) {
    const int it0 = l * TBI;
    a.nit = std::min(TBI, n_inner - it0);
    for (int t = 0; t < TBI; ++t) {
      const int it = it0 + t;
      a.beta[t] = (accelerated && it > 0 && it < n_inner) ? (float)betas_host[it - 1] : 0.f;
    }
    if (l == 0) {  // warm start in slot 0 of the problem
      a.qk_in = q;
      a.qm_in = q;  // unused: beta[0] == 0
      a.in_ps = qps;
      a.in_by_entry = 0;
      a.rep = rep;
      a.rep_all = rep_all;
    } else {
      float* in = scratch + (size_t)((l - 1) % 2) * sps * n_active;
      a.qk_in = in;
      a.qm_in = in + 2 * HW;
      a.in_ps = sps;
      a.in_by_entry = 1;
      a.rep = nullptr;
      a.rep_all = 0;
    }
    if (l == L - 1) {  // q_n to the problem's slot n_inner % 3
      a.qk_out = q + (int64_t)(n_inner % 3) * 2 * HW;
      a.qm_out = nullptr;
      a.out_ps = qps;
      a.out_by_entry = 0;
    } else {
      float* out = scratch + (size_t)(l % 2) * sps * n_active;
      a.qk_out = out;
      a.qm_out = out + 2 * HW;
      a.out_ps = sps;
      a.out_by_entry = 1;
    }
    if (launch_chain(fgp2d_tb_kernel, dim3((unsigned)tiles, (unsigned)n_active), dim3(TB_THREADS),
                     0, st, a) != cudaSuccess)
      rc = fail(PSB_ERR_CUDA, "fgp2d_tb launch failed");
  }
  cudaFreeAsync(scratch, st);
  return rc;
}

int fgp2d_run(int dtype, const void* x, int64_t xps, void* q, int64_t qps, const int32_t* active,
              int n_active, double weight, const double* wts, int rep_all, const uint8_t* rep,
              int H, int W, int n_inner, int accelerated, int nonneg, double step,
              const double* betas_host, cudaStream_t st) {
  const char* no_tb = std::getenv("PSB_NO_TB");
  // (large batches stay on the streaming kernel: at ~400 x 256^2 it runs at
  // 84 % of HBM bandwidth and beats the blocked kernel's 1.78x halo work)
  if (dtype == PSB_F32 && n_inner > TBI && H >= TBT && W >= TBT && n_active >= 1 &&
      (int64_t)n_active * H * W <= (2LL << 20) && !(no_tb && no_tb[0] == '1'))
    return fgp2d_run_tb(static_cast<const float*>(x), xps, static_cast<float*>(q), qps, active,
                        n_active, weight, wts, rep_all, rep, H, W, n_inner, accelerated, nonneg,
                        step, betas_host, st);
  for (int it = 0; it < n_inner; ++it) {
    // y_it = q_it + beta_{it-1} (q_it - q_{it-1}); beta_{-1} := 0 (y_0 = q_0)
    const double b = (accelerated && it > 0) ? betas_host[it - 1] : 0.0;
    int rc = fgp2d_iter(dtype, x, xps, q, qps, active, n_active, weight, wts, rep_all, rep, H, W,
                        it, b, step, nonneg, st);
    if (rc) return rc;
  }
  return PSB_OK;
}

int fgp2d_iter(int dtype, const void* x, int64_t xps, void* q, int64_t qps, const int32_t* active,
               int n_active, double weight, const double* wts, int rep_all, const uint8_t* rep,
               int H, int W, int it, double beta, double step, int nonneg, cudaStream_t st) {
  PSB_REQUIRE(H >= 2 && W >= 2, "fgp2d: need a 2-D grid with both sides >= 2");
  PSB_REQUIRE(n_active >= 0 && n_active <= 65535, "fgp2d: n_active out of range");
  PSB_REQUIRE(qps >= 6LL * H * W, "fgp2d: q_pstride must hold three (2,H,W) slots");
  PSB_REQUIRE(wts != nullptr || weight > 0, "tv_prox: weight must be positive");
  if (n_active == 0) return PSB_OK;
  if (dtype == PSB_F32)
    return dispatch_iter<float>(x, xps, q, qps, active, n_active, weight, wts, rep_all, rep, H, W,
                                it, beta, step, nonneg, st);
  if (dtype == PSB_F64)
    return dispatch_iter<double>(x, xps, q, qps, active, n_active, weight, wts, rep_all, rep, H, W,
                                 it, beta, step, nonneg, st);
  return fail(PSB_ERR_VALUE, "fgp2d: unknown dtype");
}

int fgp2d_finalize(int dtype, const void* x, int64_t xps, void* q, int64_t qps,
                   const int32_t* active, int n_active, int H, int W, int n_inner, int nonneg,
                   void* u, int64_t ups, cudaStream_t st) {
  PSB_REQUIRE(H >= 2 && W >= 2, "fgp2d: need a 2-D grid with both sides >= 2");
  PSB_REQUIRE(n_active >= 0 && n_active <= 65535, "fgp2d: n_active out of range");
  if (n_active == 0) return PSB_OK;
  const int64_t HW = (int64_t)H * W;
  dim3 block(256);
  dim3 grid((unsigned)std::min<int64_t>((HW + 255) / 256, 1024), n_active);
  if (dtype == PSB_F32)
    PSB_CUDA(launch_chain(fgp2d_finalize_kernel<float>, grid, block, 0, st,
                          static_cast<const float*>(x), xps, static_cast<float*>(q), qps, active,
                          H, W, n_inner, nonneg, static_cast<float*>(u), ups));
  else if (dtype == PSB_F64)
    PSB_CUDA(launch_chain(fgp2d_finalize_kernel<double>, grid, block, 0, st,
                          static_cast<const double*>(x), xps, static_cast<double*>(q), qps, active,
                          H, W, n_inner, nonneg, static_cast<double*>(u), ups));
  else
    return fail(PSB_ERR_VALUE, "fgp2d: unknown dtype");
  return PSB_OK;
}

// Beck-Teboulle momentum table, t_0 = 1, in double with the reference's
// operation order (tv.py:77-80).
void fista_betas(int n, double* out) {
  double t = 1.0;
  for (int i = 0; i < n; ++i) {
    const double t1 = (1.0 + std::sqrt(1.0 + 4.0 * t * t)) / 2.0;
    out[i] = (t - 1.0) / t1;
    t = t1;
  }
}

int tv_prox2d(int dtype, const void* x, int64_t xps, void* q, int64_t qps, const int32_t* active,
              int n_active, double weight, const double* wts, int rep_all, const uint8_t* rep,
              int H, int W, int n_inner, int accelerated, int nonneg, double step, void* u,
              int64_t ups, cudaStream_t st) {
  PSB_REQUIRE(n_inner >= 1, "TvProxState: inner_iters must be >= 1");
  PSB_REQUIRE(wts != nullptr || weight > 0, "tv_prox: weight must be positive");
  std::vector<double> beta(n_inner, 0.0);
  if (accelerated) fista_betas(n_inner, beta.data());
  int rc = fgp2d_run(dtype, x, xps, q, qps, active, n_active, weight, wts, rep_all, rep, H, W,
                     n_inner, accelerated, nonneg, step, beta.data(), st);
  if (rc) return rc;
  return fgp2d_finalize(dtype, x, xps, q, qps, active, n_active, H, W, n_inner, nonneg, u, ups, st);
}

// Accelerated projected gradient on the dual ROF problem (run_aprojgd on
// build_dual_rof(b, alpha), solvers.py:148-174 with problems.py:22-71): the
// FGP iteration with x = b, weight = alpha, step = gamma, except that FISTA
// forms its extrapolation at iteration k with (t_k - 1)/t_{k+1}, one entry
// later in the Beck-Teboulle table than FGP's (t_{k-1} - 1)/t_k (tv.py:77-80).
int aprojgd_dual_rof(int dtype, const void* b, void* q, int H, int W, double alpha, double step,
                     int iters, void* u, cudaStream_t st) {
  PSB_REQUIRE(iters >= 1, "run_aprojgd: iters must be >= 1");
  PSB_REQUIRE(alpha > 0, "DualRofProblem: alpha must be positive");
  PSB_REQUIRE(step > 0, "run_fista: gamma must be positive");
  std::vector<double> beta(iters + 1, 0.0);
  fista_betas(iters + 1, beta.data());
  const int64_t HW = (int64_t)H * W;
  int rc = fgp2d_run(dtype, b, HW, q, 6 * HW, nullptr, 1, alpha, nullptr, 0, nullptr, H, W, iters,
                     1, 0, step, beta.data() + 1, st);
  if (rc) return rc;
  return fgp2d_finalize(dtype, b, HW, q, 6 * HW, nullptr, 1, H, W, iters, 0, u, HW, st);
}

// Load the kernel before the run's first launch: with lazy module loading a
// first launch loads it on the fly, and this kernel's CTAs were then measured
// to reach the SMs before the (already enqueued) clusters, taking GPC space a
// 16-CTA cluster needs (first run 2x slower).  Called before the clusters are
// launched.
int sm_prepare() {
  static bool loaded = false;
  if (!loaded) {
    cudaFuncAttributes fa;
    PSB_CUDA(cudaFuncGetAttributes(&fa, fgp_sm_run_kernel));
    loaded = true;
  }
  return PSB_OK;
}

int sm_run(void* x, const void* b, void* h, void* q, int64_t qps, void* z, const WorkQueue& wq,
           int n_workers, const int32_t* ev_off, const int32_t* ev_k, const uint8_t* rep, int K,
           int n_inner, int accelerated, int nonneg, double weight, double gamma, double hc,
           double pg, double step, const float* betas, int32_t* bad, const ChunkSync& cs,
           bool after_clusters, cudaStream_t st) {
  if (n_workers <= 0) return PSB_OK;
  SmRunArgs a{(float*)x, (const float*)b, (float*)h, (float*)q, qps, (float*)z, wq, ev_off, ev_k,
              rep, K, n_inner, accelerated, nonneg, (float)weight, (float)gamma, (float)hc,
              (float)pg, (float)step, bad, betas, cs};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)n_workers);
  cfg.blockDim = dim3(SM_THREADS);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  if (after_clusters) {  // placed once every cluster CTA is resident (see fgp_cluster.cu)
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  PSB_CUDA(cudaLaunchKernelEx(&cfg, fgp_sm_run_kernel, a));
  PSB_LAUNCHED("fgp_sm_run");
  return PSB_OK;
}

}  // namespace psb

extern "C" {

int psb_aprojgd_dual_rof(int dtype, const void* b, void* q, int H, int W, double alpha,
                         double step, int iters, void* u, void* stream) {
  return psb::aprojgd_dual_rof(dtype, b, q, H, W, alpha, step, iters, u, psb::as_stream(stream));
}

int psb_fgp2d_iter(int dtype, const void* x, int64_t x_pstride, void* q, int64_t q_pstride,
                   const int32_t* active, int n_active, double weight, const double* weights,
                   int reproject_all, const uint8_t* reproject, int H, int W, int it,
                   double beta_prev, double step, int nonneg, void* stream) {
  return psb::fgp2d_iter(dtype, x, x_pstride, q, q_pstride, active, n_active, weight, weights,
                         reproject_all, reproject, H, W, it, beta_prev, step, nonneg,
                         psb::as_stream(stream));
}

int psb_fgp2d_finalize(int dtype, const void* x, int64_t x_pstride, void* q, int64_t q_pstride,
                       const int32_t* active, int n_active, int H, int W, int n_inner, int nonneg,
                       void* u, int64_t u_pstride, void* stream) {
  return psb::fgp2d_finalize(dtype, x, x_pstride, q, q_pstride, active, n_active, H, W, n_inner,
                             nonneg, u, u_pstride, psb::as_stream(stream));
}

int psb_tv_prox2d(int dtype, const void* x, int64_t x_pstride, void* q, int64_t q_pstride,
                  const int32_t* active, int n_active, double weight, const double* weights,
                  int reproject_all, const uint8_t* reproject, int H, int W, int n_inner,
                  int accelerated, int nonneg, double step, void* u, int64_t u_pstride,
                  void* stream) {
  return psb::tv_prox2d(dtype, x, x_pstride, q, q_pstride, active, n_active, weight, weights,
                        reproject_all, reproject, H, W, n_inner, accelerated, nonneg, step, u,
                        u_pstride, psb::as_stream(stream));
}

}  // extern "C"

// 3-D FGP TV prox for BASELINE config 5: the
// reference's 2-D algorithm (tv.py:53-89, operators.py:44-71,
// proximal.py:10-21) on a (D, H, W) volume with dual channels (z, y, x),
// Neumann zeros on the last plane of each axis and dual step 1/12.
//
// One launch = one inner iteration (fgp3d_march_kernel below): warps march
// along z over a chunk of planes keeping their row's y and u in registers;
// every voxel's q_k / q_{k-1} / x is read from HBM once (40 B/voxel-iteration
// fp32: x + q_k(3) + q_{k-1}(3) read, q_{k+1}(3) written).
//
// z-slab decomposition (BASELINE config 5 on N GPUs): a rank owns planes
// [z0, z0 + D) of a volume of depth Dg.  Plane z0-1 (below) and plane z0+D
// (above) come from halo buffers holding the neighbours' (q_k, q_{k-1}) planes
// (and x for the plane above); the boundary tests use GLOBAL plane indices, so
// a slab computes exactly what the whole-volume kernel computes on its planes.
#include "common.cuh"

namespace psb {

namespace {

template <class T>
struct Fgp3Args {
  const T* x;
  T* q;         // slots: q + (s*3 + c) * N3
  int D, H, W;  // local planes, rows, cols
  int z0, Dg;   // global index of local plane 0, global depth
  int it;
  T beta, step, w;
  int rep, nonneg;
  // halo planes: (3, H, W) dual planes of q_k / q_{k-1}; x plane (H, W) above
  const T* hb_qk;
  const T* hb_qm;
  const T* ha_qk;
  const T* ha_qm;
  const T* ha_x;
  int zchunk;  // planes per CTA along z
};

template <class T>
__device__ __forceinline__ void plane_src(const Fgp3Args<T>& a, int kl, const T*& qk, const T*& qm,
                                          int64_t& cstride, int64_t& poff) {
  // kl: local plane index in [-1, D]
  const int64_t HW = (int64_t)a.H * a.W, N3 = (int64_t)a.D * HW;
  if (kl >= 0 && kl < a.D) {
    qk = a.q + (int64_t)(a.it % 3) * 3 * N3;
    qm = a.q + (int64_t)((a.it + 2) % 3) * 3 * N3;
    cstride = N3;
    poff = (int64_t)kl * HW;
  } else if (kl < 0) {
    qk = a.hb_qk;
    qm = a.hb_qm;
    cstride = HW;
    poff = 0;
  } else {
    qk = a.ha_qk;
    qm = a.ha_qm;
    cstride = HW;
    poff = 0;
  }
}

// ProxSkip post for the identity fidelity in 3-D, fused with the FGP finalize
// (u = clamp(z + div q_n), q_n -> slot 0) -- skip.py:70-75, tv.py:86-89.
// `hb_qn` = plane z0-1 of q_n (3, H, W) or NULL at the global bottom.
template <class TO, class TF>
__global__ void proxskip_post3d_kernel(TO* __restrict__ x, const TO* __restrict__ b,
                                       TO* __restrict__ h, const TF* __restrict__ z, TF* q,
                                       const TF* __restrict__ hb_qn, int D, int H, int W, int z0,
                                       int Dg, int n_inner, int nonneg, TO gamma, TO pg,
                                       int pend, int32_t* bad, int kiter) {
  using A = Ar<TO>;
  using F = Ar<TF>;
  const int64_t HW = (int64_t)H * W, N3 = (int64_t)D * HW;
  const int slot = n_inner % 3;
  const TF* qn = q + (int64_t)slot * 3 * N3;
  bool ok = true;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N3;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int kl = (int)(i / HW);
    const int r = (int)((i % HW) / W), c = (int)(i % W);
    const int kg = z0 + kl;
    const TF vz = qn[i], vy = qn[N3 + i], vx = qn[2 * N3 + i];
    TF d = TF(0);
    if (kg < Dg - 1) d = F::add(d, vz);
    if (kg > 0) d = F::sub(d, kl > 0 ? qn[i - HW] : hb_qn[i]);
    if (r < H - 1) d = F::add(d, vy);
    if (r > 0) d = F::sub(d, qn[N3 + i - W]);
    if (c < W - 1) d = F::add(d, vx);
    if (c > 0) d = F::sub(d, qn[2 * N3 + i - 1]);
    TF uf = F::add(z[i], d);
    if (nonneg) uf = uf > TF(0) ? uf : TF(0);
    if (slot != 0) {
      q[i] = vz;
      q[N3 + i] = vy;
      q[2 * N3 + i] = vx;
    }
    TO xo = x[i];
    const TO ho = h[i], bo = b[i];
    // the `pend` deferred skip iterations since x was last stored (skip.py:68)
    for (int s = 0; s < pend; ++s)
      xo = A::add(A::sub(xo, A::mul(gamma, A::sub(xo, bo))), A::mul(gamma, ho));
    const TO xhat = A::add(A::sub(xo, A::mul(gamma, A::sub(xo, bo))), A::mul(gamma, ho));
    const TO xn = (TO)uf;
    h[i] = A::add(ho, A::mul(pg, A::sub(xn, xhat)));
    x[i] = xn;
    ok &= finite(xn);
  }
  if (!ok && bad) atomicMin(bad, kiter);
}

// ---- register z-march (v2) -------------------------------------------------
// CTA = (MTY + 2) warps; warp w owns image row i0 - 1 + w of a band of 32*V
// columns and marches along z keeping y(k), u(k) of its row in registers.
// Warps 1..MTY produce output; warp 0 (row i0-1) only supplies y_y for warp
// 1's divergence and warp MTY+1 (row i0+MTY) only supplies u for warp MTY's
// y-gradient.  Rows meet in shared memory (1 __syncthreads per plane), columns
// through shuffles plus one predicated halo column per warp edge, planes
// through registers.  HBM: x + q_k(3) + q_{k-1}(3) read, q_{k+1}(3) written
// once per voxel-iteration (40 B fp32), row/column halos re-read from L2.
constexpr int MTY = 8;

template <class T, int V>
struct Row3 {
  T y[3][V];  // z, y, x channels of the momentum point y
  T h[3];     // halo column (lane 0: c0-1, lane 31: c0+32V)
  T u[V];
  T hu;
};

// ---- cp.async staging: each lane copies its own row segment of the 7 plane
// arrays (q_k 3 ch, q_{k-1} 3 ch, x) into a 2-stage shared-memory ring one
// plane ahead of the compute, so DRAM latency overlaps a whole plane step.
__device__ __forceinline__ void cp_async_16(void* dst, const void* src, bool pred) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(n));
}
template <int B>
__device__ __forceinline__ void cp_async_small(void* dst, const void* src, bool pred) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int n = pred ? B : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(d), "l"(src), "n"(B), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <class T, int V>
__device__ __forceinline__ void copy_vec(T* dst, const T* src, bool pred) {
  if constexpr (sizeof(T) * V == 16) {
    cp_async_16(dst, src, pred);
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) cp_async_small<sizeof(T)>(dst + v, src + v, pred);
  }
}

// stage layout per warp: [7][32*V] (arrays: k0 k1 k2 m0 m1 m2 x) + halo [7][2]
template <class T, int V>
__device__ __forceinline__ void issue_plane(const Fgp3Args<T>& a, int kl, int i, int cl, bool lin,
                                            int hc, bool hval, bool mom, int lane, T* st, T* hs) {
  const T* qk;
  const T* qm;
  int64_t cs, po;
  plane_src(a, kl, qk, qm, cs, po);
  const int64_t HW = (int64_t)a.H * a.W;
  const T* xs = (kl < 0) ? nullptr : (kl < a.D ? a.x + (int64_t)kl * HW : a.ha_x);
  constexpr int BW = 32 * V;
  const T* dummy = a.x;
  const int64_t o = po + (int64_t)i * a.W + cl;
  const bool lq = lin && qk != nullptr;
  const bool lm = lq && mom;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    copy_vec<T, V>(st + c * BW + lane * V, lq ? qk + c * cs + o : dummy, lq);
    copy_vec<T, V>(st + (3 + c) * BW + lane * V, lm ? qm + c * cs + o : dummy, lm);
  }
  const bool lx = lin && xs != nullptr;
  copy_vec<T, V>(st + 6 * BW + lane * V, lx ? xs + (int64_t)i * a.W + cl : dummy, lx);
  if (lane == 0 || lane == 31) {
    const int hs_i = lane == 0 ? 0 : 1;
    const int64_t oh = po + (int64_t)i * a.W + hc;
    const bool hq = hval && qk != nullptr, hm = hq && mom, hx = hval && xs != nullptr;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      cp_async_small<sizeof(T)>(hs + c * 2 + hs_i, hq ? qk + c * cs + oh : dummy, hq);
      cp_async_small<sizeof(T)>(hs + (3 + c) * 2 + hs_i, hm ? qm + c * cs + oh : dummy, hm);
    }
    cp_async_small<sizeof(T)>(hs + 6 * 2 + hs_i, hx ? xs + (int64_t)i * a.W + hc : dummy, hx);
  }
}

template <class T, int V>
__device__ __forceinline__ void read_plane(const Fgp3Args<T>& a, bool mom, bool rp, int lane,
                                           const T* st, const T* hs, Row3<T, V>& R, T (&xv)[V],
                                           T& hx) {
  using A = Ar<T>;
  constexpr int BW = 32 * V;
  T k[3][V], m[3][V];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    ldv_s<T, V>(k[c], st + c * BW + lane * V);
    if (mom) ldv_s<T, V>(m[c], st + (3 + c) * BW + lane * V);
  }
  ldv_s<T, V>(xv, st + 6 * BW + lane * V);
  auto y_of = [&](T& v0, T& v1, T& v2, T n0, T n1, T n2) {
    if (rp) {
      const T s = A::ball_scale3(v0, v1, v2, a.w);
      v0 = A::mul(v0, s);
      v1 = A::mul(v1, s);
      v2 = A::mul(v2, s);
    }
    if (mom) {
      v0 = A::add(v0, A::mul(a.beta, A::sub(v0, n0)));
      v1 = A::add(v1, A::mul(a.beta, A::sub(v1, n1)));
      v2 = A::add(v2, A::mul(a.beta, A::sub(v2, n2)));
    }
  };
#pragma unroll
  for (int v = 0; v < V; ++v) {
    T v0 = k[0][v], v1 = k[1][v], v2 = k[2][v];
    y_of(v0, v1, v2, m[0][v], m[1][v], m[2][v]);
    R.y[0][v] = v0;
    R.y[1][v] = v1;
    R.y[2][v] = v2;
  }
  const int hi = lane == 31 ? 1 : 0;
  T h0 = hs[0 * 2 + hi], h1 = hs[1 * 2 + hi], h2 = hs[2 * 2 + hi];
  y_of(h0, h1, h2, hs[3 * 2 + hi], hs[4 * 2 + hi], hs[5 * 2 + hi]);
  R.h[0] = h0;
  R.h[1] = h1;
  R.h[2] = h2;
  hx = hs[6 * 2 + hi];
}

template <class T, int V>
__global__ void __launch_bounds__((MTY + 2) * 32, 2) fgp3d_march_kernel(Fgp3Args<T> a) {
  using A = Ar<T>;
  constexpr int BW = 32 * V;
  // row exchange (vector-aligned rows; the band's right halo column apart)
  __shared__ __align__(16) T s_yy[2][MTY + 2][BW];
  __shared__ T s_yyh[2][MTY + 2];
  __shared__ __align__(16) T s_u[2][MTY + 2][BW];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = blockIdx.x * BW;
  const int i = blockIdx.y * MTY - 1 + w;
  const int ks = blockIdx.z * a.zchunk;
  const int ke = min(a.D, ks + a.zchunk);
  if (ks >= ke) return;
  const int H = a.H, W = a.W;
  const bool row_ok = i >= 0 && i < H;
  const int cl = c0 + lane * V;
  const bool lin = row_ok && cl < W;
  const int hc = lane == 0 ? c0 - 1 : c0 + BW;
  const bool hval = row_ok && ((lane == 0 && c0 > 0) || (lane == 31 && hc < W));
  const bool mom = a.beta != T(0);
  const bool rp = a.rep && a.it == 0;
  const bool out_row = w >= 1 && w <= MTY && row_ok;
  const int64_t HW = (int64_t)H * W, N3 = (int64_t)a.D * HW;
  T* qo = a.q + (int64_t)((a.it + 1) % 3) * 3 * N3;

  // u(plane) of this row from its y (cur), y_z of the plane below (yzp, hyzp),
  // y_y of the row above (s_yy[w-1]) and the left neighbour's y_x.
  auto prim = [&](int kg, Row3<T, V>& R, const T (&yzp)[V], T hyzp, const T (&xv)[V], T hx,
                  int par) {
    T left = __shfl_up_sync(0xffffffffu, R.y[2][V - 1], 1);
    if (lane == 0) left = R.h[2];
    T yup[V];
    if (w > 0) ldv_s<T, V>(yup, &s_yy[par][w - 1][lane * V]);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int c = cl + v;
      T d = T(0);
      if (kg < a.Dg - 1) d = A::add(d, R.y[0][v]);
      if (kg > 0) d = A::sub(d, yzp[v]);
      if (i < H - 1) d = A::add(d, R.y[1][v]);
      if (i > 0) d = A::sub(d, w > 0 ? yup[v] : T(0));
      if (c < W - 1) d = A::add(d, R.y[2][v]);
      if (c > 0) d = A::sub(d, v > 0 ? R.y[2][v - 1] : left);
      T u = A::add(xv[v], d);
      R.u[v] = a.nonneg ? (u > T(0) ? u : T(0)) : u;
    }
    if (lane == 31) {  // halo column c0 + BW
      const int c = hc;
      T d = T(0);
      if (kg < a.Dg - 1) d = A::add(d, R.h[0]);
      if (kg > 0) d = A::sub(d, hyzp);
      if (i < H - 1) d = A::add(d, R.h[1]);
      if (i > 0) d = A::sub(d, w > 0 ? s_yyh[par][w - 1] : T(0));
      if (c < W - 1) d = A::add(d, R.h[2]);
      if (c > 0) d = A::sub(d, R.y[2][V - 1]);
      T u = A::add(hx, d);
      R.hu = a.nonneg ? (u > T(0) ? u : T(0)) : u;
    }
  };
  auto publish_yy = [&](const Row3<T, V>& R, int par) {
    stv<T, V>(&s_yy[par][w][lane * V], R.y[1]);
    if (lane == 31) s_yyh[par][w] = R.h[1];
  };
  auto publish_u = [&](const Row3<T, V>& R, int par) { stv<T, V>(&s_u[par][w][lane * V], R.u); };

  extern __shared__ unsigned char dyn_smem[];
  T* stage0 = reinterpret_cast<T*>(dyn_smem);
  constexpr int SW = 7 * BW;  // per-warp stage floats
  T* hs_all = stage0 + (size_t)2 * (MTY + 2) * SW;
  auto st_ptr = [&](int sidx) { return stage0 + (size_t)(sidx * (MTY + 2) + w) * SW; };
  auto hs_ptr = [&](int sidx) { return hs_all + (size_t)(sidx * (MTY + 2) + w) * 14; };

  Row3<T, V> C, N;
  T yzp[V], hyzp = T(0), xv[V], hx;
#pragma unroll
  for (int v = 0; v < V; ++v) yzp[v] = T(0);
  // prologue: y_z of plane ks-1 (synchronously), then planes ks and ks+1 in flight
  if (a.z0 + ks > 0) {
    T xd[V], hxd;
    issue_plane<T, V>(a, ks - 1, i, cl, lin, hc, hval, mom, lane, st_ptr(0), hs_ptr(0));
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    read_plane<T, V>(a, mom, rp, lane, st_ptr(0), hs_ptr(0), N, xd, hxd);
#pragma unroll
    for (int v = 0; v < V; ++v) yzp[v] = N.y[0][v];
    hyzp = N.h[0];
    __syncwarp();
  }
  issue_plane<T, V>(a, ks, i, cl, lin, hc, hval, mom, lane, st_ptr(0), hs_ptr(0));
  cp_async_commit();
  if (a.z0 + ks + 1 < a.Dg)
    issue_plane<T, V>(a, ks + 1, i, cl, lin, hc, hval, mom, lane, st_ptr(1), hs_ptr(1));
  cp_async_commit();
  cp_async_wait<1>();
  __syncwarp();
  read_plane<T, V>(a, mom, rp, lane, st_ptr(0), hs_ptr(0), C, xv, hx);
  publish_yy(C, ks & 1);
  __syncthreads();
  prim(a.z0 + ks, C, yzp, hyzp, xv, hx, ks & 1);
  publish_u(C, ks & 1);

  // One barrier per plane: y_y rows and u rows are double-buffered by plane
  // parity, so the barrier that publishes y_y(k+1) also publishes u(k) (written
  // in the previous step) for this step's y-gradient.

  for (int k = ks; k < ke; ++k) {
    const int kg = a.z0 + k;
    const bool nxt = kg + 1 < a.Dg;
    if (nxt) {
      // plane k+1 was issued one step ago into stage (k+1-ks)&1; put plane k+2
      // into the stage plane k used, then wait for plane k+1 only
      const int sn = (k + 1 - ks) & 1;
      if (kg + 2 < a.Dg)
        issue_plane<T, V>(a, k + 2, i, cl, lin, hc, hval, mom, lane, st_ptr(sn ^ 1), hs_ptr(sn ^ 1));
      cp_async_commit();
      cp_async_wait<1>();
      __syncwarp();
      read_plane<T, V>(a, mom, rp, lane, st_ptr(sn), hs_ptr(sn), N, xv, hx);
      publish_yy(N, (k + 1) & 1);
    }
    __syncthreads();
    if (nxt) {
      T yzc[V];
#pragma unroll
      for (int v = 0; v < V; ++v) yzc[v] = C.y[0][v];
      prim(kg + 1, N, yzc, C.h[0], xv, hx, (k + 1) & 1);
      publish_u(N, (k + 1) & 1);
    }
    if (out_row) {
      T right = __shfl_down_sync(0xffffffffu, C.u[0], 1);
      if (lane == 31) right = C.hu;
      T oz[V], oy[V], ox[V], udn[V];
      ldv_s<T, V>(udn, &s_u[k & 1][w + 1][lane * V]);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int c = cl + v;
        const T uc = C.u[v];
        const T gz = nxt ? A::sub(N.u[v], uc) : T(0);
        const T gy = i < H - 1 ? A::sub(udn[v], uc) : T(0);
        const T ur = v < V - 1 ? C.u[v + 1] : right;
        const T gx = c < W - 1 ? A::sub(ur, uc) : T(0);
        const T az = A::add(C.y[0][v], A::mul(a.step, gz));
        const T ay = A::add(C.y[1][v], A::mul(a.step, gy));
        const T ax = A::add(C.y[2][v], A::mul(a.step, gx));
        const T sc = A::ball_scale3(az, ay, ax, a.w);
        oz[v] = A::mul(az, sc);
        oy[v] = A::mul(ay, sc);
        ox[v] = A::mul(ax, sc);
      }
      if (lin) {
        const int64_t o = (int64_t)k * HW + (int64_t)i * W + cl;
        stv<T, V>(qo + o, oz);
        stv<T, V>(qo + N3 + o, oy);
        stv<T, V>(qo + 2 * N3 + o, ox);
      }
    } else {
      // keep the shuffle participation uniform across the warp
      (void)__shfl_down_sync(0xffffffffu, C.u[0], 1);
    }
    C = N;
  }
}

template <class T, int V>
size_t march_smem() {
  return sizeof(T) * ((size_t)2 * (MTY + 2) * 7 * 32 * V + (size_t)2 * (MTY + 2) * 14);
}

template <class T>
int launch3(const Fgp3Args<T>& a, cudaStream_t st) {
  constexpr int VMAX = 16 / sizeof(T);
  const int zc = a.zchunk;
  const int nz = (a.D + zc - 1) / zc;
  const bool vec = (a.W % VMAX == 0) && (reinterpret_cast<uintptr_t>(a.x) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(a.q) % 16 == 0);
  if (vec) {
    const size_t sm = march_smem<T, VMAX>();
    PSB_CUDA(cudaFuncSetAttribute(fgp3d_march_kernel<T, VMAX>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    dim3 grid((a.W + 32 * VMAX - 1) / (32 * VMAX), (a.H + MTY - 1) / MTY, nz);
    fgp3d_march_kernel<T, VMAX><<<grid, (MTY + 2) * 32, sm, st>>>(a);
  } else {
    const size_t sm = march_smem<T, 1>();
    PSB_CUDA(cudaFuncSetAttribute(fgp3d_march_kernel<T, 1>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    dim3 grid((a.W + 31) / 32, (a.H + MTY - 1) / MTY, nz);
    fgp3d_march_kernel<T, 1><<<grid, (MTY + 2) * 32, sm, st>>>(a);
  }
  PSB_LAUNCHED("fgp3d_march");
  return PSB_OK;
}

}  // namespace

int fgp3d_iter(int dtype, const void* x, void* q, int D, int H, int W, int z0, int Dg, int it,
               double beta, double step, double weight, int rep, int nonneg, const void* hb_qk,
               const void* hb_qm, const void* ha_qk, const void* ha_qm, const void* ha_x,
               int zchunk, cudaStream_t st) {
  PSB_REQUIRE(D >= 1 && H >= 2 && W >= 2 && Dg >= 2, "fgp3d: need a 3-D grid with sides >= 2");
  PSB_REQUIRE(z0 >= 0 && z0 + D <= Dg, "fgp3d: slab outside the volume");
  PSB_REQUIRE(weight > 0, "tv_prox: weight must be positive");
  PSB_REQUIRE(z0 == 0 || (hb_qk && hb_qm), "fgp3d: slab above plane 0 needs the halo below");
  PSB_REQUIRE(z0 + D == Dg || (ha_qk && ha_qm && ha_x), "fgp3d: slab below the top needs the halo above");
  if (zchunk <= 0) {
    // enough CTAs for ~4 waves; long chunks amortise the two halo planes
    const int64_t tiles = (int64_t)((W + 127) / 128) * ((H + MTY - 1) / MTY);
    const int64_t want = 32LL * sm_count();  // ~16 waves at 2 CTAs/SM: small tail
    int nz = (int)std::max<int64_t>(1, std::min<int64_t>(D, (want + tiles - 1) / tiles));
    zchunk = std::max(16, (D + nz - 1) / nz);
  }
  if (dtype == PSB_F32) {
    Fgp3Args<float> a{(const float*)x, (float*)q, D, H, W, z0, Dg, it, (float)beta, (float)step,
                      (float)weight, rep, nonneg, (const float*)hb_qk, (const float*)hb_qm,
                      (const float*)ha_qk, (const float*)ha_qm, (const float*)ha_x, zchunk};
    return launch3(a, st);
  }
  if (dtype == PSB_F64) {
    Fgp3Args<double> a{(const double*)x, (double*)q, D, H, W, z0, Dg, it, beta, step, weight, rep,
                       nonneg, (const double*)hb_qk, (const double*)hb_qm, (const double*)ha_qk,
                       (const double*)ha_qm, (const double*)ha_x, zchunk};
    return launch3(a, st);
  }
  return fail(PSB_ERR_VALUE, "fgp3d: unknown dtype");
}

int proxskip_post3d(int dto, int dtf, void* x, const void* b, void* h, const void* z, void* q,
                    const void* hb_qn, int D, int H, int W, int z0, int Dg, int n_inner,
                    int nonneg, double gamma, double pg, int pend, int32_t* bad, int k,
                    cudaStream_t st) {
  PSB_REQUIRE(z0 == 0 || hb_qn, "proxskip3d: slab above plane 0 needs the halo below");
  PSB_REQUIRE(pend >= 0, "proxskip3d: negative deferred-skip count");
  const int64_t N3 = (int64_t)D * H * W;
  dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((N3 + 255) / 256, 16LL * sm_count())));
  if (dto == PSB_F32 && dtf == PSB_F32)
    proxskip_post3d_kernel<float, float><<<grid, 256, 0, st>>>(
        (float*)x, (const float*)b, (float*)h, (const float*)z, (float*)q, (const float*)hb_qn, D,
        H, W, z0, Dg, n_inner, nonneg, (float)gamma, (float)pg, pend, bad, k);
  else if (dto == PSB_F64 && dtf == PSB_F64)
    proxskip_post3d_kernel<double, double><<<grid, 256, 0, st>>>(
        (double*)x, (const double*)b, (double*)h, (const double*)z, (double*)q,
        (const double*)hb_qn, D, H, W, z0, Dg, n_inner, nonneg, gamma, pg, pend, bad, k);
  else if (dto == PSB_F64 && dtf == PSB_F32)
    proxskip_post3d_kernel<double, float><<<grid, 256, 0, st>>>(
        (double*)x, (const double*)b, (double*)h, (const float*)z, (float*)q, (const float*)hb_qn,
        D, H, W, z0, Dg, n_inner, nonneg, gamma, pg, pend, bad, k);
  else
    return fail(PSB_ERR_VALUE, "proxskip3d: unsupported dtype pair");
  PSB_LAUNCHED("proxskip_post3d");
  return PSB_OK;
}

}  // namespace psb

extern "C" {

int psb_fgp3d_iter(int dtype, const void* x, void* q, int D, int H, int W, int z0, int Dg, int it,
                   double beta_prev, double step, double weight, int reproject, int nonneg,
                   const void* halo_below_qk, const void* halo_below_qm, const void* halo_above_qk,
                   const void* halo_above_qm, const void* halo_above_x, int zchunk, void* stream) {
  return psb::fgp3d_iter(dtype, x, q, D, H, W, z0, Dg, it, beta_prev, step, weight, reproject,
                         nonneg, halo_below_qk, halo_below_qm, halo_above_qk, halo_above_qm,
                         halo_above_x, zchunk, psb::as_stream(stream));
}

int psb_proxskip_post3d(int dtype_outer, int dtype_fgp, void* x, const void* b, void* h,
                        const void* z, void* q, const void* halo_below_qn, int D, int H, int W,
                        int z0, int Dg, int n_inner, int nonneg, double gamma, double pg,
                        int pend, int32_t* bad_iter, int k, void* stream) {
  return psb::proxskip_post3d(dtype_outer, dtype_fgp, x, b, h, z, q, halo_below_qn, D, H, W, z0,
                              Dg, n_inner, nonneg, gamma, pg, pend, bad_iter, k,
                              psb::as_stream(stream));
}

}  // extern "C"

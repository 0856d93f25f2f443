// 3-D FGP TV prox for BASELINE config 5: the
// reference's 2-D algorithm (tv.py:53-89, operators.py:44-71,
// proximal.py:10-21) on a (D, H, W) volume with dual channels (z, y, x),
// Neumann zeros on the last plane of each axis and dual step 1/12.
//
// One launch = one inner iteration.  2.5-D blocking: a CTA owns a TY x TX
// column tile and marches along z over a chunk of planes.  Per plane it
// stages y = q_k + beta (q_k - q_{k-1}) for the tile plus a one-voxel halo in
// shared memory, forms u = clamp(x + div y) on the tile plus the +1 row/col
// halo, and writes q_{k+1} for the previous plane; the y and u planes rotate
// through shared memory so every voxel's q_k / q_{k-1} / x is read from HBM
// once (40 B/voxel-iteration fp32: x + q_k(3) + q_{k-1}(3) read, q_{k+1}(3)
// write).
//
// z-slab decomposition (BASELINE config 5 on N GPUs): a rank owns planes
// [z0, z0 + D) of a volume of depth Dg.  Plane z0-1 (below) and plane z0+D
// (above) come from halo buffers holding the neighbours' (q_k, q_{k-1}) planes
// (and x for the plane above); the boundary tests use GLOBAL plane indices, so
// a slab computes exactly what the whole-volume kernel computes on its planes.
#include "common.cuh"

namespace psb {

namespace {

constexpr int TY = 8, TX = 32;
constexpr int RY = TY + 2, RX = TX + 2;  // y region: rows i0-1..i0+TY, cols j0-1..j0+TX

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

template <class T>
__device__ __forceinline__ void load_yplane(const Fgp3Args<T>& a, int kl, int i0, int j0,
                                            T (*sy)[RY][RX]) {
  using A = Ar<T>;
  const T* qk;
  const T* qm;
  int64_t cs, po;
  plane_src(a, kl, qk, qm, cs, po);
  const bool mom = a.beta != T(0);
  const bool rp = a.rep && a.it == 0;
  const int tid = threadIdx.y * blockDim.x + threadIdx.x, nt = blockDim.x * blockDim.y;
  for (int e = tid; e < RY * RX; e += nt) {
    const int ry = e / RX, rx = e % RX;
    const int r = i0 - 1 + ry, c = j0 - 1 + rx;
    T v0 = T(0), v1 = T(0), v2 = T(0);
    if (r >= 0 && r < a.H && c >= 0 && c < a.W && qk != nullptr) {
      const int64_t o = po + (int64_t)r * a.W + c;
      v0 = qk[o];
      v1 = qk[cs + o];
      v2 = qk[2 * cs + o];
      if (rp) {
        const T s = A::ball_scale3(v0, v1, v2, a.w);
        v0 = A::mul(v0, s);
        v1 = A::mul(v1, s);
        v2 = A::mul(v2, s);
      }
      if (mom) {
        v0 = A::add(v0, A::mul(a.beta, A::sub(v0, qm[o])));
        v1 = A::add(v1, A::mul(a.beta, A::sub(v1, qm[cs + o])));
        v2 = A::add(v2, A::mul(a.beta, A::sub(v2, qm[2 * cs + o])));
      }
    }
    sy[0][ry][rx] = v0;
    sy[1][ry][rx] = v1;
    sy[2][ry][rx] = v2;
  }
}

// u(kl) = clamp(x + div y) on rows i0..i0+TY, cols j0..j0+TX; `yc` = y(kl), `yp` = y(kl-1)
template <class T>
__device__ __forceinline__ void prim_plane(const Fgp3Args<T>& a, int kl, int i0, int j0,
                                           T (*yc)[RY][RX], T (*yp)[RY][RX],
                                           T (*su)[TX + 1]) {
  using A = Ar<T>;
  const int kg = a.z0 + kl;
  const int64_t HW = (int64_t)a.H * a.W;
  const T* xs = (kl < a.D) ? a.x + (int64_t)kl * HW : a.ha_x;
  const int tid = threadIdx.y * blockDim.x + threadIdx.x, nt = blockDim.x * blockDim.y;
  for (int e = tid; e < (TY + 1) * (TX + 1); e += nt) {
    const int uy = e / (TX + 1), ux = e % (TX + 1);
    const int ry = uy + 1, rx = ux + 1;
    const int r = i0 + uy, c = j0 + ux;
    T u = T(0);
    if (r < a.H && c < a.W) {
      T d = T(0);
      if (kg < a.Dg - 1) d = A::add(d, yc[0][ry][rx]);
      if (kg > 0) d = A::sub(d, yp[0][ry][rx]);
      if (r < a.H - 1) d = A::add(d, yc[1][ry][rx]);
      if (r > 0) d = A::sub(d, yc[1][ry - 1][rx]);
      if (c < a.W - 1) d = A::add(d, yc[2][ry][rx]);
      if (c > 0) d = A::sub(d, yc[2][ry][rx - 1]);
      u = A::add(xs[(int64_t)r * a.W + c], d);
      if (a.nonneg) u = u > T(0) ? u : T(0);
    }
    su[uy][ux] = u;
  }
}

template <class T>
__global__ void __launch_bounds__(TX * TY) fgp3d_iter_kernel(Fgp3Args<T> a) {
  using A = Ar<T>;
  __shared__ T sy[3][3][RY][RX];      // three rotating y planes (prev, cur, next)
  __shared__ T su[2][TY + 1][TX + 1];  // u planes (cur, next)
  const int i0 = blockIdx.y * TY, j0 = blockIdx.x * TX;
  const int ks = blockIdx.z * a.zchunk;
  const int ke = min(a.D, ks + a.zchunk);
  if (ks >= ke) return;
  const int64_t HW = (int64_t)a.H * a.W, N3 = (int64_t)a.D * HW;
  T* qo = a.q + (int64_t)((a.it + 1) % 3) * 3 * N3;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int r = i0 + ty, c = j0 + tx;

  int P = 0, Cc = 1, Nn = 2, UC = 0, UN = 1;
  // prologue: y(ks - 1) (only its z channel is used), y(ks), u(ks)
  if (a.z0 + ks > 0) load_yplane(a, ks - 1, i0, j0, sy[P]);
  load_yplane(a, ks, i0, j0, sy[Cc]);
  __syncthreads();
  prim_plane(a, ks, i0, j0, sy[Cc], sy[P], su[UC]);
  __syncthreads();
  for (int k = ks; k < ke; ++k) {
    const int kg = a.z0 + k;
    const bool nxt = kg + 1 < a.Dg;
    if (nxt) {
      load_yplane(a, k + 1, i0, j0, sy[Nn]);
      __syncthreads();
      prim_plane(a, k + 1, i0, j0, sy[Nn], sy[Cc], su[UN]);
      __syncthreads();
    }
    if (r < a.H && c < a.W) {
      const int ry = ty + 1, rx = tx + 1;
      const T uc = su[UC][ty][tx];
      const T gz = nxt ? A::sub(su[UN][ty][tx], uc) : T(0);
      const T gy = r < a.H - 1 ? A::sub(su[UC][ty + 1][tx], uc) : T(0);
      const T gx = c < a.W - 1 ? A::sub(su[UC][ty][tx + 1], uc) : T(0);
      const T az = A::add(sy[Cc][0][ry][rx], A::mul(a.step, gz));
      const T ay = A::add(sy[Cc][1][ry][rx], A::mul(a.step, gy));
      const T ax = A::add(sy[Cc][2][ry][rx], A::mul(a.step, gx));
      const T s = A::ball_scale3(az, ay, ax, a.w);
      const int64_t o = (int64_t)k * HW + (int64_t)r * a.W + c;
      qo[o] = A::mul(az, s);
      qo[N3 + o] = A::mul(ay, s);
      qo[2 * N3 + o] = A::mul(ax, s);
    }
    __syncthreads();
    const int t = P;
    P = Cc;
    Cc = Nn;
    Nn = t;
    UC ^= 1;
    UN ^= 1;
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
                                       int32_t* bad, int kiter) {
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
    const TO xo = x[i], ho = h[i];
    const TO xhat = A::add(A::sub(xo, A::mul(gamma, A::sub(xo, b[i]))), A::mul(gamma, ho));
    const TO xn = (TO)uf;
    h[i] = A::add(ho, A::mul(pg, A::sub(xn, xhat)));
    x[i] = xn;
    ok &= finite(xn);
  }
  if (!ok && bad) atomicMin(bad, kiter);
}

template <class T>
int launch3(const Fgp3Args<T>& a, cudaStream_t st) {
  dim3 block(TX, TY);
  const int zc = a.zchunk;
  dim3 grid((a.W + TX - 1) / TX, (a.H + TY - 1) / TY, (a.D + zc - 1) / zc);
  fgp3d_iter_kernel<T><<<grid, block, 0, st>>>(a);
  PSB_LAUNCHED("fgp3d_iter");
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
    const int64_t tiles = (int64_t)((W + TX - 1) / TX) * ((H + TY - 1) / TY);
    const int64_t want = 4LL * sm_count() * 6;
    int nz = (int)std::max<int64_t>(1, std::min<int64_t>(D, (want + tiles - 1) / tiles));
    zchunk = std::max(8, (D + nz - 1) / nz);
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
                    int nonneg, double gamma, double pg, int32_t* bad, int k, cudaStream_t st) {
  PSB_REQUIRE(z0 == 0 || hb_qn, "proxskip3d: slab above plane 0 needs the halo below");
  const int64_t N3 = (int64_t)D * H * W;
  dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((N3 + 255) / 256, 16LL * sm_count())));
  if (dto == PSB_F32 && dtf == PSB_F32)
    proxskip_post3d_kernel<float, float><<<grid, 256, 0, st>>>(
        (float*)x, (const float*)b, (float*)h, (const float*)z, (float*)q, (const float*)hb_qn, D,
        H, W, z0, Dg, n_inner, nonneg, (float)gamma, (float)pg, bad, k);
  else if (dto == PSB_F64 && dtf == PSB_F64)
    proxskip_post3d_kernel<double, double><<<grid, 256, 0, st>>>(
        (double*)x, (const double*)b, (double*)h, (const double*)z, (double*)q,
        (const double*)hb_qn, D, H, W, z0, Dg, n_inner, nonneg, gamma, pg, bad, k);
  else if (dto == PSB_F64 && dtf == PSB_F32)
    proxskip_post3d_kernel<double, float><<<grid, 256, 0, st>>>(
        (double*)x, (const double*)b, (double*)h, (const float*)z, (float*)q, (const float*)hb_qn,
        D, H, W, z0, Dg, n_inner, nonneg, gamma, pg, bad, k);
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
                        int32_t* bad_iter, int k, void* stream) {
  return psb::proxskip_post3d(dtype_outer, dtype_fgp, x, b, h, z, q, halo_below_qn, D, H, W, z0,
                              Dg, n_inner, nonneg, gamma, pg, bad_iter, k, psb::as_stream(stream));
}

}  // extern "C"

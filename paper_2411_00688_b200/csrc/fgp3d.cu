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
#include <cuda.h>
#include <cstring>
#include <cstdlib>
#include <cudaTypedefs.h>

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
  // plane subset (overlapped slab schedule): 0 = all planes [0, D),
  // 1 = interior [1, D-1) (needs no halo), 2 = the two edge planes 0, D-1
  int part;
  // optional copies of the new q_{it+1} of plane 0 / plane D-1 (3, H, W),
  // written next to the slot store: the neighbours' receive rings (peer
  // memory over NVLink) or a local send buffer
  T* send_lo;
  T* send_hi;
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
    const TO ho = h[i], bo = b[i];
    // the `pend` deferred skip iterations since x was last stored (skip.py:68;
    // fixed-point exit, common.cuh -- non-finite values were reported by the
    // skip chain that formed z)
    int unused = 0x7fffffff;
    const TO xo = skip_chain_px(x[i], bo, ho, gamma, pend, 0, &unused);
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

// ---- TMA staging (fp32, 16-B vector rows) ----------------------------------
// One elected thread loads a whole plane tile of the CTA -- rows i0-1 ..
// i0+MTY, columns c0-4 .. c0+131 (the band plus one 16-B chunk on each side
// for the halo columns) -- with three tensor-map copies (q_k: 3 channels, q_{k-1}:
// 3 channels, x); out-of-range rows / columns are zero-filled by the copy
// engine, which is what the per-lane cp.async path does with zero-size
// copies.  Completion is counted in bytes on one mbarrier per stage.
constexpr int TBW = 32 * 4 + 8;           // 136 columns per tile row
constexpr int TROWS = MTY + 2;            // 10 rows
constexpr int TQ = 3 * TROWS * TBW;       // floats of a 3-channel q tile
constexpr int TX = TROWS * TBW;           // floats of an x tile
constexpr int TQ_PAD = (TQ * 4 + 127) / 128 * 32;  // floats, 128-B aligned regions
constexpr int TX_PAD = (TX * 4 + 127) / 128 * 32;
constexpr int TSTAGE = 2 * TQ_PAD + TX_PAD;        // floats per stage

struct Fgp3Maps {
  CUtensorMap q;      // (9 = slot*3 + channel, D, H, W) main dual slots
  CUtensorMap x;      // (D, H, W)
  CUtensorMap hb_qk;  // (3, H, W) halo planes (slabs)
  CUtensorMap hb_qm;
  CUtensorMap ha_qk;
  CUtensorMap ha_qm;
  CUtensorMap ha_x;   // (H, W)
};

__device__ __forceinline__ uint32_t sm32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void tma_ld4(void* dst, const CUtensorMap* m, int c0, int c1, int c2,
                                        int c3, uint64_t* mb) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(sm32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(sm32(mb))
      : "memory");
}
__device__ __forceinline__ void tma_ld3(void* dst, const CUtensorMap* m, int c0, int c1, int c2,
                                        uint64_t* mb) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(sm32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(sm32(mb))
      : "memory");
}
__device__ __forceinline__ void tma_ld2(void* dst, const CUtensorMap* m, int c0, int c1,
                                        uint64_t* mb) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(sm32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(sm32(mb))
      : "memory");
}
__device__ __forceinline__ void mb_init(uint64_t* m) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sm32(m)));
}
__device__ __forceinline__ void mb_expect(uint64_t* m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sm32(m)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* m, unsigned parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W_%=;\n}\n" ::"r"(sm32(m)),
      "r"(parity)
      : "memory");
}

// issue plane kl (local index in [-1, D]) into stage `st` (thread 0 only)
__device__ __forceinline__ void tma_issue_plane(const Fgp3Args<float>& a, const Fgp3Maps& M,
                                                int kl, bool mom, int c0, int i0, float* st,
                                                uint64_t* mb) {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  const bool has_x = kl >= 0;  // plane z0-1 is only read for its y_z
  const unsigned bytes = (unsigned)(4 * (TQ + (mom ? TQ : 0) + (has_x ? TX : 0)));
  mb_expect(mb, bytes);
  const int sk = (a.it % 3) * 3, sm = ((a.it + 2) % 3) * 3;
  if (kl >= 0 && kl < a.D) {
    tma_ld4(st, &M.q, c0 - 4, i0, kl, sk, mb);
    if (mom) tma_ld4(st + TQ_PAD, &M.q, c0 - 4, i0, kl, sm, mb);
    tma_ld3(st + 2 * TQ_PAD, &M.x, c0 - 4, i0, kl, mb);
  } else if (kl < 0) {
    tma_ld3(st, &M.hb_qk, c0 - 4, i0, 0, mb);
    if (mom) tma_ld3(st + TQ_PAD, &M.hb_qm, c0 - 4, i0, 0, mb);
  } else {
    tma_ld3(st, &M.ha_qk, c0 - 4, i0, 0, mb);
    if (mom) tma_ld3(st + TQ_PAD, &M.ha_qm, c0 - 4, i0, 0, mb);
    tma_ld2(st + 2 * TQ_PAD, &M.ha_x, c0 - 4, i0, mb);
  }
}

// the row of warp w from a TMA stage: same values the cp.async path stages
__device__ __forceinline__ void tma_read_plane(const Fgp3Args<float>& a, bool mom, bool rp,
                                               int w, int lane, const float* st,
                                               Row3<float, 4>& R, float (&xv)[4], float& hx) {
  using A = Ar<float>;
  const float* qk = st + w * TBW + 4 + lane * 4;
  const float* qm = qk + TQ_PAD;
  const float* xs = st + 2 * TQ_PAD + w * TBW + 4 + lane * 4;
  float k[3][4], m[3][4];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    ldv_s<float, 4>(k[c], qk + c * TROWS * TBW);
    if (mom) ldv_s<float, 4>(m[c], qm + c * TROWS * TBW);
  }
  ldv_s<float, 4>(xv, xs);
  auto y_of = [&](float& v0, float& v1, float& v2, float n0, float n1, float n2) {
    if (rp) {
      const float s = A::ball_scale3(v0, v1, v2, a.w);
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
  for (int v = 0; v < 4; ++v) {
    float v0 = k[0][v], v1 = k[1][v], v2 = k[2][v];
    y_of(v0, v1, v2, mom ? m[0][v] : 0.f, mom ? m[1][v] : 0.f, mom ? m[2][v] : 0.f);
    R.y[0][v] = v0;
    R.y[1][v] = v1;
    R.y[2][v] = v2;
  }
  // halo columns: lane 0 -> column c0-1 (tile column 3), lane 31 -> c0+128 (tile column 132)
  const int hcol = lane == 31 ? 4 + 128 - (4 + lane * 4) : 3 - (4 + lane * 4);
  float h0 = qk[hcol], h1 = qk[TROWS * TBW + hcol], h2 = qk[2 * TROWS * TBW + hcol];
  float n0 = 0.f, n1 = 0.f, n2 = 0.f;
  if (mom) {
    n0 = qm[hcol];
    n1 = qm[TROWS * TBW + hcol];
    n2 = qm[2 * TROWS * TBW + hcol];
  }
  y_of(h0, h1, h2, n0, n1, n2);
  R.h[0] = h0;
  R.h[1] = h1;
  R.h[2] = h2;
  hx = xs[hcol];
}

template <class T, int V, bool TMA>
__global__ void __launch_bounds__((MTY + 2) * 32, 2) fgp3d_march_kernel(Fgp3Args<T> a, const __grid_constant__ Fgp3Maps maps) {
  using A = Ar<T>;
  constexpr int BW = 32 * V;
  // row exchange (vector-aligned rows; the band's right halo column apart)
  __shared__ __align__(16) T s_yy[2][MTY + 2][BW];
  __shared__ T s_yyh[2][MTY + 2];
  __shared__ __align__(16) T s_u[2][MTY + 2][BW];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = blockIdx.x * BW;
  const int i = blockIdx.y * MTY - 1 + w;
  int ks, ke;
  if (a.part == 0) {
    ks = blockIdx.z * a.zchunk;
    ke = min(a.D, ks + a.zchunk);
  } else if (a.part == 1) {
    ks = 1 + blockIdx.z * a.zchunk;
    ke = min(a.D - 1, ks + a.zchunk);
  } else {
    ks = blockIdx.z == 0 ? 0 : a.D - 1;
    ke = ks + 1;
    if (blockIdx.z == 1 && a.D == 1) return;
  }
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

  extern __shared__ __align__(128) unsigned char dyn_smem[];
  T* stage0 = reinterpret_cast<T*>(dyn_smem);
  constexpr int SW = 7 * BW;  // per-warp stage floats
  T* hs_all = stage0 + (size_t)2 * (MTY + 2) * SW;
  auto st_ptr = [&](int sidx) { return stage0 + (size_t)(sidx * (MTY + 2) + w) * SW; };
  auto hs_ptr = [&](int sidx) { return hs_all + (size_t)(sidx * (MTY + 2) + w) * 14; };
  // staging back ends: per-lane cp.async into per-warp rows, or (TMA) one
  // tensor-map tile per CTA and plane completing on a per-stage mbarrier
  __shared__ __align__(8) uint64_t s_tmb[2];
  unsigned tph = 0;  // TMA: parity of the next wait, per stage
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      mb_init(&s_tmb[0]);
      mb_init(&s_tmb[1]);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
  }
  auto t_stage = [&](int sidx) { return reinterpret_cast<float*>(dyn_smem) + sidx * TSTAGE; };
  auto stage_issue = [&](int kl, int sidx) {
    if constexpr (TMA) {
      if (threadIdx.x == 0)
        tma_issue_plane(a, maps, kl, mom, c0, blockIdx.y * MTY - 1, t_stage(sidx), &s_tmb[sidx]);
    } else {
      issue_plane<T, V>(a, kl, i, cl, lin, hc, hval, mom, lane, st_ptr(sidx), hs_ptr(sidx));
    }
  };
  auto stage_commit = [&]() {
    if constexpr (!TMA) cp_async_commit();
  };
  auto stage_wait = [&](int sidx, bool newer) {
    if constexpr (TMA) {
      mb_wait(&s_tmb[sidx], (tph >> sidx) & 1u);
      tph ^= 1u << sidx;
    } else {
      if (newer)
        cp_async_wait<1>();
      else
        cp_async_wait<0>();
      __syncwarp();
    }
  };
  auto stage_read = [&](int sidx, Row3<T, V>& R, T (&xr)[V], T& hxr) {
    if constexpr (TMA)
      tma_read_plane(a, mom, rp, w, lane, t_stage(sidx), R, xr, hxr);
    else
      read_plane<T, V>(a, mom, rp, lane, st_ptr(sidx), hs_ptr(sidx), R, xr, hxr);
  };

  Row3<T, V> C, N;
  T yzp[V], hyzp = T(0), xv[V], hx;
#pragma unroll
  for (int v = 0; v < V; ++v) yzp[v] = T(0);
  // prologue: y_z of plane ks-1 (synchronously), then planes ks and ks+1 in flight
  if (a.z0 + ks > 0) {
    T xd[V], hxd;
    stage_issue(ks - 1, 0);
    stage_commit();
    stage_wait(0, false);
    stage_read(0, N, xd, hxd);
#pragma unroll
    for (int v = 0; v < V; ++v) yzp[v] = N.y[0][v];
    hyzp = N.h[0];
    if constexpr (TMA)
      __syncthreads();  // every warp has read stage 0 before it is refilled
    else
      __syncwarp();
  }
  stage_issue(ks, 0);
  stage_commit();
  if (a.z0 + ks + 1 < a.Dg) stage_issue(ks + 1, 1);
  stage_commit();
  stage_wait(0, true);
  stage_read(0, C, xv, hx);
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
      // plane k+2 is read by this chunk only when k+1 < ke (no load may be
      // left in flight at exit)
      if (kg + 2 < a.Dg && k + 1 < ke) stage_issue(k + 2, sn ^ 1);
      stage_commit();
      stage_wait(sn, true);
      stage_read(sn, N, xv, hx);
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
        T* sd = k == 0 ? a.send_lo : (k == a.D - 1 ? a.send_hi : nullptr);
        if (sd) {
          const int64_t op = (int64_t)i * W + cl;
          stv<T, V>(sd + op, oz);
          stv<T, V>(sd + HW + op, oy);
          stv<T, V>(sd + 2 * HW + op, ox);
        }
        if (k == 0 && a.D == 1 && a.send_hi) {
          const int64_t op = (int64_t)i * W + cl;
          stv<T, V>(a.send_hi + op, oz);
          stv<T, V>(a.send_hi + HW + op, oy);
          stv<T, V>(a.send_hi + 2 * HW + op, ox);
        }
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

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
using EncodeTiled = PFN_cuTensorMapEncodeTiled_v12000;
EncodeTiled encode_fn() {
  static EncodeTiled fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
    (void)cudaGetLastError();
  }
  return fn;
}

// fp32 tile map: dims innermost first (W, H, ...), byte strides of dims 1.., box
bool encode_f32(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims,
                const cuuint64_t* strides, const cuuint32_t* box) {
  EncodeTiled fn = encode_fn();
  if (!fn || !base || reinterpret_cast<uintptr_t>(base) % 16) return false;
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank, const_cast<void*>(base), dims,
            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the TMA staging maps of one launch; false -> use the cp.async path
bool make_maps(const Fgp3Args<float>& a, Fgp3Maps& M) {
  const char* off = std::getenv("PSB_NO_TMA3D");
  if (off && off[0] == '1') return false;
  if (a.W % 4 != 0) return false;
  std::memset(&M, 0, sizeof(M));
  const cuuint64_t W = a.W, H = a.H, D = a.D, E = 4;
  const cuuint32_t bw = TBW, br = TROWS;
  {
    const cuuint64_t dims[4] = {W, H, D, 9}, str[3] = {W * E, W * H * E, W * H * D * E};
    const cuuint32_t box[4] = {bw, br, 1, 3};
    if (!encode_f32(&M.q, a.q, 4, dims, str, box)) return false;
  }
  {
    const cuuint64_t dims[3] = {W, H, D}, str[2] = {W * E, W * H * E};
    const cuuint32_t box[3] = {bw, br, 1};
    if (!encode_f32(&M.x, a.x, 3, dims, str, box)) return false;
  }
  const cuuint64_t hd[3] = {W, H, 3}, hs[2] = {W * E, W * H * E};
  const cuuint32_t hbx[3] = {bw, br, 3};
  if (a.hb_qk && (!encode_f32(&M.hb_qk, a.hb_qk, 3, hd, hs, hbx) ||
                  !encode_f32(&M.hb_qm, a.hb_qm, 3, hd, hs, hbx)))
    return false;
  if (a.ha_qk) {
    const cuuint64_t xd[2] = {W, H}, xs[1] = {W * E};
    const cuuint32_t xb[2] = {bw, br};
    if (!encode_f32(&M.ha_qk, a.ha_qk, 3, hd, hs, hbx) ||
        !encode_f32(&M.ha_qm, a.ha_qm, 3, hd, hs, hbx) || !encode_f32(&M.ha_x, a.ha_x, 2, xd, xs, xb))
      return false;
  }
  return true;
}

template <class T>
int launch3(const Fgp3Args<T>& a, cudaStream_t st) {
  constexpr int VMAX = 16 / sizeof(T);
  const int zc = a.zchunk;
  const int nz = a.part == 2 ? 2 : a.part == 1 ? std::max(1, (a.D - 2 + zc - 1) / zc)
                                              : (a.D + zc - 1) / zc;
  if (a.part == 1 && a.D <= 2) return PSB_OK;  // no interior planes
  const bool vec = (a.W % VMAX == 0) && (reinterpret_cast<uintptr_t>(a.x) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(a.q) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(a.send_lo) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(a.send_hi) % 16 == 0);
  Fgp3Maps maps;
  if constexpr (sizeof(T) == 4) {
    if (vec && make_maps(a, maps)) {
      const size_t sm = sizeof(float) * (size_t)2 * TSTAGE;
      PSB_CHECK(func_attr(fgp3d_march_kernel<T, VMAX, true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      dim3 grid((a.W + 32 * VMAX - 1) / (32 * VMAX), (a.H + MTY - 1) / MTY, nz);
      fgp3d_march_kernel<T, VMAX, true><<<grid, (MTY + 2) * 32, sm, st>>>(a, maps);
      PSB_LAUNCHED("fgp3d_march_tma");
      return PSB_OK;
    }
  }
  std::memset(&maps, 0, sizeof(maps));
  if (vec) {
    const size_t sm = march_smem<T, VMAX>();
    PSB_CHECK(func_attr(fgp3d_march_kernel<T, VMAX, false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    dim3 grid((a.W + 32 * VMAX - 1) / (32 * VMAX), (a.H + MTY - 1) / MTY, nz);
    fgp3d_march_kernel<T, VMAX, false><<<grid, (MTY + 2) * 32, sm, st>>>(a, maps);
  } else {
    const size_t sm = march_smem<T, 1>();
    PSB_CHECK(func_attr(fgp3d_march_kernel<T, 1, false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    dim3 grid((a.W + 31) / 32, (a.H + MTY - 1) / MTY, nz);
    fgp3d_march_kernel<T, 1, false><<<grid, (MTY + 2) * 32, sm, st>>>(a, maps);
  }
  PSB_LAUNCHED("fgp3d_march");
  return PSB_OK;
}

}  // namespace

int fgp3d_iter_part(int dtype, const void* x, void* q, int D, int H, int W, int z0, int Dg,
                    int it, double beta, double step, double weight, int rep, int nonneg,
                    const void* hb_qk, const void* hb_qm, const void* ha_qk, const void* ha_qm,
                    const void* ha_x, int zchunk, int part, void* send_lo, void* send_hi,
                    cudaStream_t st) {
  PSB_REQUIRE(D >= 1 && H >= 2 && W >= 2 && Dg >= 2, "fgp3d: need a 3-D grid with sides >= 2");
  PSB_REQUIRE(z0 >= 0 && z0 + D <= Dg, "fgp3d: slab outside the volume");
  PSB_REQUIRE(weight > 0, "tv_prox: weight must be positive");
  PSB_REQUIRE(part >= 0 && part <= 2, "fgp3d: part must be 0 (all), 1 (interior) or 2 (edges)");
  // the interior planes [1, D-1) never read a halo plane
  PSB_REQUIRE(part == 1 || z0 == 0 || (hb_qk && hb_qm),
              "fgp3d: slab above plane 0 needs the halo below");
  PSB_REQUIRE(part == 1 || z0 + D == Dg || (ha_qk && ha_qm && ha_x),
              "fgp3d: slab below the top needs the halo above");
  if (zchunk <= 0) {
    // enough CTAs for ~4 waves; long chunks amortise the two halo planes
    const int Dp = part == 1 ? std::max(1, D - 2) : D;
    const int64_t tiles = (int64_t)((W + 127) / 128) * ((H + MTY - 1) / MTY);
    const int64_t want = 32LL * sm_count();  // ~16 waves at 2 CTAs/SM: small tail
    int nz = (int)std::max<int64_t>(1, std::min<int64_t>(Dp, (want + tiles - 1) / tiles));
    zchunk = std::max(16, (Dp + nz - 1) / nz);
  }
  if (dtype == PSB_F32) {
    Fgp3Args<float> a{(const float*)x, (float*)q, D, H, W, z0, Dg, it, (float)beta, (float)step,
                      (float)weight, rep, nonneg, (const float*)hb_qk, (const float*)hb_qm,
                      (const float*)ha_qk, (const float*)ha_qm, (const float*)ha_x, zchunk,
                      part, (float*)send_lo, (float*)send_hi};
    return launch3(a, st);
  }
  if (dtype == PSB_F64) {
    Fgp3Args<double> a{(const double*)x, (double*)q, D, H, W, z0, Dg, it, beta, step, weight, rep,
                       nonneg, (const double*)hb_qk, (const double*)hb_qm, (const double*)ha_qk,
                       (const double*)ha_qm, (const double*)ha_x, zchunk, part,
                       (double*)send_lo, (double*)send_hi};
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
  return psb::fgp3d_iter_part(dtype, x, q, D, H, W, z0, Dg, it, beta_prev, step, weight,
                              reproject, nonneg, halo_below_qk, halo_below_qm, halo_above_qk,
                              halo_above_qm, halo_above_x, zchunk, 0, nullptr, nullptr,
                              psb::as_stream(stream));
}

int psb_fgp3d_iter_part(int dtype, const void* x, void* q, int D, int H, int W, int z0, int Dg,
                        int it, double beta_prev, double step, double weight, int reproject,
                        int nonneg, const void* halo_below_qk, const void* halo_below_qm,
                        const void* halo_above_qk, const void* halo_above_qm,
                        const void* halo_above_x, int zchunk, int part, void* send_lo,
                        void* send_hi, void* stream) {
  return psb::fgp3d_iter_part(dtype, x, q, D, H, W, z0, Dg, it, beta_prev, step, weight,
                              reproject, nonneg, halo_below_qk, halo_below_qm, halo_above_qk,
                              halo_above_qm, halo_above_x, zchunk, part, send_lo, send_hi,
                              psb::as_stream(stream));
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

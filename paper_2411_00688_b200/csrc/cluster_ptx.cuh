// Cluster / DSMEM / mbarrier PTX helpers shared by the cluster-resident run
// kernels (fgp_cluster.cu: 16 CTAs x 4 rows per thread, fgp_cluster8.cu:
// 8 CTAs x 8 rows per thread).
#pragma once

#include <type_traits>

#include "common.cuh"

namespace psb {

#ifdef PSB_DBG_PHASES  // timing experiment: per-phase ns of one thread per role (cluster 0)
static __device__ unsigned long long g_phase_ns[16];  // (one copy per translation unit)
#define PHASE_MARK(v) uint64_t v = gtimer_ns()
#define PHASE_ADD(slot, t0, t1)                                                 \
  do {                                                                         \
    if (blockIdx.x == 0 && (tid == 0 || tid == 128 || tid == 384))             \
      atomicAdd(&g_phase_ns[(slot) * 4 + (tid == 0 ? 0 : tid == 128 ? 1 : 2)], \
                (unsigned long long)((t1) - (t0)));                            \
  } while (0)
#else
#define PHASE_MARK(v)
#define PHASE_ADD(slot, t0, t1)
#endif

template <class TO>
__device__ __forceinline__ TO skip_update(TO xo, TO bo, TO ho, TO g) {
  using A = Ar<TO>;
  return A::add(A::sub(xo, A::mul(g, A::sub(xo, bo))), A::mul(g, ho));  // skip.py:68
}

// Packed fp32 pairs as 64-bit registers (fma/add/mul.rn.f32x2 operate on .b64):
// lo / hi = the two rows of a row pair of a column strip.  No mul is ever followed by
// an add of its result here (ptxas would contract that pair into an FFMA2).
using P2 = unsigned long long;
__device__ __forceinline__ P2 pk(float lo, float hi) {
  P2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float plo(P2 v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return lo;
}
__device__ __forceinline__ float phi(P2 v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return hi;
}
__device__ __forceinline__ P2 pfma(P2 a, P2 b, P2 c) {
  P2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ P2 padd(P2 a, P2 b) {
  P2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ P2 pmul(P2 a, P2 b) {
  P2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// 32-bit shared::cluster address of `p` in CTA `rank` of this cluster, and a load from it
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, int rank) {
  uint32_t local = (uint32_t)__cvta_generic_to_shared(p), remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank));
  return remote;
}
template <class T>
__device__ __forceinline__ T dsmem_ld(uint32_t addr) {
  if constexpr (std::is_same<T, int>::value) {
    int v;
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
  } else if constexpr (sizeof(T) == 8) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
    return v;
  } else {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
  }
}

// ---- point-to-point halo rows: st.async into the neighbour's shared memory,
// completion counted in bytes on the neighbour's mbarrier (no cluster-wide
// barrier, no memory fence on the critical path) -----------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(m)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(m)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(m)),
      "r"(parity)
      : "memory");
}
#ifdef PSB_DBG_NOGSYNC  // timing experiment only: row-group waits skipped (results invalid)
#define GWAIT(m, ph) ((void)0)
#else
#define GWAIT(m, ph) mbar_wait(m, ph)
#endif
__device__ __forceinline__ void mbar_arrive(uint64_t* m) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void st_async_f32(uint32_t raddr, float v, uint32_t rmbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];\n" ::"r"(raddr),
               "r"(__float_as_uint(v)), "r"(rmbar)
               : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t raddr, float v0, float v1, uint32_t rmbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];\n" ::"r"(raddr),
               "r"(__float_as_uint(v0)), "r"(__float_as_uint(v1)), "r"(rmbar)
               : "memory");
}

__device__ __forceinline__ void st_async_v4(uint32_t raddr, float v0, float v1, float v2, float v3,
                                            uint32_t rmbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];\n" ::"r"(raddr),
               "r"(__float_as_uint(v0)), "r"(__float_as_uint(v1)), "r"(__float_as_uint(v2)),
               "r"(__float_as_uint(v3)), "r"(rmbar)
               : "memory");
}

// MUFU.RSQ without the denormal rescaling rsqrtf() wraps around it (|a|^2 of a
// dual vector is never denormal in a way that matters: the ball test is
// min(1, w / |a|)); 1 instruction instead of ~6 per pixel.
__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

}  // namespace psb

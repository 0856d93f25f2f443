// Cluster-resident ProxSkip runs for 256 x 256 problems, fp32 outer state
// (BASELINE config 4), on 8-CTA clusters: the same run segment, schedule and
// per-pixel arithmetic as fgp_cluster.cu (skip.py:46-79, tv.py:53-89 -- see
// the header comment there), with twice the pixels per SM.
//
//   cluster = 8 CTAs x 32 rows; CTA = 512 threads = 4 row groups of 8 rows;
//   thread  = 2 columns x 8 rows, held as row pairs (t, t + 4) in float2
//             registers (packed FFMA2 / FADD2 / FMUL2 on aligned pairs; only
//             one pair per column strip end is built from two halves).
//
// 16 pixels per thread do not fit the register file with z, q_k and q_{k-1}
// all resident (80 state registers + temporaries > 128), so only q_k lives in
// registers: the prox input z and the previous dual iterate q_{k-1} are
// thread-private columns of the SM's TENSOR MEMORY (tcgen05.ld / .st, below),
// read once and written once per inner iteration.  What this buys over the
// 16-CTA form: every synchronisation of the inner loop (warp-edge columns,
// row-group rows, the DSMEM halo round trip) is paid once per 16 pixels of a
// thread instead of once per 8, eight independent pair chains per thread
// instead of four, and 8-CTA clusters tile 120 of the 148 SMs (16-CTA: 112).
// The inner loop is compiled once per row group (exchange addresses become
// immediates) on 64-bit register pairs (P2, cluster_ptx.cuh).
//
// Every pixel's arithmetic is the scalar FGP step of the other kernels
// (each f32x2 lane an IEEE fp32 op), so results are bit-identical to
// fgp_cluster_run_kernel, fgp_sm_run_kernel and the streaming path.
#include <cooperative_groups.h>

#include <type_traits>

#include "cluster_ptx.cuh"

namespace cg = cooperative_groups;

namespace psb {

namespace {

constexpr int CW = 256;                  // image width
constexpr int CRPT = 8;                  // rows per thread
constexpr int NP = CRPT / 2;             // row pairs (t, t + NP) per column strip
constexpr int CTPR = CW / 2;             // threads per row group (2 columns each)
constexpr int CRG = 4;                   // row groups per CTA
constexpr int CCL = 8;                   // CTAs per cluster
constexpr int SR = CRG * CRPT;           // rows per CTA (32)
constexpr int CH = CCL * SR;             // image height = 256
constexpr int CTHREADS = CTPR * CRG;     // 512
constexpr int CWARPS_ROW = CTPR / 32;    // 4 warps across a row group
constexpr int kMaxBetas = 1024;
static_assert(CH == 256 && CTHREADS == 512, "256 x 256 problems on 8 x 512 threads");

struct Run8Args {
  float* x;
  const float* b;
  float* h;
  float* q;  // warm-start slot 0 of problem p: q + p*qps (channel stride CH*CW)
  int64_t qps;
  WorkQueue wq;
  const int32_t* ev_off;  // [n + 1]: problem p's coin-fired iterations ev_k[ev_off[p] ..]
  const int32_t* ev_k;    // ascending, 0 .. K-1 (this run segment)
  const uint8_t* rep;     // [n]: re-project the warm start at the first prox call (tv.py:68-69)
  int K;
  int n_inner;
  int accelerated;
  float weight;
  float gamma, hc, pg;
  float step;
  int32_t* bad;        // [n]: first non-finite iteration (atomicMin)
  const float* betas;  // device table beta[0..n_inner-1]
  ChunkSync cs;
};


// ---- tensor memory as a thread-private register-spill space -------------------
// The SM's 256 KB of TMEM (512 columns x 128 lanes x 32 bit) is idle in a
// kernel without tcgen05.mma.  tcgen05.ld / .st with the .32x32b shape move
// N consecutive columns of ONE lane per thread -- lane 32 (warp % 4) + laneid --
// so the four warps that share a lane quarter split the 512 columns: every
// thread owns 128 private words, reached by one instruction per 16 / 32
// registers, on a datapath of its own (measured, tools/micro/tmem_bw.cu:
// 247 B/cycle/SM loads against 128 B/cycle/SM for shared memory, and the
// shared-memory pipe stays free for the shuffles and the edge exchange).
// wait::ld names the loaded registers as in/out operands: their consumers must
// not be scheduled above the wait (a volatile asm orders only other volatile
// asms and memory accesses, not register arithmetic)
__device__ __forceinline__ void tm_wait_ld(uint32_t (&v)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                 "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]),
                 "+r"(v[15]):);
}
__device__ __forceinline__ void tm_wait_ld(uint32_t (&v)[16], uint32_t (&w)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                 "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]),
                 "+r"(v[15]), "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]),
                 "+r"(w[6]), "+r"(w[7]), "+r"(w[8]), "+r"(w[9]), "+r"(w[10]), "+r"(w[11]), "+r"(w[12]),
                 "+r"(w[13]), "+r"(w[14]), "+r"(w[15]):);
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::); }
__device__ __forceinline__ void tm_ld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}
__device__ __forceinline__ void tm_st16(uint32_t addr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(addr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}
// one packed pair (a 64-bit register pair as it is: no gathering moves)
__device__ __forceinline__ void tm_st2(uint32_t addr, P2 v) {
  uint32_t a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(a), "=r"(b) : "l"(v));
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};\n" ::"r"(addr), "r"(a), "r"(b));
}
__device__ __forceinline__ void p2_split(P2 v, uint32_t& lo, uint32_t& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(v));
}
__device__ __forceinline__ P2 p2_join(uint32_t lo, uint32_t hi) {
  P2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}
// thread-private TMEM columns: [0,32) q_{k-1}: words 4 (k NP + P) + {0,1} the
// y pair, + {2,3} the x pair of column k, pair P (one 2-word store per register
// pair as it is, two 16-word loads); [32,48) z: words 4 P + 2 k + {0,1}
constexpr uint32_t kTmQ = 0, kTmZ = 32;

// row-group mbarriers addressed as one base register + immediate byte offset
template <int OFF>
__device__ __forceinline__ void gb_arrive(uint32_t base) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0+%1];\n" ::"r"(base), "n"(OFF) : "memory");
}
template <int OFF>
__device__ __forceinline__ void gb_wait(uint32_t base, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0+%1], %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(base),
      "n"(OFF), "r"(parity)
      : "memory");
}
#ifdef PSB_DBG_NOGSYNC
#define GBWAIT(off, ph) ((void)0)
#else
#define GBWAIT(off, ph) gb_wait<(off)>(gb, ph)
#endif

// row t of a column strip held as pairs (t, t + NP)
__device__ __forceinline__ float& rowref(float2 (&v)[NP], int t) {
  return t < NP ? v[t].x : v[t - NP].y;
}

constexpr size_t kStageBytes = (size_t)3 * SR * CW * sizeof(float);           // x, b, h rows
constexpr size_t kDynBytes = kStageBytes;

template <bool NONNEG>
__global__ void __launch_bounds__(CTHREADS, 1) fgp_cluster8_run_kernel(Run8Args a) {
  using F = Ar<float>;
  cg::cluster_group cluster = cg::this_cluster();
  const int cr = (int)cluster.block_rank();
  const int tid = threadIdx.x;
  const int jt = tid % CTPR, rg = tid / CTPR;  // column pair, row group
  const int j0 = 2 * jt;                        // columns j0, j0 + 1
  // the warp index broadcast from lane 0: the compiler then knows it is
  // warp-uniform and keeps what derives from it (tensor-memory addresses,
  // warp-edge slots) on the uniform datapath
  const int warp_u = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int lane = tid & 31, wc = warp_u & (CWARPS_ROW - 1);
  const int row0 = cr * SR + rg * CRPT;
  const bool rg_top = rg == 0, rg_bot = rg == CRG - 1;
  const bool has_up = cr > 0, has_dn = cr < CCL - 1;
  constexpr int64_t HW = (int64_t)CH * CW;

  // halo rows received from the neighbour CTAs, double-buffered by round parity
  __shared__ __align__(16) float rx_dn[2][CW][2];  // CTA below's first row of y (y, x)
  __shared__ __align__(8) float rx_up[2][CW];      // CTA above's last row of y (y)
  __shared__ __align__(8) uint64_t mb_dn[2], mb_up[2];
  __shared__ __align__(16) float rx_z[CW];  // CTA below's first row of z, once per prox call
  __shared__ __align__(8) uint64_t mb_z;
  // row-group mbarriers, one phase per inner iteration (see fgp_cluster.cu)
  // (one array: every barrier is the base register plus an immediate)
  __shared__ __align__(8) uint64_t gbar[4 * CRG];
  constexpr int kE1 = 0, kE2 = CRG, kYY = 2 * CRG, kU = 3 * CRG;  // + row group
  __shared__ __align__(8) float s_rg_yy[CRG][CW];  // each row group's last-row y_y
  __shared__ __align__(8) float s_rg_u[CRG][CW];   // each row group's first-row u
  // warp-edge columns as row pairs: s_edge_yx[rg][P][w + 1] = last column of
  // warp w (slot 0 stays zero), s_edge_u[rg][P][w] = first column of warp w
  __shared__ __align__(16) P2 s_edge_yx[CRG][NP][CWARPS_ROW + 1];
  __shared__ __align__(16) P2 s_edge_u[CRG][NP][CWARPS_ROW];
  // the finalize's own exchange rows (q_n's last row per group, q_n's warp-edge
  // columns): separate from the inner loop's, so no barrier is needed between
  // the last inner iteration and these writes
  __shared__ __align__(8) float s_fin_yy[CRG][CW];
  __shared__ __align__(16) P2 s_fin_edge[CRG][NP][CWARPS_ROW + 1];
  __shared__ float s_beta[kMaxBetas];
  __shared__ int s_next[2];
  __shared__ uint32_t s_tm_base;
  extern __shared__ __align__(16) unsigned char dyn_raw[];
  float* sx = reinterpret_cast<float*>(dyn_raw);  // [SR][CW]
  float* sb = sx + SR * CW;
  float* sh = sb + SR * CW;

  const float g = a.gamma;
  const float w = a.weight;
  constexpr bool nonneg = NONNEG;
  for (int e = tid; e < a.n_inner && e < kMaxBetas; e += CTHREADS) s_beta[e] = a.betas[e];
  if (tid < CRG * NP) s_edge_yx[tid / NP][tid % NP][0] = s_fin_edge[tid / NP][tid % NP][0] = pk(0.f, 0.f);
  if (tid == 0) {
    mbar_init(&mb_dn[0], 1);
    mbar_init(&mb_dn[1], 1);
    mbar_init(&mb_up[0], 1);
    mbar_init(&mb_up[1], 1);
    mbar_init(&mb_z, 1);
    for (int gi = 0; gi < CRG; ++gi) {
      mbar_init(&gbar[kE1 + gi], CTPR);
      mbar_init(&gbar[kE2 + gi], CTPR);
      mbar_init(&gbar[kYY + gi], CTPR);
      mbar_init(&gbar[kU + gi], CTPR);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (tid < 32) {  // warp 0 takes the SM's whole tensor memory (one CTA per SM)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        smem_u32(&s_tm_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // this thread's 128 columns of its lane (bits 31:16 lane, 15:0 column)
  const uint32_t tm = s_tm_base + ((uint32_t)((warp_u & 3) * 32) << 16) + (uint32_t)((warp_u >> 2) * 128);
  // every CTA of this grid is resident: the SM-worker kernel (a programmatic
  // dependent) may now be placed on the SMs the clusters left
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  cluster_arrive();  // every CTA's mbarriers exist before anyone pushes
  cluster_wait();
  constexpr unsigned BYTES_DN = CW * 2 * 4, BYTES_UP = CW * 4;
  const uint32_t up_rx_remote = dsmem_addr(&rx_dn[0][0][0], has_up ? cr - 1 : cr);  // my top row -> CTA above
  const uint32_t up_mb_remote = dsmem_addr(&mb_dn[0], has_up ? cr - 1 : cr);
  const uint32_t dn_rx_remote = dsmem_addr(&rx_up[0][0], has_dn ? cr + 1 : cr);  // my bottom row -> CTA below
  const uint32_t dn_mb_remote = dsmem_addr(&mb_up[0], has_dn ? cr + 1 : cr);
  const uint32_t z_rx_remote = dsmem_addr(&rx_z[0], has_up ? cr - 1 : cr);
  const uint32_t z_mb_remote = dsmem_addr(&mb_z, has_up ? cr - 1 : cr);
  const uint32_t gb = smem_u32(&gbar[0]);
  unsigned zph = 0;    // prox calls so far (mb_z phases)
  unsigned round = 0;  // halo rounds so far (round r lands in buffer r & 1)
  unsigned gph = 0;    // inner iterations so far (row-group mbarrier phases)
  const bool arm = lane == 0 && wc == 0;
  auto push_up = [&](float ty0, float tx0, float ty1, float tx1) {  // top group, has_up
#ifdef PSB_DBG_NOHALO
    return;
#endif
    const unsigned b = round & 1;
    st_async_v4(up_rx_remote + 4u * (b * CW * 2 + j0 * 2), ty0, tx0, ty1, tx1, up_mb_remote + 8u * b);
  };
  auto push_dn = [&](float by0, float by1) {  // bottom group, has_dn
#ifdef PSB_DBG_NOHALO
    return;
#endif
    const unsigned b = round & 1;
    st_async_v2(dn_rx_remote + 4u * (b * CW + j0), by0, by1, dn_mb_remote + 8u * b);
  };
  auto recv_up = [&](unsigned r) {  // top group, has_up
    const unsigned b = r & 1, ph = (r >> 1) & 1;
#ifdef PSB_DBG_NOHALO
    return b;
#endif
    if (arm) mbar_expect_tx(&mb_up[b], BYTES_UP);
    mbar_wait(&mb_up[b], ph);
    return b;
  };
  auto recv_dn = [&](unsigned r) {  // bottom group, has_dn
    const unsigned b = r & 1, ph = (r >> 1) & 1;
#ifdef PSB_DBG_NOHALO
    return b;
#endif
    if (arm) mbar_expect_tx(&mb_dn[b], BYTES_DN);
    mbar_wait(&mb_dn[b], ph);
    return b;
  };
  const bool right_fetch = lane == 31 && wc < CWARPS_ROW - 1;
  const bool last_col = lane == 31 && wc == CWARPS_ROW - 1;  // owns global column W-1

  const uint32_t next_remote = dsmem_addr(&s_next[0], 0);
  uint64_t t_claim = 0;
  for (unsigned pj = 0;; ++pj) {
    // rank 0 claims the next problem; everyone reads it after the barrier
    if (cr == 0 && tid == 0) s_next[pj & 1] = wq_claim(a.wq);
    cluster_arrive();
    cluster_wait();
    const int pos = dsmem_ld<int>(next_remote + 4u * (pj & 1));
    if (pos < 0) break;
    const int p = a.wq.order[pos];
    float* xp = a.x + (int64_t)p * HW;
    const float* bp = a.b + (int64_t)p * HW;
    float* hp = a.h + (int64_t)p * HW;
    float* q0 = a.q + (int64_t)p * a.qps;
    const int e0 = a.ev_off[p], e1 = a.ev_off[p + 1];
    const bool rep = a.rep[p];
    if (a.cs.ready) {  // this problem's input chunk has arrived
      if (tid == 0) chunk_wait(a.cs, p);
      __syncthreads();
    }
    if (cr == 0 && tid == 0) t_claim = gtimer_ns();
    // stage this CTA's rows of x, b, h (each thread its own elements) and the
    // warm-start duals; a streamed run starts cold (x = h = 0, q_warm = 0
    // implied, device buffers uninitialised)
    const bool cold = a.cs.ready != nullptr;
    float2 qky[2][NP], qkx[2][NP];  // q_k: per column k, row pairs
    {
      const bool ldq = !(cold || e1 == e0);
#pragma unroll
      for (int t = 0; t < CRPT; ++t) {
        const int lr = rg * CRPT + t;
        const int64_t o = (int64_t)(row0 + t) * CW + j0;
        const float2 zero2 = make_float2(0.f, 0.f);
        const float2 xv = cold ? zero2 : *reinterpret_cast<const float2*>(xp + o);
        const float2 bv = *reinterpret_cast<const float2*>(bp + o);
        const float2 hv = cold ? zero2 : *reinterpret_cast<const float2*>(hp + o);
        const float2 qy = ldq ? *reinterpret_cast<const float2*>(q0 + o) : zero2;
        const float2 qx = ldq ? *reinterpret_cast<const float2*>(q0 + HW + o) : zero2;
        *reinterpret_cast<float2*>(&sx[lr * CW + j0]) = xv;
        *reinterpret_cast<float2*>(&sb[lr * CW + j0]) = bv;
        *reinterpret_cast<float2*>(&sh[lr * CW + j0]) = hv;
        rowref(qky[0], t) = qy.x;
        rowref(qky[1], t) = qy.y;
        rowref(qkx[0], t) = qx.x;
        rowref(qkx[1], t) = qx.y;
      }
    }
    int kbad = 0x7fffffff;
    int kprev = -1;
    for (int e = e0; e < e1; ++e) {
      const int kk = a.ev_k[e];
      const int m = kk - kprev - 1;  // skip iterations kprev+1 .. kk-1 before this prox call
      const int kf = kprev + 1;
      // (no barrier here: x, b, h and the spill columns are thread-private, the
      // inner loop's exchange buffers were last read before the previous
      // call's finalize barrier, and rx_z is rewritten only after this CTA's
      // final-round push of that call)
      PHASE_MARK(ph_a);
      // ---- prologue: skips, prox input, warm start ----------------------------
      {
        // this thread's 2 columns x CRPT rows of x, b, h
        float2 xv[CRPT], bv[CRPT], hv[CRPT];
#pragma unroll
        for (int t = 0; t < CRPT; ++t) {
          const int sj = (rg * CRPT + t) * CW + j0;
          xv[t] = *reinterpret_cast<const float2*>(&sx[sj]);
          bv[t] = *reinterpret_cast<const float2*>(&sb[sj]);
          hv[t] = *reinterpret_cast<const float2*>(&sh[sj]);
        }
        if (m > 0) {
          // the m skipped iterations (skip.py:68) of all 16 pixels side by side;
          // the update is a fixed map of x, so once no pixel changes any more
          // the remaining steps change nothing either (skip_chain_px, common.cuh)
          for (int sk = 0; sk < m; ++sk) {
            bool changed = false;
#pragma unroll
            for (int t = 0; t < CRPT; ++t) {
              const float nx = skip_step(xv[t].x, bv[t].x, hv[t].x, g);
              const float ny = skip_step(xv[t].y, bv[t].y, hv[t].y, g);
              changed |= !same_bits(nx, xv[t].x) | !same_bits(ny, xv[t].y);
              xv[t] = make_float2(nx, ny);
            }
            if (!changed) break;
          }
          bool fin = true;
#pragma unroll
          for (int t = 0; t < CRPT; ++t) fin &= finite(xv[t].x) & finite(xv[t].y);
          if (!fin) {  // slow path: the first non-finite step, from the x still in shared memory
#pragma unroll
            for (int t = 0; t < CRPT; ++t) {
              const int sj = (rg * CRPT + t) * CW + j0;
              (void)skip_chain_px(sx[sj], bv[t].x, hv[t].x, g, m, kf, &kbad);
              (void)skip_chain_px(sx[sj + 1], bv[t].y, hv[t].y, g, m, kf, &kbad);
            }
          }
#pragma unroll
          for (int t = 0; t < CRPT; ++t)
            *reinterpret_cast<float2*>(&sx[(rg * CRPT + t) * CW + j0]) = xv[t];
        }
        float2 z[2][NP];
#pragma unroll
        for (int t = 0; t < CRPT; ++t) {
          rowref(z[0], t) = F::add(F::sub(xv[t].x, F::mul(g, F::sub(xv[t].x, bv[t].x))), F::mul(a.hc, hv[t].x));
          rowref(z[1], t) = F::add(F::sub(xv[t].y, F::mul(g, F::sub(xv[t].y, bv[t].y))), F::mul(a.hc, hv[t].y));
        }
        // my first row of z goes to the CTA above (its bottom group computes u
        // of that row itself); the row from the CTA below is awaited in the
        // first inner iteration, where it is first used
        if (rg_top && has_up) st_async_v2(z_rx_remote + 4u * j0, z[0][0].x, z[1][0].x, z_mb_remote);
        if (e == e0) {  // warm start (staged above), re-projected if the weight changed
#pragma unroll
          for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int t = 0; t < CRPT; ++t) {
              float vy = rowref(qky[k], t), vx = rowref(qkx[k], t);
              if (rep) {
                const float sc = F::ball_scale(vy, vx, w);
                vy *= sc;
                vx *= sc;
              }
              // q_y on the last row and q_x on the last column stay 0
              // (operators.py:66-70): zero padding instead of boundary masks
              if (row0 + t == CH - 1) vy = 0.f;
              if (j0 + k == CW - 1) vx = 0.f;
              rowref(qky[k], t) = vy;
              rowref(qkx[k], t) = vx;
            }
        }
        {
          uint32_t zw[16];
#pragma unroll
          for (int P = 0; P < NP; ++P) {
            zw[4 * P + 0] = __float_as_uint(z[0][P].x), zw[4 * P + 1] = __float_as_uint(z[0][P].y);
            zw[4 * P + 2] = __float_as_uint(z[1][P].x), zw[4 * P + 3] = __float_as_uint(z[1][P].y);
          }
          tm_st16(tm + kTmZ, zw);
          tm_wait_st();
        }
      }
      float z_ex[2] = {0.f, 0.f};  // the CTA-below's first row of z (bottom group, first iteration)
      const unsigned zpar = zph & 1u;
      ++zph;
      // After the first call of a problem the warm start's boundary rows are
      // the previous call's final round (no exchange); halo rows travel as
      // momentum iterates y (fgp_cluster.cu)
      const bool reuse = e > e0;
      const unsigned round0 = reuse ? round - 1 : round;  // this call's warm-start round
      auto y0_of = [](float q) { return fmaf(0.f, fmaf(q, -1.f, q), q); };
      if (!reuse) {
#ifndef PSB_DBG_NOHALO
        if (rg_top && has_up)
          push_up(y0_of(qky[0][0].x), y0_of(qkx[0][0].x), y0_of(qky[1][0].x), y0_of(qkx[1][0].x));
        if (rg_bot && has_dn) push_dn(y0_of(qky[0][NP - 1].y), y0_of(qky[1][NP - 1].y));
#endif
        ++round;
      }

      // One inner iteration: y from (q_k registers, q_{k-1} tensor memory),
      // q_k -> tensor memory (the next q_{k-1}), the new iterate -> q_k
      // registers.  Row group 0 is the top group (halo from the CTA above),
      // CRG - 1 the bottom group, the others carry no halo code.
      auto run_inner = [&](auto rg_tag) {
        // one copy per row group: the group index is a compile-time constant,
        // so every shared-memory exchange address below is the CTA's window
        // base plus an immediate
        constexpr int RG = decltype(rg_tag)::value;
        constexpr bool TOP = RG == 0, BOT = RG == CRG - 1;
        // the loop-carried iterate as 64-bit register pairs (P2), so the values
        // cross the back-edge as pairs and need no re-pairing moves
        P2 QY[2][NP], QX[2][NP];
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
          for (int P = 0; P < NP; ++P) {
            QY[k][P] = pk(qky[k][P].x, qky[k][P].y);
            QX[k][P] = pk(qkx[k][P].x, qkx[k][P].y);
          }
        const P2 m1 = pk(-1.f, -1.f);
        const float wr = w * kBallShrink;
        const P2 st2 = pk(a.step, a.step), w2 = pk(wr, wr);
        auto inner = [&](int it, auto first_tag) {
          constexpr bool FIRST = decltype(first_tag)::value;
          const unsigned ph = gph & 1u;
          const float beta = (a.accelerated && it > 0) ? s_beta[it - 1] : 0.f;
          const P2 b2 = pk(beta, beta);
          P2 yy[2][NP], yx[2][NP];
          // q_{k-1} from tensor memory (two 16-word loads), y, then q_k goes
          // where q_{k-1} was (the previous iteration's stores have landed:
          // wait::st below, before this load)
          {
            uint32_t m0[16], m1w[16];  // column 0 / column 1: 4 P + {0,1} y pair, + {2,3} x pair
            if constexpr (!FIRST) {
              tm_ld16(tm + kTmQ, m0);
              tm_ld16(tm + kTmQ + 16, m1w);
              tm_wait_ld(m0, m1w);
            }
#pragma unroll
            for (int k = 0; k < 2; ++k)
#pragma unroll
              for (int P = 0; P < NP; ++P) {
                P2 vy = QY[k][P], vx = QX[k][P];  // (the momentum restarts with every call)
                if constexpr (!FIRST) {
                  const uint32_t(&mw)[16] = k == 0 ? m0 : m1w;
                  vy = p2_join(mw[4 * P], mw[4 * P + 1]);
                  vx = p2_join(mw[4 * P + 2], mw[4 * P + 3]);
                }
                yy[k][P] = pfma(b2, pfma(vy, m1, QY[k][P]), QY[k][P]);
                yx[k][P] = pfma(b2, pfma(vx, m1, QX[k][P]), QX[k][P]);
              }
            // q_k becomes q_{k-1} (its halo entries for the y pushed below are kept)
#pragma unroll
            for (int k = 0; k < 2; ++k)
#pragma unroll
              for (int P = 0; P < NP; ++P) {
                tm_st2(tm + kTmQ + 4 * (k * NP + P), QY[k][P]);
                tm_st2(tm + kTmQ + 4 * (k * NP + P) + 2, QX[k][P]);
              }
          }
          uint32_t zw[16];
          tm_ld16(tm + kTmZ, zw);  // (waited for before the first u below)
          float old_e[4];
          if constexpr (TOP) {
            old_e[0] = plo(QY[0][0]), old_e[1] = plo(QX[0][0]), old_e[2] = plo(QY[1][0]), old_e[3] = plo(QX[1][0]);
          }
          if constexpr (BOT) {
            old_e[0] = phi(QY[0][NP - 1]), old_e[1] = phi(QY[1][NP - 1]);
          }
          if constexpr (!BOT) {  // last-row y_y for the group below
            *reinterpret_cast<float2*>(&s_rg_yy[RG][j0]) = make_float2(phi(yy[0][NP - 1]), phi(yy[1][NP - 1]));
            gb_arrive<8 * (kYY + RG)>(gb);
          }
          if (lane == 31) {
#pragma unroll
            for (int P = 0; P < NP; ++P) s_edge_yx[RG][P][wc + 1] = yx[1][P];
          }
          gb_arrive<8 * (kE1 + RG)>(gb);
          float2 yyA = make_float2(0.f, 0.f);  // TOP: y row above (zeros at row 0)
          float ex_y[2] = {0.f, 0.f}, ex_x[2] = {0.f, 0.f}, ledge_x = 0.f;  // BOT: row below
          if constexpr (TOP) {
            if (has_up) {
              const bool warm = FIRST && reuse;  // (already received: the previous call's final round)
              const unsigned par = warm ? (round0 & 1u) : recv_up(round0 + it);
              yyA = *reinterpret_cast<const float2*>(&rx_up[par][j0]);
              if (warm) yyA = make_float2(y0_of(yyA.x), y0_of(yyA.y));
            }
          }
          if constexpr (BOT) {
            if (has_dn) {
              const bool warm = FIRST && reuse;
              const unsigned par = warm ? (round0 & 1u) : recv_dn(round0 + it);
              const float4 v = *reinterpret_cast<const float4*>(&rx_dn[par][j0][0]);
              ex_y[0] = v.x, ex_x[0] = v.y, ex_y[1] = v.z, ex_x[1] = v.w;
              if (j0 > 0) ledge_x = rx_dn[par][j0 - 1][1];
              if (warm) {
                ex_y[0] = y0_of(ex_y[0]), ex_x[0] = y0_of(ex_x[0]);
                ex_y[1] = y0_of(ex_y[1]), ex_x[1] = y0_of(ex_x[1]);
                ledge_x = y0_of(ledge_x);
              }
            }
          }
          GBWAIT(8 * (kE1 + RG), ph);
          tm_wait_ld(zw);  // z
          // left neighbours of column 0: shuffles inside the warp, the warp to
          // the left's last column from shared memory (zeros left of column 0)
          P2 left[NP];
#pragma unroll
          for (int P = 0; P < NP; ++P)
            left[P] = pk(__shfl_up_sync(0xffffffffu, plo(yx[1][P]), 1),
                         __shfl_up_sync(0xffffffffu, phi(yx[1][P]), 1));
          if (lane == 0) {
#pragma unroll
            for (int P = 0; P < NP; ++P) left[P] = s_edge_yx[RG][P][wc];
          }
          float yy_above[2] = {yyA.x, yyA.y};
          P2 u[2][NP];
          // ((0 + yy) - yy_up) + yx - yx_left, boundary terms zero-padded; u = z + d
          auto u_pairs = [&](int P) {  // both columns of pair P
            const ulonglong2 zv = make_ulonglong2(p2_join(zw[4 * P], zw[4 * P + 1]),
                                                  p2_join(zw[4 * P + 2], zw[4 * P + 3]));
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const P2 ab2 = P == 0 ? pk(yy_above[k], plo(yy[k][NP - 1])) : yy[k][P > 0 ? P - 1 : 0];
              const P2 l2 = k == 0 ? left[P] : yx[0][P];
              const P2 d1 = padd(pfma(ab2, m1, yy[k][P]), yx[k][P]);
              const P2 d2 = pfma(l2, m1, d1);
              const P2 v = padd(k == 0 ? zv.x : zv.y, d2);
              u[k][P] = nonneg ? pk(fmaxf(plo(v), 0.f), fmaxf(phi(v), 0.f)) : v;
            }
          };
          if constexpr (BOT) {  // pairs 1.. need no row of another group
#pragma unroll
            for (int P = 1; P < NP; ++P) u_pairs(P);
          }
          if constexpr (!TOP) {
            GBWAIT(8 * (kYY + RG - 1), ph);
            const float2 ya2 = *reinterpret_cast<const float2*>(&s_rg_yy[RG - 1][j0]);
            yy_above[0] = ya2.x;
            yy_above[1] = ya2.y;
          }
          u_pairs(0);
          if constexpr (!BOT) {
#pragma unroll
            for (int P = 1; P < NP; ++P) u_pairs(P);
          }
          float u_below[2] = {0.f, 0.f};
          if constexpr (BOT && FIRST) {
            if (has_dn) {  // the z row pushed by the CTA below in its prologue
              if (arm) mbar_expect_tx(&mb_z, CW * 4);
              mbar_wait(&mb_z, zpar);
              const float2 zr = *reinterpret_cast<const float2*>(&rx_z[j0]);
              z_ex[0] = zr.x;
              z_ex[1] = zr.y;
            }
          }
          if constexpr (BOT) {
            if (has_dn) {  // u of the CTA-below's first row, from its y row
#pragma unroll
              for (int k = 0; k < 2; ++k) {
                const float d = ((ex_y[k] - phi(yy[k][NP - 1])) + ex_x[k]) - (k == 0 ? ledge_x : ex_x[0]);
                const float v = z_ex[k] + d;
                u_below[k] = nonneg ? fmaxf(v, 0.f) : v;
              }
            } else {  // the global last row: gy = 0 (below := u)
              u_below[0] = phi(u[0][NP - 1]);
              u_below[1] = phi(u[1][NP - 1]);
            }
          }
          if constexpr (!TOP) {  // first-row u for the group above
            *reinterpret_cast<float2*>(&s_rg_u[RG][j0]) = make_float2(plo(u[0][0]), plo(u[1][0]));
            gb_arrive<8 * (kU + RG)>(gb);
          }
          if (lane == 0) {
#pragma unroll
            for (int P = 0; P < NP; ++P) s_edge_u[RG][P][wc] = u[0][P];
          }
          gb_arrive<8 * (kE2 + RG)>(gb);
          GBWAIT(8 * (kE2 + RG), ph);
          // right neighbour of column 1: shuffles (lane 31 keeps its own column 1
          // at the global last column: gx = 0), the warp to the right's first
          // column from shared memory
          P2 right[NP];
#pragma unroll
          for (int P = 0; P < NP; ++P)
            right[P] = pk(__shfl_down_sync(0xffffffffu, plo(u[0][P]), 1),
                          __shfl_down_sync(0xffffffffu, phi(u[0][P]), 1));
          if (right_fetch) {
#pragma unroll
            for (int P = 0; P < NP; ++P) right[P] = s_edge_u[RG][P][wc + 1];
          }
          if (wc == CWARPS_ROW - 1) {  // (warp-uniform: only the last warp column pays the selects)
#pragma unroll
            for (int P = 0; P < NP; ++P) right[P] = lane == 31 ? u[1][P] : right[P];
          }
          auto q_pair = [&](int k, int P) {
            const P2 bl2 = P == NP - 1 ? pk(phi(u[k][0]), u_below[k]) : u[k][P < NP - 1 ? P + 1 : 0];
            const P2 rt = k == 0 ? u[1][P] : right[P];
            const P2 gy = pfma(u[k][P], m1, bl2);
            const P2 gx = pfma(u[k][P], m1, rt);
            const P2 ay = pfma(st2, gy, yy[k][P]);
            const P2 ax = pfma(st2, gx, yx[k][P]);
            const P2 m2 = pfma(ay, ay, pmul(ax, ax));
            const P2 rs = pk(rsqrt_approx(plo(m2)), rsqrt_approx(phi(m2)));
            const P2 s0 = pmul(w2, rs);
            const P2 sc = pk(fminf(1.f, plo(s0)), fminf(1.f, phi(s0)));  // w / max(w, |a|)
            QY[k][P] = pmul(ay, sc);
            QX[k][P] = pmul(ax, sc);
          };
          // halo rows of the new iterate: y_{it+1} (or q_n after the last iteration)
          const float b1 = (a.accelerated && it + 1 < a.n_inner) ? s_beta[it] : 0.f;
          if constexpr (TOP) {  // pair 0 holds row 0: compute it, push, then the rest
            q_pair(0, 0);
            q_pair(1, 0);
            if (has_up) {
              float v[4] = {plo(QY[0][0]), plo(QX[0][0]), plo(QY[1][0]), plo(QX[1][0])};
              if (it + 1 < a.n_inner) {
#pragma unroll
                for (int i = 0; i < 4; ++i) v[i] = fmaf(b1, fmaf(old_e[i], -1.f, v[i]), v[i]);
              }
              push_up(v[0], v[1], v[2], v[3]);
            }
#pragma unroll
            for (int P = 1; P < NP - 1; ++P) {
              q_pair(0, P);
              q_pair(1, P);
            }
            GBWAIT(8 * (kU + RG + 1), ph);
            const float2 ub = *reinterpret_cast<const float2*>(&s_rg_u[RG + 1][j0]);
            u_below[0] = ub.x;
            u_below[1] = ub.y;
            q_pair(0, NP - 1);
            q_pair(1, NP - 1);
          } else if constexpr (BOT) {  // pair NP-1 holds the last row: compute it, push, then the rest
            q_pair(0, NP - 1);
            q_pair(1, NP - 1);
            if (has_dn) {
              float v[2] = {phi(QY[0][NP - 1]), phi(QY[1][NP - 1])};
              if (it + 1 < a.n_inner) {
#pragma unroll
                for (int i = 0; i < 2; ++i) v[i] = fmaf(b1, fmaf(old_e[i], -1.f, v[i]), v[i]);
              }
              push_dn(v[0], v[1]);
            }
#pragma unroll
            for (int P = 0; P < NP - 1; ++P) {
              q_pair(0, P);
              q_pair(1, P);
            }
          } else {
#pragma unroll
            for (int P = 0; P < NP - 1; ++P) {
              q_pair(0, P);
              q_pair(1, P);
            }
            GBWAIT(8 * (kU + RG + 1), ph);
            const float2 ub = *reinterpret_cast<const float2*>(&s_rg_u[RG + 1][j0]);
            u_below[0] = ub.x;
            u_below[1] = ub.y;
            q_pair(0, NP - 1);
            q_pair(1, NP - 1);
          }
          tm_wait_st();  // q_{k-1} is in place for the next iteration's load
          ++round;
          ++gph;
        };
        inner(0, std::true_type{});
        for (int it = 1; it < a.n_inner; ++it) inner(it, std::false_type{});
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
          for (int P = 0; P < NP; ++P) {
            qky[k][P] = make_float2(plo(QY[k][P]), phi(QY[k][P]));
            qkx[k][P] = make_float2(plo(QX[k][P]), phi(QX[k][P]));
          }
      };
      PHASE_MARK(ph_b);
      if (rg == 0)
        run_inner(std::integral_constant<int, 0>{});
      else if (rg == 1)
        run_inner(std::integral_constant<int, 1>{});
      else if (rg == 2)
        run_inner(std::integral_constant<int, 2>{});
      else
        run_inner(std::integral_constant<int, 3>{});
      static_assert(CRG == 4, "one inner-loop copy per row group");

      PHASE_MARK(ph_c);
      // ---- epilogue: finalize u = clamp(z + div q_n) + ProxSkip post -----------
      // q_n's row / column halos inside the CTA go through the finalize's own
      // buffers (no barrier before these writes), z comes back from tensor
      // memory while the barrier is pending
      *reinterpret_cast<float2*>(&s_fin_yy[rg][j0]) =
          make_float2(rowref(qky[0], CRPT - 1), rowref(qky[1], CRPT - 1));
      if (lane == 31) {
#pragma unroll
        for (int P = 0; P < NP; ++P) s_fin_edge[rg][P][wc + 1] = pk(qkx[1][P].x, qkx[1][P].y);
      }
      uint32_t zw[16];
      tm_ld16(tm + kTmZ, zw);
      float yy_above[2] = {0.f, 0.f};
      {
        const unsigned r = round0 + a.n_inner;
        const unsigned pe = r & 1, ph = (r >> 1) & 1;
#ifndef PSB_DBG_NOHALO
        if (rg_bot && has_dn) {
          if (arm) mbar_expect_tx(&mb_dn[pe], BYTES_DN);
          mbar_wait(&mb_dn[pe], ph);
        }
        if (rg_top && has_up) {
          if (arm) mbar_expect_tx(&mb_up[pe], BYTES_UP);
          mbar_wait(&mb_up[pe], ph);
        }
#endif
        if (rg_top && has_up) {
          yy_above[0] = rx_up[pe][j0];
          yy_above[1] = rx_up[pe][j0 + 1];
        }
      }
      __syncthreads();
      float2 qleft[NP];
#pragma unroll
      for (int P = 0; P < NP; ++P) {
        qleft[P].x = __shfl_up_sync(0xffffffffu, qkx[1][P].x, 1);
        qleft[P].y = __shfl_up_sync(0xffffffffu, qkx[1][P].y, 1);
      }
      if (lane == 0) {
#pragma unroll
        for (int P = 0; P < NP; ++P) {
          const P2 e2 = s_fin_edge[rg][P][wc];
          qleft[P] = make_float2(plo(e2), phi(e2));
        }
      }
      if (!rg_top) {
        const float2 ya = *reinterpret_cast<const float2*>(&s_fin_yy[rg - 1][j0]);
        yy_above[0] = ya.x;
        yy_above[1] = ya.y;
      }
      bool ok = true;
      float2 zf[2][NP];
      tm_wait_ld(zw);
#pragma unroll
      for (int P = 0; P < NP; ++P) {
        zf[0][P] = make_float2(__uint_as_float(zw[4 * P]), __uint_as_float(zw[4 * P + 1]));
        zf[1][P] = make_float2(__uint_as_float(zw[4 * P + 2]), __uint_as_float(zw[4 * P + 3]));
      }
#pragma unroll
      for (int t = 0; t < CRPT; ++t) {
        const int sj = (rg * CRPT + t) * CW + j0;
        const float2 xo = *reinterpret_cast<const float2*>(&sx[sj]);  // x after the skips (prologue)
        const float2 bo = *reinterpret_cast<const float2*>(&sb[sj]);
        const float2 ho = *reinterpret_cast<const float2*>(&sh[sj]);
        float xn[2], hn[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const float left = k == 0 ? rowref(qleft, t) : rowref(qkx[0], t);
          const int r = row0 + t, j = j0 + k;
          float d = 0.f;
          if (r < CH - 1) d += rowref(qky[k], t);
          if (r > 0) d -= (t > 0 ? rowref(qky[k], t > 0 ? t - 1 : 0) : yy_above[k]);
          if (j < CW - 1) d += rowref(qkx[k], t);
          if (j > 0) d -= left;
          float uf = rowref(zf[k], t) + d;
          if (nonneg) uf = fmaxf(uf, 0.f);
          const float xok = k == 0 ? xo.x : xo.y, bok = k == 0 ? bo.x : bo.y, hok = k == 0 ? ho.x : ho.y;
          const float xhat = skip_update(xok, bok, hok, g);
          xn[k] = uf;
          hn[k] = F::add(hok, F::mul(a.pg, F::sub(uf, xhat)));
          ok &= finite(uf);
        }
        *reinterpret_cast<float2*>(&sh[sj]) = make_float2(hn[0], hn[1]);
        *reinterpret_cast<float2*>(&sx[sj]) = make_float2(xn[0], xn[1]);
      }
      if (!ok) kbad = min(kbad, kk);
      kprev = kk;
      PHASE_MARK(ph_d);
      PHASE_ADD(0, ph_a, ph_b);
      PHASE_ADD(1, ph_b, ph_c);
      PHASE_ADD(2, ph_c, ph_d);
    }  // prox calls

    // ---- trailing skips, write-back -------------------------------------------
    const int m = a.K - 1 - kprev;
#pragma unroll
    for (int t = 0; t < CRPT; ++t) {
      const int sj = (rg * CRPT + t) * CW + j0;
      const int64_t o = (int64_t)(row0 + t) * CW + j0;
      const float2 hv = *reinterpret_cast<const float2*>(&sh[sj]);
      const float2 xv = *reinterpret_cast<const float2*>(&sx[sj]);
      const float2 bv = *reinterpret_cast<const float2*>(&sb[sj]);
      float2 xo;
      xo.x = skip_chain_px(xv.x, bv.x, hv.x, g, m, kprev + 1, &kbad);
      xo.y = skip_chain_px(xv.y, bv.y, hv.y, g, m, kprev + 1, &kbad);
      *reinterpret_cast<float2*>(xp + o) = xo;
      if (e1 > e0 || cold) *reinterpret_cast<float2*>(hp + o) = hv;
      if (e1 > e0) {
        *reinterpret_cast<float2*>(q0 + o) = make_float2(rowref(qky[0], t), rowref(qky[1], t));
        *reinterpret_cast<float2*>(q0 + HW + o) = make_float2(rowref(qkx[0], t), rowref(qkx[1], t));
      }
    }
    if (kbad != 0x7fffffff && a.bad) atomicMin(a.bad + p, kbad);
    chunk_done(a.cs, p, 16 / CCL, tid == 0);  // this CTA's rows of the problem are written
    if (cr == 0 && tid == 0) wq_record(a.wq, 2, pos, t_claim);
  }  // problems
  cluster_arrive();  // no CTA leaves while a neighbour may still push into it
  cluster_wait();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(s_tm_base));
  // launched as a programmatic dependent of the 16-CTA cluster kernel (mixed
  // run): this grid completes only after that one (a no-op otherwise)
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

}  // namespace

int cluster8_ctas() { return CCL; }

// 8-CTA clusters of the run kernel resident on this device at once (cached)
int cluster8_count() {
  static int max_clusters = 0;
  if (max_clusters == 0) {
    int mc = 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CCL * 64);
    cfg.blockDim = dim3(CTHREADS);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CCL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.dynamicSmemBytes = kDynBytes;
    auto kern = fgp_cluster8_run_kernel<false>;
    if (func_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDynBytes) != PSB_OK ||
        cudaOccupancyMaxActiveClusters(&mc, kern, &cfg) != cudaSuccess || mc <= 0) {
      (void)cudaGetLastError();
      mc = 1;
    }
    max_clusters = mc;
  }
  return max_clusters;
}

template <bool NN>
static int launch_run8(const Run8Args& a, int G, bool dependent, cudaStream_t st) {
  auto kern = fgp_cluster8_run_kernel<NN>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)G * CCL);
  cfg.blockDim = dim3(CTHREADS);
  cfg.dynamicSmemBytes = kDynBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CCL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // placed once every CTA of the preceding (16-CTA cluster) kernel is resident
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = dependent ? 2 : 1;
  PSB_CHECK(func_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDynBytes));
  PSB_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  PSB_LAUNCHED("fgp_cluster8_run");
  return PSB_OK;
}

// fp32 outer state only (the fp64 instantiation stays on the 16-CTA kernel)
int cluster8_run(void* x, const void* b, void* h, void* q, int64_t qps, const WorkQueue& wq, int G,
                 const int32_t* ev_off, const int32_t* ev_k, const uint8_t* rep, int K, int n_inner,
                 int accelerated, int nonneg, double weight, double gamma, double hc, double pg,
                 double step, const float* betas, int32_t* bad, const ChunkSync& cs, bool dependent,
                 cudaStream_t st) {
  if (G <= 0) return PSB_OK;
  Run8Args a{(float*)x, (const float*)b, (float*)h, (float*)q, qps, wq, ev_off, ev_k, rep, K, n_inner,
             accelerated, (float)weight, (float)gamma, (float)hc, (float)pg, (float)step, bad, betas, cs};
  return nonneg ? launch_run8<true>(a, G, dependent, st) : launch_run8<false>(a, G, dependent, st);
}

}  // namespace psb

#ifdef PSB_DBG_PHASES
extern "C" int psb_debug_phases8(double* out16) {
  unsigned long long h[16];
  cudaMemcpyFromSymbol(h, psb::g_phase_ns, sizeof(h));
  for (int i = 0; i < 16; ++i) out16[i] = (double)h[i];
  return 0;
}
#endif

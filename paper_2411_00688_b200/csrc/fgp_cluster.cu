// Cluster-resident ProxSkip runs for 256 x 256 problems (BASELINE configs 1
// and 4).  ONE launch performs a whole run segment (K outer iterations) of
// every problem: each 16-CTA thread-block cluster takes its problems one after
// another (static longest-first assignment computed on the host) and, for a
// problem, walks its coin-fired iterations k_1 < k_2 < ... in order:
//
//   pre   : the skip iterations since the previous prox call,
//           x <- (x - g(x - b)) + g h, each one executed in registers in the
//           reference's op order, then the prox input
//           z = (x - g(x - b)) + hc h                      (skip.py:66-70)
//   FGP   : all n_inner accelerated iterations (tv.py:75-80) with the
//           problem's z, q_k, q_{k-1} resident in REGISTERS of the cluster
//           (16 SMs, 512 threads each, a column strip of 8 rows per thread);
//           row halos cross CTA boundaries as st.async pushes into the
//           neighbour's shared memory completing on its mbarrier, column
//           halos through warp shuffles and shared memory
//   post  : finalize u = clamp(z + div q_n) (tv.py:89), control variate
//           h <- h + (p/g)(u - xhat), x <- u                (skip.py:68-75)
//
// then applies the trailing skip iterations and writes x, h and the warm
// start back.  Between two prox calls of a problem its x, b, h stay in shared
// memory and its dual iterate q in registers, so HBM sees each problem once
// per run segment (~20 B/px in + ~16 B/px out) instead of ~1,450 B/px per
// prox call for 50 streaming FGP launches + pre + post, and there is no
// per-iteration launch or grid-wide step boundary at all: the per-problem
// work items are independent (the reference runs each config-4 problem on
// its own), which is what lets a single launch balance them across clusters.
//
// Every x update of the reference is executed, in the reference's order, with
// the same fp arithmetic as the streaming kernels; only the HBM round trips
// between iterations disappear.
#include <cooperative_groups.h>

#include <type_traits>

#include "cluster_ptx.cuh"

namespace cg = cooperative_groups;

namespace psb {

namespace {

constexpr int CW = 256;    // image width
constexpr int CCOLS = 2;   // columns per thread
constexpr int CRPT = 4;    // rows per thread
constexpr int CTPR = CW / CCOLS;           // threads per row group (128)
constexpr int CRG = 4;                     // row groups per CTA
constexpr int CCL = 16;                    // CTAs per cluster
constexpr int CH = CCL * CRG * CRPT;       // image height = 256
constexpr int CTHREADS = CTPR * CRG;       // 512 (8 pixels per thread: up to 128 registers)
constexpr int CWARPS_ROW = CTPR / 32;      // 4 warps across a row group
constexpr int kMaxBetas = 1024;       // momentum table staged in shared memory

template <class TO>
struct RunArgs {
  TO* x;
  const TO* b;
  TO* h;
  float* q;               // warm-start slot 0 of problem p: q + p*qps (channel stride CH*CW)
  int64_t qps;
  WorkQueue wq;            // problems claimed dynamically (common.cuh)
  const int32_t* ev_off;   // [n + 1]: problem p's coin-fired iterations ev_k[ev_off[p] ..]
  const int32_t* ev_k;     // ascending, 0 .. K-1 (this run segment)
  const uint8_t* rep;      // [n]: re-project the warm start at the first prox call (tv.py:68-69)
  int K;
  int n_inner;
  int accelerated;
  float weight;
  TO gamma, hc, pg;
  float step;
  int32_t* bad;            // [n]: first non-finite iteration (atomicMin)
  const float* betas;      // device table beta[0..n_inner-1]
  ChunkSync cs;            // optional input/output chunk streaming (common.cuh)
};

static_assert(CRG * CRPT == 16, "16 rows per CTA");

// Thread tile: 2 adjacent columns x CRPT (= 4) rows.  Each column strip is
// held as row PAIRS (t, t + 2) in float2 registers, so Blackwell's packed
// f32x2 FFMA2 / FADD2 / FMUL2 work on naturally aligned register pairs: the
// vertical neighbours of pair P are the pairs P^1 (one strip end builds a
// pair from two halves), the horizontal neighbour of column 0 is column 1 of
// the same thread, and only one column per side crosses to another lane
// (one shuffle per row and direction instead of two).  rowref(v, t) names
// row t of a column strip (t a compile-time constant after unrolling).
constexpr int NP = CRPT / 2;
static_assert(NP == 2, "row pairs (t, t+2) of a 4-row strip");
__device__ __forceinline__ float& rowref(float2 (&v)[NP], int t) {
  return (t & 1) ? ((t >> 1) ? v[1].y : v[1].x) : ((t >> 1) ? v[0].y : v[0].x);
}

// Exchange pattern per inner iteration: at the end of iteration t every CTA
// pushes its first row of q (both channels) to the CTA above and its last row
// of q (row channel) to the CTA below (st.async + the receiver's mbarrier,
// round-parity double buffers); at the start of t+1 each CTA waits for its
// neighbours' rows and rebuilds the halo y rows itself (momentum from the
// previously received rows).  The bottom row group also recomputes u for the
// first row of the CTA below, so no u ever crosses a CTA boundary.  Row groups
// inside a CTA and warp edges exchange through shared memory.
template <class TO, bool NONNEG>
__global__ void __launch_bounds__(CTHREADS, 1) fgp_cluster_run_kernel(RunArgs<TO> a) {
  using A = Ar<TO>;
  using F = Ar<float>;
  cg::cluster_group cluster = cg::this_cluster();
  const int cr = (int)cluster.block_rank();
  const int tid = threadIdx.x;
  const int jt = tid % CTPR, rg = tid / CTPR;  // column pair, row group
  const int j0 = 2 * jt;                        // columns j0, j0 + 1
  const int lane = tid & 31, wc = jt >> 5;
  const int row0 = cr * (CRG * CRPT) + rg * CRPT;
  const bool rg_top = rg == 0, rg_bot = rg == CRG - 1;
  const bool has_up = cr > 0, has_dn = cr < CCL - 1;
  constexpr int64_t HW = (int64_t)CH * CW;
  constexpr int SR = CRG * CRPT;  // rows of this CTA

  // halo rows received from the neighbours, double-buffered by round parity
  __shared__ __align__(16) float rx_dn[2][CW][2];  // CTA below's first row of q (y, x)
  __shared__ __align__(8) float rx_up[2][CW];      // CTA above's last row of q (y)
  __shared__ __align__(8) uint64_t mb_dn[2], mb_up[2];
  // the CTA below's first row of the prox input z, pushed once per prox call
  __shared__ __align__(16) float rx_z[CW];
  __shared__ __align__(8) uint64_t mb_z;
  // point-to-point row-group synchronisation of the inner loop (one phase per
  // inner iteration, 128 arrivals = every thread of the producing group):
  // gE1/gE2[g]: group g's warp-edge columns of y_x / u are in shared memory;
  // gYY[g]: group g's last-row y_y is out (for g+1); gU[g]: group g's
  // first-row u is out (for g-1)
  __shared__ __align__(8) uint64_t gE1[CRG], gE2[CRG], gYY[CRG], gU[CRG];
  __shared__ __align__(8) float s_rg_yy[CRG][CW];  // each row group's last-row y_y (for the group below)
  __shared__ __align__(8) float s_rg_u[CRG][CW];   // each row group's first-row u (for the group above)
  // warp-edge columns as row pairs: s_edge_yx[rg][.][w + 1] = last column of
  // warp w (slot 0 stays zero: nothing left of column 0; [NP].x = the halo
  // row's y_x), s_edge_u[rg][.][w] = first column of warp w
  __shared__ __align__(16) float2 s_edge_yx[CRG][NP + 1][CWARPS_ROW + 1];
  __shared__ __align__(16) float2 s_edge_u[CRG][NP][CWARPS_ROW];
  __shared__ float s_beta[kMaxBetas];
  __shared__ int s_next[2];  // rank 0: the claimed queue position, by problem parity
  // the problem's x, b, h rows of this CTA, resident for the whole problem
  extern __shared__ __align__(16) unsigned char stage_raw[];
  TO* sx = reinterpret_cast<TO*>(stage_raw);  // [SR][CW]
  TO* sb = sx + SR * CW;
  TO* sh = sb + SR * CW;

  const TO g = a.gamma;
  const float w = a.weight;
  constexpr bool nonneg = NONNEG;
  for (int e = tid; e < a.n_inner && e < kMaxBetas; e += CTHREADS) s_beta[e] = a.betas[e];
  if (tid < CRG * (NP + 1)) s_edge_yx[tid / (NP + 1)][tid % (NP + 1)][0] = make_float2(0.f, 0.f);
  if (tid == 0) {
    mbar_init(&mb_dn[0], 1);
    mbar_init(&mb_dn[1], 1);
    mbar_init(&mb_up[0], 1);
    mbar_init(&mb_up[1], 1);
    mbar_init(&mb_z, 1);
    for (int gi = 0; gi < CRG; ++gi) {
      mbar_init(&gE1[gi], CTPR);
      mbar_init(&gE2[gi], CTPR);
      mbar_init(&gYY[gi], CTPR);
      mbar_init(&gU[gi], CTPR);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // every CTA of this grid is resident: the SM-worker kernel (launched after
  // this one as a programmatic dependent) may now be placed on the SMs the
  // clusters left, without taking GPC space a cluster needs
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  cluster_arrive();  // every CTA's mbarriers exist before anyone pushes
  cluster_wait();
  // Round r carries the rows published after iteration r-1 (round 0: the warm
  // start) and lands in buffer r&1; the counter runs across prox calls.
  constexpr unsigned BYTES_DN = CW * 2 * 4, BYTES_UP = CW * 4;
  const uint32_t up_rx_remote = dsmem_addr(&rx_dn[0][0][0], cr > 0 ? cr - 1 : cr);   // my top row -> CTA above
  const uint32_t up_mb_remote = dsmem_addr(&mb_dn[0], cr > 0 ? cr - 1 : cr);
  const uint32_t dn_rx_remote = dsmem_addr(&rx_up[0][0], cr < CCL - 1 ? cr + 1 : cr); // my bottom row -> CTA below
  const uint32_t dn_mb_remote = dsmem_addr(&mb_up[0], cr < CCL - 1 ? cr + 1 : cr);
  // my first row of z -> the CTA above (once per prox call)
  const uint32_t z_rx_remote = dsmem_addr(&rx_z[0], cr > 0 ? cr - 1 : cr);
  const uint32_t z_mb_remote = dsmem_addr(&mb_z, cr > 0 ? cr - 1 : cr);
  unsigned zph = 0;  // prox calls so far (mb_z phases)
  unsigned round = 0;
  unsigned gph = 0;  // inner iterations so far (row-group mbarrier phases)
  auto push_rows = [&](float ty0, float tx0, float ty1, float tx1, float by0, float by1) {
#ifdef PSB_DBG_NOHALO
    return;
#endif
    const unsigned b = round & 1;
    if (rg_top && cr > 0)
      st_async_v4(up_rx_remote + 4u * (b * CW * 2 + j0 * 2), ty0, tx0, ty1, tx1, up_mb_remote + 8u * b);
    if (rg_bot && cr < CCL - 1)
      st_async_v2(dn_rx_remote + 4u * (b * CW + j0), by0, by1, dn_mb_remote + 8u * b);
  };
  // wait for round `r` (consumer side); returns the buffer index
  // warp-uniform roles: the bottom row group waits for the CTA below, the top
  // one for the CTA above; lane 0 of the role's first warp arms the barrier
  const bool wait_dn = rg_bot && cr < CCL - 1, wait_up = rg_top && cr > 0;
  const bool arm = lane == 0 && wc == 0;
  auto recv_rows = [&](unsigned r) {
    const unsigned b = r & 1, ph = (r >> 1) & 1;
#ifdef PSB_DBG_NOHALO
    return b;
#endif
    if (wait_dn) {
      if (arm) mbar_expect_tx(&mb_dn[b], BYTES_DN);
      mbar_wait(&mb_dn[b], ph);
    }
    if (wait_up) {
      if (arm) mbar_expect_tx(&mb_up[b], BYTES_UP);
      mbar_wait(&mb_up[b], ph);
    }
    return b;
  };
  // role-specialised halves of push_rows / recv_rows for the inner loop
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
  const bool last_row_thread = rg_bot && !has_dn;  // owns global row H-1 (t = CRPT-1)
  const bool right_fetch = lane == 31 && wc < CWARPS_ROW - 1;
  const bool last_col = lane == 31 && wc == CWARPS_ROW - 1;  // owns global column W-1

  const uint32_t next_remote = dsmem_addr(&s_next[0], 0);
  uint64_t t_claim = 0;
  for (unsigned pj = 0;; ++pj) {
  // rank 0 claims the next problem; everyone reads it after the barrier
  // (slot pj & 1 was last read before the previous problem's barrier)
  if (cr == 0 && tid == 0) s_next[pj & 1] = wq_claim(a.wq);
  cluster_arrive();
  cluster_wait();
  const int pos = dsmem_ld<int>(next_remote + 4u * (pj & 1));
  if (pos < 0) break;
  const int p = a.wq.order[pos];
  TO* xp = a.x + (int64_t)p * HW;
  const TO* bp = a.b + (int64_t)p * HW;
  TO* hp = a.h + (int64_t)p * HW;
  float* q0 = a.q + (int64_t)p * a.qps;
  const int e0 = a.ev_off[p], e1 = a.ev_off[p + 1];
  const bool rep = a.rep[p];
  if (a.cs.ready) {  // this problem's input chunk has arrived
    if (tid == 0) chunk_wait(a.cs, p);
    __syncthreads();
  }
  if (cr == 0 && tid == 0) t_claim = gtimer_ns();
  // stage this CTA's rows of x, b, h (each thread its own elements; the CTA
  // above reads row 0 after the next cluster barrier)
  // (a streamed run starts cold: x = h = 0 and q_warm = 0 are implied and
  // the device buffers are not initialised -- psb_proxskip_denoise_run_streamed)
  const bool cold = a.cs.ready != nullptr;
  // per column k: z, q_k, q_{k-1} as row pairs
  float2 z[2][NP], qky[2][NP], qkx[2][NP], qmy[2][NP], qmx[2][NP];
  // the warm-start duals (slot 0) are loaded here with x, b, h so the first
  // prox call does not pay a second HBM round trip
#pragma unroll
  for (int t = 0; t < CRPT; ++t) {
    const int lr = rg * CRPT + t;
    const int64_t o = (int64_t)(row0 + t) * CW + j0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      sx[lr * CW + j0 + k] = cold ? TO(0) : xp[o + k];
      sb[lr * CW + j0 + k] = bp[o + k];
      sh[lr * CW + j0 + k] = cold ? TO(0) : hp[o + k];
      rowref(qky[k], t) = cold || e1 == e0 ? 0.f : q0[o + k];
      rowref(qkx[k], t) = cold || e1 == e0 ? 0.f : q0[HW + o + k];
    }
  }
  int kbad = 0x7fffffff;
  int kprev = -1;
  for (int e = e0; e < e1; ++e) {
  const int kk = a.ev_k[e];
  const int m = kk - kprev - 1;  // skip iterations kprev+1 .. kk-1 before this prox call
  const int kf = kprev + 1;
  // (no cluster-wide barrier per prox call: the only data crossing CTAs are
  // the halo rows and the z row, each tracked by the receiver's mbarrier)
  __syncthreads();
  PHASE_MARK(ph_a);
  // ---- prologue: skips, prox input, warm start ------------------------------
  // The m skipped iterations since the last prox call (skip.py:68), executed
  // in the reference's op order; x after them goes back to shared memory for
  // the epilogue.  A non-finite x stays non-finite under the skip update, so
  // only the final x is tested; the slow path finds the first bad iteration.
  auto prox_input = [&](int sj) {
    const TO bo = sb[sj], ho = sh[sj];
    const TO xo = skip_chain_px(sx[sj], bo, ho, g, m, kf, &kbad);
    if (m > 0) sx[sj] = xo;
    return (float)A::add(A::sub(xo, A::mul(g, A::sub(xo, bo))), A::mul(a.hc, ho));
  };
#pragma unroll
  for (int k = 0; k < 2; ++k) {
#pragma unroll
    for (int t = 0; t < CRPT; ++t) {
      const int lr = rg * CRPT + t;
      const int sj = lr * CW + j0 + k;
      rowref(z[k], t) = prox_input(sj);
      if (e == e0) {  // warm start (staged above), re-projected if the weight changed
        float vy = rowref(qky[k], t), vx = rowref(qkx[k], t);
        if (rep) {
          const float sc = F::ball_scale(vy, vx, w);
          vy *= sc;
          vx *= sc;
        }
        // The reference's divergence ignores q_y on the last row and q_x on
        // the last column (operators.py:66-70) and the gradient is 0 there,
        // so those entries stay 0 from a cold start; zeroing them here lets
        // the inner loop drop every boundary test (zero padding, not masks).
        if (row0 + t == CH - 1) vy = 0.f;
        if (j0 + k == CW - 1) vx = 0.f;
        rowref(qky[k], t) = vy;
        rowref(qkx[k], t) = vx;
      }
    }
#pragma unroll
    for (int P = 0; P < NP; ++P) {
      qmy[k][P] = qky[k][P];  // the momentum restarts with every call (tv.py:72)
      qmx[k][P] = qkx[k][P];
    }
  }
  // the bottom row group also owns the CTA-below's first row for u: its z
  // arrives from that CTA (st.async on mb_z); mine goes to the CTA above
  if (rg_top && has_up)
    st_async_v2(z_rx_remote + 4u * j0, z[0][0].x, z[1][0].x, z_mb_remote);
  float z_ex[2] = {0.f, 0.f};
  if (rg_bot && has_dn) {
    if (arm) mbar_expect_tx(&mb_z, CW * 4);
    mbar_wait(&mb_z, zph & 1u);
    z_ex[0] = rx_z[j0];
    z_ex[1] = rx_z[j0 + 1];
  }
  ++zph;
  // After the first call of a problem the warm start is the previous call's
  // q_n, whose boundary rows arrived in that call's final round: the first
  // inner iteration reads them from there (and forms y_0 itself) instead of
  // exchanging them again -- one DSMEM round trip less per prox call.
  const bool reuse = e > e0;
  const unsigned round0 = reuse ? round - 1 : round;  // this call's warm-start round
  // Halo rows travel as MOMENTUM iterates y (the receiver uses them as they
  // are): the warm-start round carries y_0 = fma(0, q_0 - q_0, q_0), round
  // it + 1 (it + 1 < n) carries y_{it+1} = fma(beta_{it+1}, q_{it+1} - q_it,
  // q_{it+1}) -- the values the owner computes for its own pixels, bit for bit
  // -- and the last round q_n itself (the finalize reads q_n).
  if (!reuse) {
    float v[6];
    const float y0s[6] = {qky[0][0].x, qkx[0][0].x, qky[1][0].x, qkx[1][0].x, qky[0][1].y,
                          qky[1][1].y};
#pragma unroll
    for (int i = 0; i < 6; ++i) v[i] = fmaf(0.f, fmaf(y0s[i], -1.f, y0s[i]), y0s[i]);
    push_rows(v[0], v[1], v[2], v[3], v[4], v[5]);
    ++round;
  }
  // y_0 of a halo value q (beta_0 = 0), exactly as the owner forms it
  auto y0_of = [](float q) { return fmaf(0.f, fmaf(q, -1.f, q), q); };

  // One inner iteration; reads (QK, QM), writes the new iterate into QM.
  // Each pixel's arithmetic is the scalar FGP step (each f32x2 lane an IEEE
  // fp32 op; a - b = fma(b, -1, a)).  ROLE (warp-uniform, fixed per warp):
  // 0 = top row group (halo row from the CTA above), 1 = middle groups (all
  // neighbours inside the CTA), 2 = bottom group (halo row from the CTA
  // below, computes u of that row itself) -- one specialised copy each, so
  // the middle groups carry no halo code at all.
  auto run_inner = [&](auto role_tag) {
    constexpr int ROLE = decltype(role_tag)::value;
    constexpr bool TOP = ROLE == 0, BOT = ROLE == 2;
    // Row groups synchronise point to point through the gE1/gE2/gYY/gU
    // mbarriers (one phase per inner iteration) instead of two CTA-wide
    // barriers: a group waits only for the data it reads -- its own warps'
    // edge columns and one row of each adjacent group -- so the groups run
    // skewed and the boundary groups compute their halo pair first: the top
    // group pushes its first row to the CTA above before it needs the middle
    // group's u, the bottom group pushes its last row before it needs the
    // middle group's y.  Shared-memory reuse across iterations is ordered by
    // the same waits (a group cannot reach iteration t+1's write of a row
    // before its readers have passed their wait for iteration t).
    auto inner = [&](float2(&QKy)[2][NP], float2(&QKx)[2][NP], float2(&QMy)[2][NP],
                     float2(&QMx)[2][NP], int it) {
      const unsigned ph = gph & 1u;
      const float beta = (a.accelerated && it > 0) ? s_beta[it - 1] : 0.f;
      const float2 b2 = make_float2(beta, beta), m1 = make_float2(-1.f, -1.f);
      float2 yy[2][NP], yx[2][NP];
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int P = 0; P < NP; ++P) {
          yy[k][P] = __ffma2_rn(b2, __ffma2_rn(QMy[k][P], m1, QKy[k][P]), QKy[k][P]);
          yx[k][P] = __ffma2_rn(b2, __ffma2_rn(QMx[k][P], m1, QKx[k][P]), QKx[k][P]);
        }
      if constexpr (!BOT) {  // last-row y_y for the group below
        s_rg_yy[rg][j0] = yy[0][1].y;  // row CRPT-1
        s_rg_yy[rg][j0 + 1] = yy[1][1].y;
        mbar_arrive(&gYY[rg]);
      }
      if (lane == 31) {
#pragma unroll
        for (int P = 0; P < NP; ++P) s_edge_yx[rg][P][wc + 1] = yx[1][P];
      }
      mbar_arrive(&gE1[rg]);
      float2 yyA = make_float2(0.f, 0.f);             // TOP: y row above (zeros at row 0)
      float ex_y[2] = {0.f, 0.f}, ex_x[2] = {0.f, 0.f}, ledge_x = 0.f;  // BOT: row below
      if constexpr (TOP) {
        if (has_up) {
          const bool warm = reuse && it == 0;  // (already received: final round)
          const unsigned par = warm ? (round0 & 1u) : recv_up(round0 + it);
          yyA = *reinterpret_cast<const float2*>(&rx_up[par][j0]);
          if (warm) yyA = make_float2(y0_of(yyA.x), y0_of(yyA.y));
        }
      }
      if constexpr (BOT) {
        if (has_dn) {
          const bool warm = reuse && it == 0;  // (already received: final round)
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
      GWAIT(&gE1[rg], ph);
      // left neighbours of column 0: shuffles inside the warp, the warp to the
      // left's last column from shared memory (zeros left of column 0); column
      // 1's left neighbour is this thread's column 0
      float2 left[NP];
#pragma unroll
      for (int P = 0; P < NP; ++P) {
        left[P].x = __shfl_up_sync(0xffffffffu, yx[1][P].x, 1);
        left[P].y = __shfl_up_sync(0xffffffffu, yx[1][P].y, 1);
      }
      if (lane == 0) {
#pragma unroll
        for (int P = 0; P < NP; ++P) left[P] = s_edge_yx[rg][P][wc];
      }
      float yy_above[2] = {yyA.x, yyA.y};
      float2 u[2][NP];
      // ((0 + yy) - yy_up) + yx - yx_left, boundary terms zero-padded; u = z + d
      auto u_pair = [&](int k, int P) {
        const float2 ab2 = P == 0 ? make_float2(yy_above[k], yy[k][1].x) : yy[k][0];
        const float2 l2 = k == 0 ? left[P] : yx[0][P];
        const float2 d1 = __fadd2_rn(__ffma2_rn(ab2, m1, yy[k][P]), yx[k][P]);
        const float2 d2 = __ffma2_rn(l2, m1, d1);
        const float2 v = __fadd2_rn(z[k][P], d2);
        u[k][P] = nonneg ? make_float2(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f)) : v;
      };
      if constexpr (BOT) {  // pair 1 (rows 1, 3) needs no row above
        u_pair(0, 1);
        u_pair(1, 1);
      }
      if constexpr (!TOP) {
        GWAIT(&gYY[rg - 1], ph);
        const float2 ya2 = *reinterpret_cast<const float2*>(&s_rg_yy[rg - 1][j0]);
        yy_above[0] = ya2.x;
        yy_above[1] = ya2.y;
      }
      u_pair(0, 0);
      u_pair(1, 0);
      if constexpr (!BOT) {
        u_pair(0, 1);
        u_pair(1, 1);
      }
      float u_below[2];
      if constexpr (BOT) {
        if (has_dn) {  // u of the CTA-below's first row, from its y row
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const float d = ((ex_y[k] - yy[k][1].y) + ex_x[k]) - (k == 0 ? ledge_x : ex_x[0]);
            const float v = z_ex[k] + d;
            u_below[k] = nonneg ? fmaxf(v, 0.f) : v;
          }
        } else {  // the global last row: gy = 0 (below := u)
          u_below[0] = u[0][1].y;
          u_below[1] = u[1][1].y;
        }
      }
      if constexpr (!TOP) {  // first-row u for the group above
        s_rg_u[rg][j0] = u[0][0].x;
        s_rg_u[rg][j0 + 1] = u[1][0].x;
        mbar_arrive(&gU[rg]);
      }
      if (lane == 0) {
#pragma unroll
        for (int P = 0; P < NP; ++P) s_edge_u[rg][P][wc] = u[0][P];
      }
      mbar_arrive(&gE2[rg]);
      GWAIT(&gE2[rg], ph);
      // right neighbour of column 1: shuffles (lane 31 keeps its own column 1 at
      // the global last column: gx = 0), the warp to the right's first column
      // from shared memory; column 0's right neighbour is column 1
      float2 right[NP];
#pragma unroll
      for (int P = 0; P < NP; ++P) {
        right[P].x = __shfl_down_sync(0xffffffffu, u[0][P].x, 1);
        right[P].y = __shfl_down_sync(0xffffffffu, u[0][P].y, 1);
      }
      if (right_fetch) {
#pragma unroll
        for (int P = 0; P < NP; ++P) right[P] = s_edge_u[rg][P][wc + 1];
      }
      if (last_col) {
#pragma unroll
        for (int P = 0; P < NP; ++P) right[P] = u[1][P];
      }
      const float wr = w * kBallShrink;  // (common.cuh)
      const float2 st2 = make_float2(a.step, a.step), w2 = make_float2(wr, wr);
      auto q_pair = [&](int k, int P) {
        const float2 bl2 = P == 0 ? u[k][1] : make_float2(u[k][0].y, u_below[k]);
        const float2 rt = k == 0 ? u[1][P] : right[P];
        const float2 gy = __ffma2_rn(u[k][P], m1, bl2);
        const float2 gx = __ffma2_rn(u[k][P], m1, rt);
        const float2 ay = __ffma2_rn(st2, gy, yy[k][P]);
        const float2 ax = __ffma2_rn(st2, gx, yx[k][P]);
        const float2 m2 = __ffma2_rn(ay, ay, __fmul2_rn(ax, ax));
        float2 sc = __fmul2_rn(w2, make_float2(rsqrt_approx(m2.x), rsqrt_approx(m2.y)));
        sc.x = fminf(1.f, sc.x);  // w / max(w, |a|)
        sc.y = fminf(1.f, sc.y);
        QMy[k][P] = __fmul2_rn(ay, sc);
        QMx[k][P] = __fmul2_rn(ax, sc);
      };
      // halo rows of the new iterate: y_{it+1} (or q_n after the last iteration)
      const float b1 = (a.accelerated && it + 1 < a.n_inner) ? s_beta[it] : 0.f;
      if constexpr (TOP) {  // pair 0 holds row 0: compute it, push, then pair 1
        q_pair(0, 0);
        q_pair(1, 0);
        if (has_up) {
          float v[4] = {QMy[0][0].x, QMx[0][0].x, QMy[1][0].x, QMx[1][0].x};
          if (it + 1 < a.n_inner) {
            const float o[4] = {QKy[0][0].x, QKx[0][0].x, QKy[1][0].x, QKx[1][0].x};
#pragma unroll
            for (int i = 0; i < 4; ++i) v[i] = fmaf(b1, fmaf(o[i], -1.f, v[i]), v[i]);
          }
          push_up(v[0], v[1], v[2], v[3]);
        }
        GWAIT(&gU[rg + 1], ph);
        const float2 ub = *reinterpret_cast<const float2*>(&s_rg_u[rg + 1][j0]);
        u_below[0] = ub.x;
        u_below[1] = ub.y;
        q_pair(0, 1);
        q_pair(1, 1);
      } else if constexpr (BOT) {  // pair 1 holds row 3: compute it, push, then pair 0
        q_pair(0, 1);
        q_pair(1, 1);
        if (has_dn) {
          float v[2] = {QMy[0][1].y, QMy[1][1].y};
          if (it + 1 < a.n_inner) {
            const float o[2] = {QKy[0][1].y, QKy[1][1].y};
#pragma unroll
            for (int i = 0; i < 2; ++i) v[i] = fmaf(b1, fmaf(o[i], -1.f, v[i]), v[i]);
          }
          push_dn(v[0], v[1]);
        }
        q_pair(0, 0);
        q_pair(1, 0);
      } else {
        GWAIT(&gU[rg + 1], ph);
        const float2 ub = *reinterpret_cast<const float2*>(&s_rg_u[rg + 1][j0]);
        u_below[0] = ub.x;
        u_below[1] = ub.y;
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
          for (int P = 0; P < NP; ++P) q_pair(k, P);
      }
      ++round;
      ++gph;
    };

    int it = 0;
    for (; it + 1 < a.n_inner; it += 2) {
      inner(qky, qkx, qmy, qmx, it);      // new iterate in qm*
      inner(qmy, qmx, qky, qkx, it + 1);  // new iterate in qk*
    }
    if (it < a.n_inner) {
      inner(qky, qkx, qmy, qmx, it);
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int P = 0; P < NP; ++P) {
          qky[k][P] = qmy[k][P];
          qkx[k][P] = qmx[k][P];
        }
    }
  };
  PHASE_MARK(ph_b);
  if (rg_top)
    run_inner(std::integral_constant<int, 0>{});
  else if (rg_bot)
    run_inner(std::integral_constant<int, 2>{});
  else
    run_inner(std::integral_constant<int, 1>{});

  PHASE_MARK(ph_c);
  // ---- epilogue: finalize u = clamp(z + div q_n) + ProxSkip post -------------
  __syncthreads();  // every group is past its last inner iteration's reads
  const unsigned pe = recv_rows(round0 + a.n_inner);
  float yy_above[2] = {0.f, 0.f};
  if (rg_top && has_up) {
    yy_above[0] = rx_up[pe][j0];
    yy_above[1] = rx_up[pe][j0 + 1];
  }
  s_rg_yy[rg][j0] = rowref(qky[0], CRPT - 1);
  s_rg_yy[rg][j0 + 1] = rowref(qky[1], CRPT - 1);
  if (lane == 31) {
#pragma unroll
    for (int P = 0; P < NP; ++P) s_edge_yx[rg][P][wc + 1] = qkx[1][P];
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
    for (int P = 0; P < NP; ++P) qleft[P] = s_edge_yx[rg][P][wc];
  }
  if (!rg_top) {
    yy_above[0] = s_rg_yy[rg - 1][j0];
    yy_above[1] = s_rg_yy[rg - 1][j0 + 1];
  }
  bool ok = true;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
#pragma unroll
    for (int t = 0; t < CRPT; ++t) {
      const float left = k == 0 ? rowref(qleft, t) : rowref(qkx[0], t);
      const int r = row0 + t, j = j0 + k;
      float d = 0.f;
      if (r < CH - 1) d += rowref(qky[k], t);
      if (r > 0) d -= (t > 0 ? rowref(qky[k], t - 1) : yy_above[k]);
      if (j < CW - 1) d += rowref(qkx[k], t);
      if (j > 0) d -= left;
      float uf = rowref(z[k], t) + d;
      if (nonneg) uf = fmaxf(uf, 0.f);
      const int sj = (rg * CRPT + t) * CW + j;
      const TO xo = sx[sj];  // x after the skips (prologue)
      const TO bo = sb[sj], ho = sh[sj];
      const TO xhat = skip_update(xo, bo, ho, g);
      const TO xn = (TO)uf;
      sh[sj] = A::add(ho, A::mul(a.pg, A::sub(xn, xhat)));
      sx[sj] = xn;
      ok &= finite(xn);
    }
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
  for (int k = 0; k < 2; ++k) {
#pragma unroll
    for (int t = 0; t < CRPT; ++t) {
      const int sj = (rg * CRPT + t) * CW + j0 + k;
      const int64_t o = (int64_t)(row0 + t) * CW + j0 + k;
      const TO ho = sh[sj];
      const TO xo = skip_chain_px(sx[sj], sb[sj], ho, g, m, kprev + 1, &kbad);
      xp[o] = xo;
      if (e1 > e0 || cold) hp[o] = ho;
      if (e1 > e0) {
        q0[o] = rowref(qky[k], t);
        q0[HW + o] = rowref(qkx[k], t);
      }
    }
  }
  if (kbad != 0x7fffffff && a.bad) atomicMin(a.bad + p, kbad);
  chunk_done(a.cs, p, 1, tid == 0);  // this CTA's rows of the problem are written
  if (cr == 0 && tid == 0) wq_record(a.wq, 0, pos, t_claim);
  // The next problem's staging may overwrite row 0 of this CTA only after the
  // CTA above has read it: it did so in the prologue of this problem's last
  // prox call, before its first push of that call, which this CTA waited for.
  }  // problems
  cluster_arrive();  // no CTA leaves while a neighbour may still push into it
  cluster_wait();
}

}  // namespace

bool cluster_shape_ok(int H, int W) { return H == CH && W == CW; }

static size_t stage_bytes(int dto) {
  return (size_t)(dto == PSB_F64 ? 8 : 4) * 3 * CRG * CRPT * CW;
}

// 16-CTA clusters of the run kernel resident on this device at once (cached)
int cluster_count() {
  static int max_clusters = 0;
  if (max_clusters == 0) {
    int mc = 0;
    if (psb_cluster_max_active(&mc) != PSB_OK || mc <= 0) mc = 1;
    max_clusters = mc;
  }
  return max_clusters;
}

template <class TO, bool NN>
static int launch_run(const RunArgs<TO>& a, int G, int dto, cudaStream_t st) {
  auto kern = fgp_cluster_run_kernel<TO, NN>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)G * CCL);
  cfg.blockDim = dim3(CTHREADS);
  cfg.dynamicSmemBytes = stage_bytes(dto);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CCL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  PSB_CHECK(func_attr(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  PSB_CHECK(func_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes));
  PSB_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  PSB_LAUNCHED("fgp_cluster_run");
  return PSB_OK;
}

int cluster_run(int dto, void* x, const void* b, void* h, void* q, int64_t qps,
                const WorkQueue& wq, int G, const int32_t* ev_off, const int32_t* ev_k,
                const uint8_t* rep, int K, int n_inner, int accelerated, int nonneg,
                double weight, double gamma, double hc, double pg, double step,
                const float* betas, int32_t* bad, const ChunkSync& cs, cudaStream_t st) {
  if (G <= 0) return PSB_OK;
  if (dto == PSB_F32) {
    RunArgs<float> a{(float*)x, (const float*)b, (float*)h, (float*)q, qps, wq, ev_off, ev_k, rep,
                     K, n_inner, accelerated, (float)weight, (float)gamma, (float)hc, (float)pg,
                     (float)step, bad, betas, cs};
    return nonneg ? launch_run<float, true>(a, G, dto, st) : launch_run<float, false>(a, G, dto, st);
  }
  if (dto == PSB_F64) {
    RunArgs<double> a{(double*)x, (const double*)b, (double*)h, (float*)q, qps, wq, ev_off, ev_k,
                      rep, K, n_inner, accelerated, (float)weight, gamma, hc, pg, (float)step, bad,
                      betas, cs};
    return nonneg ? launch_run<double, true>(a, G, dto, st) : launch_run<double, false>(a, G, dto, st);
  }
  return fail(PSB_ERR_VALUE, "cluster run: unknown dtype");
}

}  // namespace psb

#ifdef PSB_DBG_PHASES
extern "C" int psb_debug_phases(double* out16) {
  unsigned long long h[16];
  cudaMemcpyFromSymbol(h, psb::g_phase_ns, sizeof(h));
  for (int i = 0; i < 16; ++i) out16[i] = (double)h[i];
  return 0;
}
#endif

extern "C" int psb_cluster_max_active(int* out) {
  using namespace psb;
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
  cfg.dynamicSmemBytes = stage_bytes(PSB_F64);
  auto kern = fgp_cluster_run_kernel<float, false>;
  PSB_CHECK(func_attr(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  PSB_CHECK(func_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes));
  PSB_CUDA(cudaOccupancyMaxActiveClusters(out, kern, &cfg));
  return PSB_OK;
}

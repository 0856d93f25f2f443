// Native run driver for ProxSkip TV denoising (BASELINE configs 1 and 4).
//
// The Bernoulli coins of every problem and iteration are known before the run
// (drawn on the host from the reference's Philox streams, skip.py:27-28), so
// the driver resolves the control flow up front: it compacts the coin table
// into per-iteration active lists, uploads them once, and enqueues
//     pre(all problems) -> n_inner x fgp2d_iter(active) -> post(active)
// per outer iteration without any host synchronisation.  With use_graph the
// whole launch sequence is captured into one CUDA graph first (a 256^2 FGP
// iteration is only a few microseconds of GPU work, so launch cost matters).
#include <climits>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <chrono>

#include "common.cuh"

namespace psb {

int fgp2d_iter(int dtype, const void* x, int64_t xps, void* q, int64_t qps, const int32_t* active,
               int n_active, double weight, const double* wts, int rep_all, const uint8_t* rep,
               int H, int W, int it, double beta, double step, int nonneg, cudaStream_t st);
int proxskip_pre(int dto, int dtf, void* x, const void* gb, int ident, const void* h, void* z,
                 int64_t n, int64_t HW, const uint8_t* coins, double gamma, double hcoef,
                 int32_t* bad, int k, cudaStream_t st);
int proxskip_post(int dto, int dtf, void* x, const void* gb, int ident, void* h, const void* z,
                  void* q, int64_t qps, const int32_t* active, int n_active, int H, int W,
                  int n_inner, int nonneg, double gamma, double pg, int32_t* bad, int k,
                  cudaStream_t st);
void fista_betas(int n, double* out);
int blur_grad2d(int dtype, const void* u, const void* b, void* g, int H, int W,
                const double* taps2d, const double* taps1d, int k, int separable, void* scratch,
                cudaStream_t st);
bool cluster_shape_ok(int H, int W);
int cluster_count();
int cluster8_count();
int cluster8_run(void* x, const void* b, void* h, void* q, int64_t qps, const WorkQueue& wq, int G,
                 const int32_t* ev_off, const int32_t* ev_k, const uint8_t* rep, int K, int n_inner,
                 int accelerated, int nonneg, double weight, double gamma, double hc, double pg,
                 double step, const float* betas, int32_t* bad, const ChunkSync& cs, bool dependent,
                 cudaStream_t st);
int sm_prepare();
int sm_run(void* x, const void* b, void* h, void* q, int64_t qps, void* z, const WorkQueue& wq,
           int n_workers, const int32_t* ev_off, const int32_t* ev_k, const uint8_t* rep, int K,
           int n_inner, int accelerated, int nonneg, double weight, double gamma, double hc,
           double pg, double step, const float* betas, int32_t* bad, const ChunkSync& cs,
           bool after_clusters, cudaStream_t st);
int cluster_run(int dto, void* x, const void* b, void* h, void* q, int64_t qps,
                const WorkQueue& wq, int G, const int32_t* ev_off, const int32_t* ev_k,
                const uint8_t* rep, int K, int n_inner, int accelerated, int nonneg,
                double weight, double gamma, double hc, double pg, double step,
                const float* betas, int32_t* bad, const ChunkSync& cs, cudaStream_t st);
int fgp2d_run(int dtype, const void* x, int64_t xps, void* q, int64_t qps, const int32_t* active,
              int n_active, double weight, const double* wts, int rep_all, const uint8_t* rep,
              int H, int W, int n_inner, int accelerated, int nonneg, double step,
              const double* betas_host, cudaStream_t st);
int fista_extrap(int dto, void* x, void* xprev, void* xbar, int64_t count, double beta,
                 cudaStream_t st);
int fista_pre(int dto, int dtf, const void* xbar, const void* gb, int ident, void* z, int64_t count,
              double gamma, cudaStream_t st);

// Fidelity A of the implicit splitting.  kind 0: identity (g = x - b fused
// into the outer kernels); kind 1: periodic blur (g = A^T(Ax - b) by the
// fused separable kernel, or the bit-exact direct path, into `g`).
int blur_grad_pre2d(int dto, int dtf, const void* x, const void* b, void* g, int H, int W,
                    const double* taps1d, int k, void* x_next, const void* h, void* z,
                    double gamma, double hcoef, int coin, int32_t* bad, int kiter,
                    cudaStream_t st);

struct Fidelity {
  int kind = 0;
  const double* taps2d = nullptr;
  const double* taps1d = nullptr;
  int ksize = 0;
  int separable = 1;
  void* g = nullptr;
  void* scratch = nullptr;
  // FISTA (algo 1): x_prev and xbar buffers (n*H*W of the outer dtype each)
  int fista = 0;
  void* xprev = nullptr;
  void* xbar = nullptr;
};

namespace {

// Stream-ordered scratch: allocated and released on the caller's stream, so
// the driver returns as soon as the run is enqueued (a synchronous cudaFree
// would block the host -- and any timer that waits for the call -- until the
// device is idle).
struct DevBuf {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
};

}  // namespace

// page-locked copy of the last cluster run's work-queue statistics
static unsigned long long* queue_stats_host() {
  static unsigned long long* p = nullptr;
  if (p == nullptr) {
    void* h = nullptr;
    if (cudaHostAlloc(&h, 6 * sizeof(unsigned long long), cudaHostAllocDefault) != cudaSuccess)
      return nullptr;
    p = static_cast<unsigned long long*>(h);
    for (int i = 0; i < 6; ++i) p[i] = 0;
  }
  return p;
}

int proxskip_tv_run(const Fidelity& fid, int dto, int dtf, void* x, const void* b, void* h, void* z,
                    void* q, int64_t n, int H, int W, const uint8_t* coins_host, int K,
                    double gamma, double p, double alpha, int n_inner, int accelerated, int nonneg,
                    double* last_weight, int64_t* prox_count, int32_t* bad, int use_graph,
                    double* elapsed, double* fgp_time, void* x_hist, cudaStream_t user_stream,
                    const ChunkSync* chunks = nullptr) {
  PSB_REQUIRE(fid.kind == 0 || n == 1, "proxskip run: a blur fidelity runs one problem at a time");
  PSB_REQUIRE(gamma > 0, "run_proxskip: gamma must be positive");
  PSB_REQUIRE(p > 0 && p <= 1, "SkipConfig: p must be in (0, 1]");
  PSB_REQUIRE(alpha > 0, "build_tv_recon: alpha must be positive");
  PSB_REQUIRE(n_inner >= 1, "TvProxState: inner_iters must be >= 1");
  PSB_REQUIRE(H >= 2 && W >= 2, "grad_forward: need a 2-D grid with both sides >= 2");
  PSB_REQUIRE(n >= 1 && n <= 65535, "proxskip run: batch size out of range");
  if (K <= 0) return PSB_OK;
  // PSB_DEBUG_HOST=1: host microseconds of this call's phases on stderr
  const char* dbg_host = std::getenv("PSB_DEBUG_HOST");
  const bool dbg_h = dbg_host && dbg_host[0] == '1';
  auto now_us = [] {
    return std::chrono::duration<double, std::micro>(
               std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  const double th0 = dbg_h ? now_us() : 0.0;
  double th1 = 0, th2 = 0, th3 = 0, th4 = 0;
  const int64_t HW = (int64_t)H * W;
  const int64_t qps = 6 * HW;
  // skip.py:64,70,74 -- scalars formed in double exactly as the reference does
  const double hcoef = gamma - gamma / p;
  const double weight = (gamma / p) * alpha;  // prox_g(u, gamma/p) -> tv_prox(u, step*alpha)
  const double pg = p / gamma;

  // Active lists + per-entry reprojection flags (tv.py:68-69 fires only on the
  // first call of this run whose weight differs from the stored last_weight).
  std::vector<int32_t> act;
  std::vector<uint8_t> rep;
  std::vector<int64_t> off(K + 1, 0);
  std::vector<uint8_t> seen(n, 0);
  act.reserve((size_t)(K * n * p * 1.2) + 16);
  rep.reserve((size_t)(K * n * p * 1.2) + 16);
  auto fired = [&](int64_t i) {
    act.push_back((int32_t)i);
    const double lw = last_weight[i];
    uint8_t r = 0;
    if (!seen[i]) {
      r = (!std::isnan(lw) && lw != weight) ? 1 : 0;
      seen[i] = 1;
    }
    rep.push_back(r);
    prox_count[i] += 1;
  };
  for (int k = 0; k < K; ++k) {  // (coins are sparse: eight at a time, zero words skipped)
    const uint8_t* row = coins_host + (int64_t)k * n;
    int64_t i = 0;
    for (; i + 8 <= n; i += 8) {
      uint64_t w8;
      std::memcpy(&w8, row + i, 8);
      while (w8) {  // (little-endian: byte j of the word is coin i + j)
        const int j = __builtin_ctzll(w8) >> 3;
        fired(i + j);
        w8 &= ~(0xFFull << (8 * j));
      }
    }
    for (; i < n; ++i)
      if (row[i]) fired(i);
    off[k + 1] = (int64_t)act.size();
  }
  for (int64_t i = 0; i < n; ++i)
    if (seen[i]) last_weight[i] = weight;

  std::vector<double> beta(n_inner, 0.0);
  if (accelerated) fista_betas(n_inner, beta.data());
  if (dbg_h) th1 = now_us();

  // Cluster-resident path (csrc/fgp_cluster.cu): 256 x 256 identity-fidelity
  // problems with an fp32 FGP.  Skipped iterations are deferred per problem
  // and executed in registers at the next prox call / the final flush.
  const char* no_cluster = std::getenv("PSB_NO_CLUSTER");
  // (an iterate history needs x materialised every iteration: streaming path)
  const bool use_cluster = fid.kind == 0 && dtf == PSB_F32 && cluster_shape_ok(H, W) &&
                           n_inner <= 1024 && !(no_cluster && no_cluster[0] == '1') &&
                           x_hist == nullptr && !fid.fista;
  PSB_REQUIRE(!fid.fista || (fid.xprev && fid.xbar), "fista: x_prev / xbar buffers missing");
  ChunkSync cs = chunks ? *chunks : ChunkSync{};
  PSB_REQUIRE(cs.ready == nullptr ||
                  (use_cluster && !use_graph && cs.done && cs.bounds && cs.n_chunks > 0 &&
                   cs.bounds[0] == 0 && cs.bounds[cs.n_chunks] == n),
              "streamed run: needs the cluster path (256x256, fp32 FGP, no graph) and a "
              "chunking that covers the batch");
  std::vector<int32_t> chunk_of;  // problem -> input chunk (streamed runs)
  if (cs.ready) {
    chunk_of.resize(n);
    for (int c = 0; c < cs.n_chunks; ++c) {
      PSB_REQUIRE(cs.bounds[c] <= cs.bounds[c + 1], "streamed run: chunk bounds not ascending");
      for (int64_t i = cs.bounds[c]; i < cs.bounds[c + 1]; ++i) chunk_of[i] = c;
    }
  }
  // FISTA's outer momentum (solvers.py:156-160): beta_k = (t_k - 1)/t_{k+1}, t_0 = 1
  std::vector<double> fbeta;
  if (fid.fista) {
    fbeta.resize(K);
    fista_betas(K, fbeta.data());
  }
  const size_t x_bytes = (size_t)n * HW * (dto == PSB_F32 ? 4 : 8);
  // Cluster path schedule: every problem's coin-fired iterations (CSR), its
  // re-projection flag, and the claim order of the device work queue
  // (common.cuh): by input chunk, then longest first (a prox call costs
  // n_inner cluster iterations, a skip iteration next to nothing).
  std::vector<int32_t> ev_off, ev_k, order;
  std::vector<float> qcost, qsuffix;
  std::vector<uint8_t> rep_p;
  std::vector<float> beta_f;
  int G = 0, NW = 0;
  // fp32 outer state runs on 8-CTA clusters (fgp_cluster8.cu: 16 px per
  // thread, q_k in registers, q_{k-1} and z in tensor memory): bit-identical to
  // the 16-CTA kernel, 15 % faster per SM, and 15 clusters tile 120 of the 148
  // SMs (seven 16-CTA clusters: 112).  fp64 outer state (mixed-precision single
  // problems) stays on the 16-CTA kernel.  PSB_CLUSTER8=0: 16-CTA clusters
  // only; PSB_CLUSTER8=2: 16-CTA clusters plus the 8-CTA clusters that fit in
  // the GPC space they leave (tests, comparisons).
  const char* c8 = std::getenv("PSB_CLUSTER8");
  const bool no8 = c8 && c8[0] == '0';
  const bool mix8 = c8 && c8[0] == '2';
  // (a batch smaller than the 16-CTA capacity runs on 16-CTA clusters: 16 SMs
  // per problem finish a problem 1.7x sooner than 8, and nothing waits)
  const bool use8 = dto == PSB_F32 && !no8 && !mix8 &&
                    (n > cluster_count() || (c8 && c8[0] == '1'));
  int G8 = 0;
  const int ccl = use8 ? 8 : 16;
  if (use_cluster) {
    ev_off.assign(n + 1, 0);
    for (size_t e = 0; e < act.size(); ++e) ev_off[act[e] + 1] += 1;
    for (int64_t i = 0; i < n; ++i) ev_off[i + 1] += ev_off[i];
    ev_k.resize(act.size());
    rep_p.assign(n, 0);
    std::vector<int32_t> fill(ev_off.begin(), ev_off.end() - 1);
    for (int k = 0; k < K; ++k)  // ascending k per problem
      for (int64_t e = off[k]; e < off[k + 1]; ++e) {
        const int32_t i = act[e];
        if (fill[i] == ev_off[i]) rep_p[i] = rep[e];
        ev_k[fill[i]++] = k;
      }
    // SMs the clusters leave idle run fgp_sm_run_kernel (one problem per SM,
    // L2-resident), launched as a programmatic dependent of the cluster
    // kernel so it is placed only after every cluster is resident.  (Not
    // inside a captured graph, and not for fp64 outer state.)  Test hooks:
    // PSB_NO_SMWORK=1 runs clusters only, PSB_SM_ONLY=1 SM workers only.
    const char* no_sm = std::getenv("PSB_NO_SMWORK");
    const char* sm_only = std::getenv("PSB_SM_ONLY");
    const bool only_sm = sm_only && sm_only[0] == '1' && dto == PSB_F32 && !use_graph;
    G = only_sm ? 0 : (int)std::min<int64_t>(n, use8 ? cluster8_count() : cluster_count());
    if (only_sm) {  // PSB_SM_WORKERS caps the worker count (profiling the 36-SM share)
      const char* nws = std::getenv("PSB_SM_WORKERS");
      const int cap = nws ? std::max(1, std::atoi(nws)) : sm_count();
      NW = (int)std::min<int64_t>(n, std::min(cap, sm_count()));
    }
    else if (n > G && dto == PSB_F32 && !use_graph && !(no_sm && no_sm[0] == '1')) {
      if (mix8) G8 = (int)std::min<int64_t>(n - G, std::max(0, cluster8_count() - 2 * G));
      NW = std::max(0, sm_count() - G * ccl - G8 * 8);
    }
    auto cost = [&](int32_t i) { return (float)(ev_off[i + 1] - ev_off[i]) * n_inner + 2.0f; };
    // claim order: by input chunk, then longest first, ties in index order --
    // a counting sort over (chunk, K - prox calls)
    {
      const int nch = cs.ready ? cs.n_chunks : 1;
      std::vector<int32_t> start((size_t)nch * (K + 1) + 1, 0);
      auto bucket = [&](int64_t i) {
        const int c = cs.ready ? chunk_of[i] : 0;
        return (size_t)c * (K + 1) + (size_t)(K - (ev_off[i + 1] - ev_off[i]));
      };
      for (int64_t i = 0; i < n; ++i) start[bucket(i) + 1] += 1;
      for (size_t bkt = 1; bkt < start.size(); ++bkt) start[bkt] += start[bkt - 1];
      order.resize(n);
      for (int64_t i = 0; i < n; ++i) order[start[bucket(i)]++] = (int32_t)i;
    }
    qcost.resize(n);
    qsuffix.assign(n + 1, 0.0f);
    for (int64_t i = 0; i < n; ++i) qcost[i] = cost(order[i]);
    for (int64_t i = n - 1; i >= 0; --i) qsuffix[i] = qsuffix[i + 1] + qcost[i];
    beta_f.resize(n_inner);
    for (int i = 0; i < n_inner; ++i) beta_f[i] = (float)beta[i];
  }

  // The whole schedule goes to the device as ONE buffer (one allocation, one
  // copy): the coin table (streaming path only), active lists, re-projection
  // flags and, for the cluster path, deferred-skip counts and the momentum table.
  std::vector<unsigned char> pack;
  auto put = [&](const void* src, size_t bytes) {
    const size_t at = (pack.size() + 15) & ~size_t(15);
    pack.resize(at + bytes);
    if (bytes) std::memcpy(pack.data() + at, src, bytes);
    return at;
  };
  const size_t o_coins = use_cluster ? 0 : put(coins_host, (size_t)K * n);
  const size_t o_act = use_cluster ? 0 : put(act.data(), act.size() * sizeof(int32_t));
  const size_t o_rep = use_cluster ? 0 : put(rep.data(), rep.size());
  size_t o_evo = 0, o_evk = 0, o_repp = 0, o_beta = 0, o_head = 0, o_stats = 0, o_order = 0,
         o_cost = 0, o_suffix = 0;
  if (use_cluster) {
    o_evo = put(ev_off.data(), ev_off.size() * sizeof(int32_t));
    o_evk = put(ev_k.data(), ev_k.size() * sizeof(int32_t));
    o_repp = put(rep_p.data(), rep_p.size());
    o_beta = put(beta_f.data(), beta_f.size() * sizeof(float));
    const uint64_t zeros[7] = {0, 0, 0, 0, 0, 0, 0};  // queue head + rate statistics start at 0
    o_head = put(zeros, sizeof(uint32_t));
    o_stats = put(zeros, 6 * sizeof(uint64_t));
    o_order = put(order.data(), order.size() * sizeof(int32_t));
    o_cost = put(qcost.data(), qcost.size() * sizeof(float));
    o_suffix = put(qsuffix.data(), qsuffix.size() * sizeof(float));
  }
  const size_t o_chunkof = chunk_of.empty() ? 0 : put(chunk_of.data(), chunk_of.size() * sizeof(int32_t));
  if (dbg_h) th2 = now_us();
  DevBuf d_sched;
  d_sched.st = user_stream;
  keep_pool_cached();
  PSB_CUDA(cudaMallocAsync(&d_sched.p, std::max<size_t>(pack.size(), 16), user_stream));
  // through a page-locked staging buffer kept across calls (a pageable source
  // makes cudaMemcpyAsync stage and wait, ~0.2 ms per call); an event guards
  // its reuse
  {
    static std::mutex mu;
    static void* stage = nullptr;
    static size_t stage_cap = 0;
    static cudaEvent_t stage_free = nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if (stage_free == nullptr) PSB_CUDA(cudaEventCreateWithFlags(&stage_free, cudaEventDisableTiming));
    else PSB_CUDA(cudaEventSynchronize(stage_free));
    if (pack.size() > stage_cap) {
      if (stage) cudaFreeHost(stage);
      stage = nullptr;
      stage_cap = 0;
      const size_t want = std::max<size_t>(2 * pack.size(), (size_t)1 << 20);
      if (cudaHostAlloc(&stage, want, cudaHostAllocDefault) == cudaSuccess) stage_cap = want;
      else (void)cudaGetLastError();
    }
    cudaStreamCaptureStatus cap_status = cudaStreamCaptureStatusNone;
    (void)cudaStreamIsCapturing(user_stream, &cap_status);
    if (stage_cap >= pack.size() && cap_status == cudaStreamCaptureStatusNone) {
      std::memcpy(stage, pack.data(), pack.size());
      PSB_CUDA(cudaMemcpyAsync(d_sched.p, stage, pack.size(), cudaMemcpyHostToDevice, user_stream));
      PSB_CUDA(cudaEventRecord(stage_free, user_stream));
    } else {
      // (pageable source: cudaMemcpyAsync stages `pack` before it returns)
      PSB_CUDA(cudaMemcpyAsync(d_sched.p, pack.data(), pack.size(), cudaMemcpyHostToDevice,
                               user_stream));
    }
  }
  unsigned char* dev = static_cast<unsigned char*>(d_sched.p);
  if (!chunk_of.empty()) cs.chunk_of = reinterpret_cast<const int32_t*>(dev + o_chunkof);
  const uint8_t* coins_d = dev + o_coins;
  const int32_t* act_d = reinterpret_cast<const int32_t*>(dev + o_act);
  const uint8_t* rep_d = dev + o_rep;
  auto i32 = [&](size_t o) { return reinterpret_cast<const int32_t*>(dev + o); };

  // Deblurring (separable blur, not FISTA): the gradient kernel also does the
  // pre step; a skipped iteration writes x-hat to the other of two x buffers
  // (the kernel still stages x halos), so x lives in x or x_alt by turns.
  const char* nf = std::getenv("PSB_NO_FUSED_PRE");  // the two-kernel form (tests)
  const bool no_fuse = nf && nf[0] == '1';
  const bool fuse_pre = fid.kind == 1 && fid.separable && !fid.fista && !use_cluster && !no_fuse;
  DevBuf d_xalt;
  d_xalt.st = user_stream;
  void* xcur = x;
  void* xalt = nullptr;
  if (fuse_pre) {
    PSB_CUDA(cudaMallocAsync(&d_xalt.p, (size_t)HW * (dto == PSB_F32 ? 4 : 8), user_stream));
    xalt = d_xalt.p;
  }

  if (dbg_h) th3 = now_us();
  CapturedRun cap;
  if (int rc0 = cap.begin(user_stream, use_graph != 0)) return rc0;
  cudaStream_t st = cap.st;

  // inside a capture an event record must be an explicit (external) graph node
  // to be usable for timing afterwards
  const unsigned rec_flags = use_graph ? cudaEventRecordExternal : cudaEventRecordDefault;
  IterClock clk;
  clk.begin(elapsed, K, st, use_graph != 0);
  // optional per-iteration timing of the FGP burst (bench roofline)
  std::vector<cudaEvent_t> fev;
  if (fgp_time) {
    fev.resize(2 * (size_t)K, nullptr);
    for (auto& e : fev) PSB_CUDA(cudaEventCreate(&e));
  }
  int rc = PSB_OK;
  if (use_cluster) {  // the whole segment in one launch
    if (fgp_time) cudaEventRecordWithFlags(fev[0], st, rec_flags);
    const float* beta_d = reinterpret_cast<const float*>(dev + o_beta);
    WorkQueue wq;
    wq.head = reinterpret_cast<unsigned int*>(dev + o_head);
    wq.stats = reinterpret_cast<unsigned long long*>(dev + o_stats);
    wq.order = i32(o_order);
    wq.cost = reinterpret_cast<const float*>(dev + o_cost);
    wq.suffix = reinterpret_cast<const float*>(dev + o_suffix);
    wq.n = (int)n;
    wq.clusters = use8 ? 0 : G;
    wq.clusters8 = use8 ? G : G8;
    if (NW > 0) rc = sm_prepare();  // module loaded before the clusters launch
    // (never in a streamed run: the synchronisation below would wait for
    // kernels that wait for copies the caller has not enqueued yet)
    const char* dbg = cs.ready ? nullptr : std::getenv("PSB_DEBUG_TIMES");
    cudaEvent_t d0 = nullptr, d1 = nullptr;
    if (dbg) {
      cudaEventCreate(&d0);
      cudaEventCreate(&d1);
      cudaEventRecord(d0, st);
    }
    if (rc == PSB_OK)
      rc = use8 ? cluster8_run(x, b, h, q, qps, wq, G, i32(o_evo), i32(o_evk), dev + o_repp, K,
                               n_inner, accelerated, nonneg, weight, gamma, hcoef, pg, 0.125,
                               beta_d, bad, cs, false, st)
                : cluster_run(dto, x, b, h, q, qps, wq, G, i32(o_evo), i32(o_evk), dev + o_repp, K,
                              n_inner, accelerated, nonneg, weight, gamma, hcoef, pg, 0.125, beta_d,
                              bad, cs, st);
    // The SM workers follow in the same stream as a programmatic dependent:
    // they are placed once every cluster CTA has started (griddepcontrol.
    // launch_dependents at the top of the cluster kernel), so they can never
    // take GPC space a 16-CTA cluster needs, and they finish only after the
    // clusters (griddepcontrol.wait at their end) -- no host gate, no second
    // stream.
    // mixed run: the extra 8-CTA clusters follow as a programmatic dependent
    // (placed after every 16-CTA cluster, before the SM workers)
    if (G8 > 0 && rc == PSB_OK)
      rc = cluster8_run(x, b, h, q, qps, wq, G8, i32(o_evo), i32(o_evk), dev + o_repp, K, n_inner,
                        accelerated, nonneg, weight, gamma, hcoef, pg, 0.125, beta_d, bad, cs,
                        G > 0, st);
    if (NW > 0 && rc == PSB_OK)
      rc = sm_run(x, b, h, q, qps, z, wq, NW, i32(o_evo), i32(o_evk), dev + o_repp, K, n_inner,
                  accelerated, nonneg, weight, gamma, hcoef, pg, 0.125, beta_d, bad, cs, G > 0, st);
    // queue statistics of this run for psb_queue_stats (page-locked copy,
    // valid once the stream has drained)
    if (rc == PSB_OK && !use_graph) {
      unsigned long long* hs = queue_stats_host();
      if (hs && cudaMemcpyAsync(hs, wq.stats, 6 * sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, st) != cudaSuccess)
        rc = fail(PSB_ERR_CUDA, "queue statistics copy failed");
    }
    if (dbg) {
      cudaEventRecord(d1, st);
      cudaDeviceSynchronize();
      float a = 0;
      cudaEventElapsedTime(&a, d0, d1);
      uint64_t stt[6] = {0, 0, 0, 0, 0, 0};
      cudaMemcpy(stt, wq.stats, sizeof(stt), cudaMemcpyDeviceToHost);
      fprintf(stderr,
              "[psb] %d 16-CTA clusters + %d 8-CTA clusters + %d sm workers: %.3f ms; cluster16 "
              "%.1f ns/unit over %llu units, cluster8 %.1f over %llu, worker %.1f over %llu\n",
              use8 ? 0 : G, use8 ? G : G8, NW, a, stt[1] ? (double)stt[0] / stt[1] : 0.0,
              (unsigned long long)stt[1], stt[5] ? (double)stt[4] / stt[5] : 0.0,
              (unsigned long long)stt[5], stt[3] ? (double)stt[2] / stt[3] : 0.0,
              (unsigned long long)stt[3]);
      cudaEventDestroy(d0);
      cudaEventDestroy(d1);
    }
    if (fgp_time) cudaEventRecordWithFlags(fev[1], st, rec_flags);
  }
  for (int k = 0; k < K && rc == PSB_OK && !use_cluster; ++k) {
    if (k > 0 && (rc = cap.tick(k - 1, K)) != PSB_OK) break;
    if (k > 0) clk.mark(k - 1, st);
    if (x_hist && k > 0 && rc == PSB_OK)  // iterate of outer iteration k-1 (device IterationLog)
      if (cudaMemcpyAsync(static_cast<char*>(x_hist) + (k - 1) * x_bytes, xcur, x_bytes,
                          cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        rc = fail(PSB_ERR_CUDA, "x history copy failed");
    const int ident = fid.kind == 0;
    if (fid.fista) {  // xbar = x + beta (x - x_prev); z = xbar - gamma g(xbar)
      rc = fista_extrap(dto, x, fid.xprev, fid.xbar, n * HW, fbeta[k], st);
      if (!rc && !ident)
        rc = blur_grad2d(dto, fid.xbar, b, fid.g, H, W, fid.taps2d, fid.taps1d, fid.ksize,
                         fid.separable, fid.scratch, st);
      if (!rc) rc = fista_pre(dto, dtf, fid.xbar, ident ? b : fid.g, ident, z, n * HW, gamma, st);
      if (rc) break;
    } else if (fuse_pre) {
      const int coin = coins_host[k] ? 1 : 0;
      rc = blur_grad_pre2d(dto, dtf, xcur, b, fid.g, H, W, fid.taps1d, fid.ksize, xalt, h, z,
                           gamma, hcoef, coin, bad, k, st);
      if (rc) break;
      if (!coin) std::swap(xcur, xalt);
    } else {
    if (!ident) {
      rc = blur_grad2d(dto, x, b, fid.g, H, W, fid.taps2d, fid.taps1d, fid.ksize, fid.separable,
                       fid.scratch, st);
      if (rc) break;
    }
    rc = proxskip_pre(dto, dtf, x, ident ? b : fid.g, ident, h, z, n, HW, coins_d + (int64_t)k * n,
                      gamma, hcoef, bad, k, st);
    }
    const int na = (int)(off[k + 1] - off[k]);
    if (rc || na == 0) continue;
    if (fgp_time) cudaEventRecordWithFlags(fev[2 * k], st, rec_flags);
    rc = fgp2d_run(dtf, z, HW, q, qps, act_d + off[k], na, weight, nullptr, 0, rep_d + off[k], H, W,
                   n_inner, accelerated, nonneg, 0.125, beta.data(), st);
    if (fgp_time) cudaEventRecordWithFlags(fev[2 * k + 1], st, rec_flags);
    if (rc == PSB_OK)
      rc = proxskip_post(dto, dtf, xcur, ident ? b : fid.g, ident, fid.fista ? nullptr : h, z, q, qps,
                         act_d + off[k], na, H, W, n_inner, nonneg, gamma, pg, bad, k, st);
  }

  if (dbg_h) {
    th4 = now_us();
    fprintf(stderr, "[psb host] active lists %.0f us, schedule %.0f us, pack + copy %.0f us, launches %.0f us\n",
            th1 - th0, th2 - th1, th3 - th2, th4 - th3);
  }
  if (x_hist && rc == PSB_OK)
    if (cudaMemcpyAsync(static_cast<char*>(x_hist) + (size_t)(K - 1) * x_bytes, xcur, x_bytes,
                        cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      rc = fail(PSB_ERR_CUDA, "x history copy failed");
  if (xcur != x && rc == PSB_OK &&
      cudaMemcpyAsync(x, xcur, x_bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    rc = fail(PSB_ERR_CUDA, "x copy-back failed");
  if (rc == PSB_OK) clk.mark(K - 1, st);
  // The schedule buffer is released stream-ordered after the run (DevBuf).
  rc = cap.end(rc);
  if (fgp_time) {
    cudaError_t e = cudaStreamSynchronize(use_graph ? user_stream : st);
    if (rc == PSB_OK && e != cudaSuccess)
      rc = fail(PSB_ERR_CUDA, std::string("run: ") + cudaGetErrorString(e));
    for (int k = 0; k < K; ++k) {
      float ms = 0.f;
      fgp_time[k] = 0.0;
      // (cluster path: one launch for the segment, its time in fgp_time[0])
      if (rc == PSB_OK && (use_cluster ? k == 0 : off[k + 1] > off[k])) {
        if (cudaEventElapsedTime(&ms, fev[2 * k], fev[2 * k + 1]) == cudaSuccess)
          fgp_time[k] = ms * 1e-3;
        else
          fgp_time[k] = std::nan(""), (void)cudaGetLastError();
      }
    }
    for (auto e : fev) cudaEventDestroy(e);
  }
  if (elapsed) {
    cudaError_t e = cudaStreamSynchronize(use_graph ? user_stream : st);
    if (rc == PSB_OK && e != cudaSuccess)
      rc = fail(PSB_ERR_CUDA, std::string("run: ") + cudaGetErrorString(e));
  }
  clk.finish(elapsed, use_graph ? user_stream : st, rc == PSB_OK);
  return rc;
}

}  // namespace psb

extern "C" int psb_queue_stats(double* out6) {
  PSB_REQUIRE(out6 != nullptr, "queue_stats: output missing");
  const unsigned long long* hs = psb::queue_stats_host();
  for (int i = 0; i < 6; ++i) out6[i] = hs ? (double)hs[i] : 0.0;
  return PSB_OK;
}

extern "C" int psb_proxskip_denoise_run(int dtype_outer, int dtype_fgp, void* x, const void* b,
                                        void* h, void* z, void* q, int64_t n, int H, int W,
                                        const uint8_t* coins_host, int K, double gamma, double p,
                                        double alpha, int n_inner, int accelerated, int nonneg,
                                        double* last_weight_host, int64_t* prox_count_host,
                                        int32_t* bad_iter, int use_graph, double* elapsed_host,
                                        double* fgp_time_host, void* x_hist, int algo, void* aux,
                                        void* stream) {
  psb::Fidelity fid;
  fid.fista = algo == 1;
  fid.xprev = aux;
  fid.xbar = aux ? static_cast<char*>(aux) + (size_t)n * H * W * (dtype_outer == PSB_F32 ? 4 : 8)
                 : nullptr;
  return psb::proxskip_tv_run(fid, dtype_outer, dtype_fgp, x, b, h, z, q, n, H, W, coins_host, K,
                              gamma, p, alpha, n_inner, accelerated, nonneg, last_weight_host,
                              prox_count_host, bad_iter, use_graph, elapsed_host, fgp_time_host,
                              x_hist, psb::as_stream(stream));
}

extern "C" int psb_proxskip_denoise_run_streamed(
    int dtype_outer, int dtype_fgp, void* x, const void* b, void* h, void* z, void* q, int64_t n,
    int H, int W, const uint8_t* coins_host, int K, double gamma, double p, double alpha,
    int n_inner, int accelerated, int nonneg, double* last_weight_host, int64_t* prox_count_host,
    int32_t* bad_iter, const int32_t* ready, int32_t* done, const int64_t* bounds_host,
    int n_chunks, void* stream) {
  psb::Fidelity fid;
  psb::ChunkSync cs;
  cs.ready = ready;
  cs.done = done;
  cs.bounds = bounds_host;
  cs.n_chunks = n_chunks;
  return psb::proxskip_tv_run(fid, dtype_outer, dtype_fgp, x, b, h, z, q, n, H, W, coins_host, K,
                              gamma, p, alpha, n_inner, accelerated, nonneg, last_weight_host,
                              prox_count_host, bad_iter, 0, nullptr, nullptr, nullptr,
                              psb::as_stream(stream), &cs);
}

// Stream memory operations (driver API, resolved at run time through the
// runtime's entry-point query so the library does not link libcuda).
namespace {
typedef int (*StreamValueFn)(void* stream, unsigned long long addr, uint32_t value,
                             unsigned int flags);
StreamValueFn stream_fn(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<StreamValueFn>(fn);
}
}  // namespace

extern "C" int psb_stream_memops_supported(int* out) {
  int dev = 0, v = 0;
  *out = 0;
  PSB_CUDA(cudaGetDevice(&dev));
  // CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_MEM_OPS_V1 (driver attribute 92) is
  // not exposed by the runtime enum; probe by resolving the entry points
  (void)v;
  *out = stream_fn("cuStreamWriteValue32") != nullptr && stream_fn("cuStreamWaitValue32") != nullptr;
  return PSB_OK;
}

extern "C" int psb_stream_write_u32(void* stream, void* dptr, uint32_t value) {
  static StreamValueFn fn = stream_fn("cuStreamWriteValue32");
  if (!fn) return psb::fail(PSB_ERR_CUDA, "cuStreamWriteValue32 unavailable");
  // CU_STREAM_WRITE_VALUE_DEFAULT: a memory fence precedes the write, so the
  // chunk copied before it on this stream is visible when the flag is
  if (fn(stream, reinterpret_cast<unsigned long long>(dptr), value, 0) != 0)
    return psb::fail(PSB_ERR_CUDA, "cuStreamWriteValue32 failed");
  return PSB_OK;
}

extern "C" int psb_stream_wait_geq_u32(void* stream, void* dptr, uint32_t value) {
  static StreamValueFn fn = stream_fn("cuStreamWaitValue32");
  if (!fn) return psb::fail(PSB_ERR_CUDA, "cuStreamWaitValue32 unavailable");
  // CU_STREAM_WAIT_VALUE_GEQ = 0x0: (int32_t)(*addr - value) >= 0
  if (fn(stream, reinterpret_cast<unsigned long long>(dptr), value, 0x0) != 0)
    return psb::fail(PSB_ERR_CUDA, "cuStreamWaitValue32 failed");
  return PSB_OK;
}

// Chunked host<->device streaming of a batch (the e2e path of
// run_proxskip_batched): one call enqueues every chunk's copy and its stream
// memory operation, so the host spends microseconds, not a Python round trip,
// per chunk.  H2D: copy chunk c, then ready[c] = 1 (fenced write).  D2H (on
// its own stream, so results leave while later inputs still arrive): wait
// until done[c] >= unit * (items in chunk c), then copy chunk c back.
extern "C" int psb_chunked_h2d(void* dst, const void* src_host, int64_t item_bytes,
                               const int64_t* bounds, int n_chunks, int32_t* ready, void* stream) {
  PSB_REQUIRE(item_bytes > 0 && n_chunks >= 0 && bounds, "chunked h2d: bad sizes");
  static StreamValueFn wr = stream_fn("cuStreamWriteValue32");
  if (!wr) return psb::fail(PSB_ERR_CUDA, "cuStreamWriteValue32 unavailable");
  auto st = psb::as_stream(stream);
  for (int c = 0; c < n_chunks; ++c) {
    const int64_t lo = bounds[c], k = bounds[c + 1] - bounds[c];
    PSB_REQUIRE(k >= 0, "chunked h2d: bounds not ascending");
    PSB_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + lo * item_bytes,
                             static_cast<const char*>(src_host) + lo * item_bytes,
                             (size_t)(k * item_bytes), cudaMemcpyHostToDevice, st));
    if (wr(stream, reinterpret_cast<unsigned long long>(ready + c), 1u, 0) != 0)
      return psb::fail(PSB_ERR_CUDA, "cuStreamWriteValue32 failed");
  }
  return PSB_OK;
}

extern "C" int psb_chunked_d2h(void* dst_host, const void* src, int64_t item_bytes,
                               const int64_t* bounds, int n_chunks, const int32_t* done,
                               uint32_t unit, void* stream) {
  PSB_REQUIRE(item_bytes > 0 && n_chunks >= 0 && bounds, "chunked d2h: bad sizes");
  static StreamValueFn wt = stream_fn("cuStreamWaitValue32");
  if (!wt) return psb::fail(PSB_ERR_CUDA, "cuStreamWaitValue32 unavailable");
  auto st = psb::as_stream(stream);
  for (int c = 0; c < n_chunks; ++c) {
    const int64_t lo = bounds[c], k = bounds[c + 1] - bounds[c];
    PSB_REQUIRE(k >= 0, "chunked d2h: bounds not ascending");
    if (wt(stream, reinterpret_cast<unsigned long long>(done + c), unit * (uint32_t)k, 0x0) != 0)
      return psb::fail(PSB_ERR_CUDA, "cuStreamWaitValue32 failed");
    PSB_CUDA(cudaMemcpyAsync(static_cast<char*>(dst_host) + lo * item_bytes,
                             static_cast<const char*>(src) + lo * item_bytes,
                             (size_t)(k * item_bytes), cudaMemcpyDeviceToHost, st));
  }
  return PSB_OK;
}

// Peer memory for the config-5 slab exchange: a rank exports
// its receive rings / flags with a CUDA IPC handle, its z-neighbours map them
// and deposit halo planes there directly (kernel stores or copies over
// NVLink), ordered by stream memory operations on the flags.
extern "C" int psb_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  PSB_REQUIRE(bytes >= 0, "psb_copy_async: negative size");
  if (bytes == 0) return PSB_OK;
  PSB_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, psb::as_stream(stream)));
  return PSB_OK;
}

extern "C" int psb_ipc_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }

// dptr may point inside a larger allocation (torch's caching allocator hands
// out sub-blocks of its segments): the handle names the allocation, *offset
// is dptr's distance from its base, added back by the importer.
extern "C" int psb_ipc_get_handle(const void* dptr, void* handle_out, int64_t* offset) {
  typedef int (*RangeFn)(unsigned long long* base, size_t* size, unsigned long long dptr);
  static RangeFn range = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<RangeFn>(fn);
  }();
  if (!range) return psb::fail(PSB_ERR_CUDA, "cuMemGetAddressRange unavailable");
  unsigned long long base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<unsigned long long>(dptr)) != 0)
    return psb::fail(PSB_ERR_CUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  PSB_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle_out, &h, sizeof(h));
  *offset = (int64_t)(reinterpret_cast<unsigned long long>(dptr) - base);
  return PSB_OK;
}

extern "C" int psb_ipc_open_handle(const void* handle, void** dptr_out) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  PSB_CUDA(cudaIpcOpenMemHandle(dptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return PSB_OK;
}

extern "C" int psb_ipc_close(void* dptr) {
  PSB_CUDA(cudaIpcCloseMemHandle(dptr));
  return PSB_OK;
}

extern "C" int psb_proxskip_deblur_run(int dtype_outer, int dtype_fgp, void* x, const void* b,
                                       void* h, void* z, void* q, void* g, void* scratch, int H,
                                       int W, const double* taps2d, const double* taps1d,
                                       int ksize, int separable, const uint8_t* coins_host, int K,
                                       double gamma, double p, double alpha, int n_inner,
                                       int accelerated, int nonneg, double* last_weight_host,
                                       int64_t* prox_count_host, int32_t* bad_iter, int use_graph,
                                       double* elapsed_host, double* fgp_time_host, void* x_hist,
                                       int algo, void* aux, void* stream) {
  psb::Fidelity fid;
  fid.kind = 1;
  fid.fista = algo == 1;
  fid.xprev = aux;
  fid.xbar = aux ? static_cast<char*>(aux) + (size_t)H * W * (dtype_outer == PSB_F32 ? 4 : 8)
                 : nullptr;
  fid.taps2d = taps2d;
  fid.taps1d = taps1d;
  fid.ksize = ksize;
  fid.separable = separable;
  fid.g = g;
  fid.scratch = scratch;
  return psb::proxskip_tv_run(fid, dtype_outer, dtype_fgp, x, b, h, z, q, 1, H, W, coins_host, K,
                              gamma, p, alpha, n_inner, accelerated, nonneg, last_weight_host,
                              prox_count_host, bad_iter, use_graph, elapsed_host, fgp_time_host,
                              x_hist, psb::as_stream(stream));
}

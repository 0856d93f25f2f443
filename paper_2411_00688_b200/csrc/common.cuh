// Shared device/host helpers for libpsb200 (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>
#include <cmath>
#include <algorithm>
#include <utility>
#include <mutex>
#include <tuple>

#include "../../include/psb200.h"

namespace psb {

// ---- error reporting (psb_last_error) ---------------------------------------
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);

#define PSB_CUDA(call)                                                             \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return ::psb::fail(PSB_ERR_CUDA, std::string(#call) + ": " +                 \
                                           cudaGetErrorString(e_));                \
  } while (0)

#define PSB_LAUNCHED(name)                                                         \
  do {                                                                             \
    cudaError_t e_ = cudaGetLastError();                                           \
    if (e_ != cudaSuccess)                                                         \
      return ::psb::fail(PSB_ERR_CUDA, std::string(name) + " launch: " +           \
                                           cudaGetErrorString(e_));                \
  } while (0)

#define PSB_CHECK(call)                                                            \
  do {                                                                             \
    const int rc_ = (call);                                                        \
    if (rc_ != PSB_OK) return rc_;                                                 \
  } while (0)

#define PSB_REQUIRE(cond, msg)                                                     \
  do {                                                                             \
    if (!(cond)) return ::psb::fail(PSB_ERR_VALUE, msg);                           \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();

// ---- arithmetic -------------------------------------------------------------
// The double instantiation must round every operation separately, exactly like
// numpy (SURVEY 8(c+)): use the _rn intrinsics, which ptxas never contracts
// into FMA.  The float instantiation is the production path and may contract.
template <class T> struct Ar;

template <> struct Ar<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double sqrt(double a) { return __dsqrt_rn(a); }
  // proximal.py:19-21: r * q / max(r, |q|), |q| = sqrt(a*a + b*b), no FMA.
  static __device__ __forceinline__ double ball_scale(double a, double b, double r) {
    double m = __dsqrt_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)));
    return __ddiv_rn(r, fmax(r, m));
  }
  static __device__ __forceinline__ double ball_scale3(double a, double b, double c, double r) {
    double m = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)), __dmul_rn(c, c)));
    return __ddiv_rn(r, fmax(r, m));
  }
};

// fp32 ball projections use the radius r * kBallShrink: rsqrt.approx (<= ~2^-22
// relative error) plus the roundings of the scale and of q' = a * s could
// otherwise leave |q'| a few ulp above r, and the reference's feasibility test
// (tv.py:98-100, 1e-10 slack) would reject the fp32 dual iterate.  With the
// 2^-20 shrink |q'| <= r holds for every input; the projected duals move by
// < 1e-6 relative, far inside the fp32 parity tolerance.  (fp64 projections are
// the reference's exact formula.)
constexpr float kBallShrink = 1.0f - 0x1p-20f;

template <> struct Ar<float> {
  static __device__ __forceinline__ float add(float a, float b) { return a + b; }
  static __device__ __forceinline__ float sub(float a, float b) { return a - b; }
  static __device__ __forceinline__ float mul(float a, float b) { return a * b; }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
  static __device__ __forceinline__ float sqrt(float a) { return __fsqrt_rn(a); }
  // Same projection with one MUFU (no denormal rescaling): min(1, r/|q|).
  static __device__ __forceinline__ float rsq(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
  }
  static __device__ __forceinline__ float ball_scale(float a, float b, float r) {
    return fminf(1.0f, (r * kBallShrink) * rsq(fmaf(a, a, b * b)));
  }
  static __device__ __forceinline__ float ball_scale3(float a, float b, float c, float r) {
    return fminf(1.0f, (r * kBallShrink) * rsq(fmaf(a, a, fmaf(b, b, c * c))));
  }
};

// ---- vector loads -----------------------------------------------------------
template <class T, int V> struct Vec { T v[V]; };

template <class T, int V>
__device__ __forceinline__ void ldv(T (&d)[V], const T* p) {
  if constexpr (sizeof(T) * V == 16) {
    float4 r = __ldg(reinterpret_cast<const float4*>(p));
    const T* s = reinterpret_cast<const T*>(&r);
#pragma unroll
    for (int i = 0; i < V; ++i) d[i] = s[i];
  } else if constexpr (sizeof(T) * V == 8) {
    float2 r = __ldg(reinterpret_cast<const float2*>(p));
    const T* s = reinterpret_cast<const T*>(&r);
#pragma unroll
    for (int i = 0; i < V; ++i) d[i] = s[i];
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) d[i] = __ldg(p + i);
  }
}

// Vector store (the kernels never re-read what they write in the same launch,
// so all loads above may use the read-only path).
// Vector load without the read-only path (shared memory, or data written
// earlier by the same kernel).
template <class T, int V>
__device__ __forceinline__ void ldv_s(T (&d)[V], const T* p) {
  if constexpr (sizeof(T) * V == 16) {
    const float4 r = *reinterpret_cast<const float4*>(p);
    const T* s = reinterpret_cast<const T*>(&r);
#pragma unroll
    for (int i = 0; i < V; ++i) d[i] = s[i];
  } else if constexpr (sizeof(T) * V == 8) {
    const float2 r = *reinterpret_cast<const float2*>(p);
    const T* s = reinterpret_cast<const T*>(&r);
#pragma unroll
    for (int i = 0; i < V; ++i) d[i] = s[i];
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) d[i] = p[i];
  }
}

template <class T, int V>
__device__ __forceinline__ void stv(T* p, const T (&s)[V]) {
  if constexpr (sizeof(T) * V == 16) {
    float4 r;
    T* d = reinterpret_cast<T*>(&r);
#pragma unroll
    for (int i = 0; i < V; ++i) d[i] = s[i];
    *reinterpret_cast<float4*>(p) = r;
  } else if constexpr (sizeof(T) * V == 8) {
    float2 r;
    T* d = reinterpret_cast<T*>(&r);
#pragma unroll
    for (int i = 0; i < V; ++i) d[i] = s[i];
    *reinterpret_cast<float2*>(p) = r;
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) p[i] = s[i];
  }
}

template <class T> __device__ __forceinline__ bool finite(T v) { return isfinite(v); }

__device__ __forceinline__ bool same_bits(float a, float b) {
  return __float_as_uint(a) == __float_as_uint(b);
}
__device__ __forceinline__ bool same_bits(double a, double b) {
  return __double_as_longlong(a) == __double_as_longlong(b);
}

// one skipped ProxSkip iteration of the identity fidelity (skip.py:68)
template <class T>
__device__ __forceinline__ T skip_step(T x, T b, T h, T g) {
  using A = Ar<T>;
  return A::add(A::sub(x, A::mul(g, A::sub(x, b))), A::mul(g, h));
}

// m skipped ProxSkip iterations of the identity fidelity,
// x <- (x - g (x - b)) + g h (skip.py:68), with the reference's roundings.
// The update is a fixed map of x (b, h, g do not change across a run of
// skips), so once it returns its input bit for bit every later step does too
// and the loop stops there: the result is exactly the m-step result.  A
// non-finite x stays non-finite under the map, so only the final x is
// tested; *first_bad = min(*first_bad, kfirst + first non-finite step).
template <class T>
__device__ __forceinline__ T skip_chain_px(T x, T b, T h, T g, int m, int kfirst,
                                           int* first_bad) {
  using A = Ar<T>;
  const T x0 = x;
  for (int s = 0; s < m; ++s) {
    const T xn = A::add(A::sub(x, A::mul(g, A::sub(x, b))), A::mul(g, h));
    if (same_bits(xn, x)) break;
    x = xn;
  }
  if (m > 0 && !finite(x)) {
    T xr = x0;
    for (int s = 0; s < m; ++s) {
      xr = A::add(A::sub(xr, A::mul(g, A::sub(xr, b))), A::mul(g, h));
      if (!finite(xr)) {
        *first_bad = min(*first_bad, kfirst + s);
        break;
      }
    }
  }
  return x;
}

// ---- host->device chunk streaming (run drivers) ------------------------------
// The run kernels can start before their inputs have arrived: problem p's
// chunk c = p / chunk is ready once ready[c] != 0 (written by the copy stream
// after the chunk's H2D copy, cuStreamWriteValue32), and every finished
// problem adds 16 to done[c] (a cluster: 1 per CTA; an SM worker: 16), which
// the copy stream waits for (cuStreamWaitValue32 >= 16 * problems) before the
// chunk's D2H copy.  ready[n_chunks] is an error flag: a wait that times out
// (20 s) sets it instead of hanging the device.
struct ChunkSync {
  const int32_t* ready = nullptr;  // null: inputs already resident
  int32_t* done = nullptr;
  const int32_t* chunk_of = nullptr;  // [n] chunk index of each problem (device)
  const int64_t* bounds = nullptr;    // [n_chunks + 1] chunk starts (HOST, driver only)
  int n_chunks = 0;
};

__device__ __forceinline__ void chunk_wait(const ChunkSync& cs, int p) {
  if (cs.ready == nullptr) return;
  const int32_t* f = cs.ready + cs.chunk_of[p];
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  const int32_t* err = cs.ready + cs.n_chunks;
  for (;;) {
    int v, e;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    if (v) return;
    // a wait that already timed out elsewhere aborts every later wait at once
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(e) : "l"(err) : "memory");
    if (e) return;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 20000000000ull) {
      atomicExch(const_cast<int32_t*>(cs.ready) + cs.n_chunks, 1);
      return;
    }
    __nanosleep(2000);
  }
}

// after this thread's writes of problem p: (all threads) fence; one thread adds
__device__ __forceinline__ void chunk_done(const ChunkSync& cs, int p, int add, bool leader) {
  if (cs.done == nullptr) return;
  __threadfence();
  __syncthreads();
  if (leader) atomicAdd(cs.done + cs.chunk_of[p], add);
}

// ---- dynamic problem queue (run drivers, configs 1 / 4) ----------------------
// The cluster run kernel and the SM-worker kernel claim problems from ONE
// device queue: `order` lists the problems by input chunk, then longest first
// (cost = prox calls x n_inner + 2), and `head` is the next position.  A
// cluster claims with one atomicAdd.  An SM worker (about 20x slower per
// problem than a 16-SM cluster) claims position i only while its expected
// time for that problem does not exceed the clusters' expected time for the
// rest of the queue -- both rates measured on the fly (globaltimer ns per cost
// unit of finished problems, `stats`), so no cost ratio is assumed and the run
// ends with the clusters, not with an SM worker's last problem.  Which kernel
// runs a problem never changes a result (the two kernels are bit-identical).
struct WorkQueue {
  unsigned int* head = nullptr;         // next position of `order` to claim (zero at run start)
  unsigned long long* stats = nullptr;  // [6]: ns, cost of the 16-CTA clusters, the SM workers, the 8-CTA clusters
  const int32_t* order = nullptr;       // [n] problem indices in claim order
  const float* cost = nullptr;          // [n] cost units of order[i]
  const float* suffix = nullptr;        // [n + 1] sum of cost[i .. n)
  int n = 0;
  int clusters = 0;                     // 16-CTA clusters claiming beside the SM workers
  int clusters8 = 0;                    // 8-CTA clusters
};

__device__ __forceinline__ uint64_t gtimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// cluster side: next position, or -1 when the queue is empty
__device__ __forceinline__ int wq_claim(const WorkQueue& q) {
  const unsigned i = atomicAdd(q.head, 1u);
  return i < (unsigned)q.n ? (int)i : -1;
}

// SM-worker side (see above); -1: nothing worth taking
__device__ __forceinline__ int wq_claim_worker(const WorkQueue& q) {
  for (;;) {
    unsigned i;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(i) : "l"(q.head) : "memory");
    if (i >= (unsigned)q.n) return -1;
    if (q.clusters + q.clusters8 > 0) {
      unsigned long long s[6];
#pragma unroll
      for (int k = 0; k < 6; ++k)
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(s[k]) : "l"(q.stats + k) : "memory");
      // the clusters' capacity in cost units per ns, each kind at its measured
      // rate (a kind without a finished problem yet: the other's, an 8-CTA
      // cluster counting as half a 16-CTA cluster)
      double r16 = s[0] > 0 ? (double)s[1] / (double)s[0] : 0.0;
      double r8 = s[4] > 0 ? (double)s[5] / (double)s[4] : 0.0;
      if (r16 == 0.0) r16 = 2.0 * r8;
      if (r8 == 0.0) r8 = 0.5 * r16;
      const double cap = q.clusters * r16 + q.clusters8 * r8;
      if (cap > 0.0 && s[3] > 0) {
        const double t_worker = (double)s[2] / (double)s[3] * (double)q.cost[i];
        const double t_rest = (double)q.suffix[i + 1] / cap;
        if (t_worker > t_rest) return -1;
      }
    }
    if (atomicCAS(q.head, i, i + 1) == i) return (int)i;
  }
}

// a finished problem's time and cost (role 0: 16-CTA cluster, 1: SM worker, 2: 8-CTA cluster)
__device__ __forceinline__ void wq_record(const WorkQueue& q, int role, int pos, uint64_t t0) {
  atomicAdd(q.stats + 2 * role, (unsigned long long)(gtimer_ns() - t0));
  atomicAdd(q.stats + 2 * role + 1, (unsigned long long)q.cost[pos]);
}

// ---- stream-ordered allocations stay cached ------------------------------------
// The default memory pool returns freed blocks to the OS at the next
// synchronisation (release threshold 0), so every cudaMallocAsync of a run
// driver (schedule, scratch) paid a fresh allocation, ~0.2 ms.  Raise the
// threshold once per device: freed blocks stay in the pool for the next call.
inline void keep_pool_cached() {
  static std::mutex mu;
  static std::vector<int> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  std::lock_guard<std::mutex> lock(mu);
  for (int d : done)
    if (d == dev) return;
  cudaMemPool_t pool = nullptr;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    (void)cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  (void)cudaGetLastError();
  done.push_back(dev);
}

// ---- kernel attributes, set once ---------------------------------------------
// cudaFuncSetAttribute on a function that has launches in flight can make the
// driver wait for them, which serialises back-to-back launches of a long
// kernel; set each (device, kernel, attribute) value once per process.
inline int func_attr(const void* fn, cudaFuncAttribute attr, int value) {
  static std::mutex mu;
  static std::vector<std::tuple<int, const void*, int, int>> done;  // device, fn, attr, value
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  std::tuple<int, const void*, int, int>* hit = nullptr;
  for (auto& t : done)
    if (std::get<0>(t) == dev && std::get<1>(t) == fn && std::get<2>(t) == (int)attr) hit = &t;
  // a larger dynamic shared memory limit already covers a smaller request
  if (hit && (std::get<3>(*hit) == value ||
              (attr == cudaFuncAttributeMaxDynamicSharedMemorySize && std::get<3>(*hit) > value)))
    return PSB_OK;
  const cudaError_t e = cudaFuncSetAttribute(fn, attr, value);
  if (e != cudaSuccess)
    return fail(PSB_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  if (hit)
    std::get<3>(*hit) = value;
  else
    done.emplace_back(dev, fn, (int)attr, value);
  return PSB_OK;
}
template <class K>
int func_attr(K* kern, cudaFuncAttribute attr, int value) {
  return func_attr(reinterpret_cast<const void*>(kern), attr, value);
}

// ---- optional CUDA-graph capture of a run driver's launch sequence ---------
// Capture needs a capturable (non-legacy) stream: the run is enqueued on a
// private stream ordered after the caller's stream, captured, instantiated,
// launched once, and the caller's stream is ordered after it.  Without
// use_graph the launches go to the caller's stream directly.
struct CapturedRun {
  cudaStream_t user = nullptr, st = nullptr, priv = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  bool graph = false;
  int begin(cudaStream_t user_stream, bool use_graph) {
    user = st = user_stream;
    graph = use_graph;
    if (!graph) return PSB_OK;
    PSB_CUDA(cudaStreamCreateWithFlags(&priv, cudaStreamNonBlocking));
    PSB_CUDA(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
    PSB_CUDA(cudaEventCreateWithFlags(&ev_out, cudaEventDisableTiming));
    PSB_CUDA(cudaEventRecord(ev_in, user));
    PSB_CUDA(cudaStreamWaitEvent(priv, ev_in, 0));
    st = priv;
    PSB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    return PSB_OK;
  }
  // Chunked capture: every `chunk` outer iterations the graph captured so far
  // is instantiated and launched, and capture restarts on the same stream, so
  // the host builds chunk c+1 while the device runs chunk c (one graph of a
  // whole 1000-iteration run cost ~17 ms of capture + instantiation before
  // the first kernel ran).  Call after outer iteration k was enqueued.
  int chunk = 32;
  int tick(int k, int K) {
    if (!graph || (k + 1) % chunk != 0 || k + 1 >= K) return PSB_OK;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaError_t e = cudaStreamEndCapture(st, &g);
    int rc = PSB_OK;
    if (e != cudaSuccess)
      rc = fail(PSB_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    if (rc == PSB_OK && (e = cudaGraphInstantiate(&exec, g, 0)) != cudaSuccess)
      rc = fail(PSB_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    if (rc == PSB_OK && (e = cudaGraphLaunch(exec, st)) != cudaSuccess)
      rc = fail(PSB_ERR_CUDA, std::string("graph launch: ") + cudaGetErrorString(e));
    if (exec) cudaGraphExecDestroy(exec);
    if (g) cudaGraphDestroy(g);
    // capture restarts even after an error: end() always ends one capture
    e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    if (rc == PSB_OK && e != cudaSuccess)
      rc = fail(PSB_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    return rc;
  }
  // ends the capture (always), launches the graph if rc is still OK
  int end(int rc) {
    if (!graph) return rc;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaError_t e = cudaStreamEndCapture(st, &g);
    if (rc == PSB_OK && e != cudaSuccess)
      rc = fail(PSB_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    if (rc == PSB_OK && (e = cudaGraphInstantiate(&exec, g, 0)) != cudaSuccess)
      rc = fail(PSB_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    if (rc == PSB_OK && (e = cudaGraphLaunch(exec, st)) != cudaSuccess)
      rc = fail(PSB_ERR_CUDA, std::string("graph launch: ") + cudaGetErrorString(e));
    cudaEventRecord(ev_out, st);
    cudaStreamWaitEvent(user, ev_out, 0);
    if (exec) cudaGraphExecDestroy(exec);  // deferred by the runtime until the launch completes
    if (g) cudaGraphDestroy(g);
    cudaEventDestroy(ev_in);
    cudaEventDestroy(ev_out);
    cudaStreamDestroy(priv);
    (void)cudaGetLastError();
    return rc;
  }
};

// ---- sparse per-iteration device clock of the run drivers ------------------
// An event record is a graph node that costs several microseconds inside a
// captured run -- as much as a whole 256^2 iteration -- so the drivers record
// the device clock at most ~64 times per run (every `stride`-th iteration and
// the last one) and fill elapsed[k] in between by linear interpolation; the
// final value (the run's total device time) is exact.
struct IterClock {
  std::vector<cudaEvent_t> ev;  // ev[0] = start, ev[j + 1] = after iteration at[j]
  std::vector<int> at;
  int K = 0, stride = 1;
  unsigned flags = 0;
  bool on = false;
  void begin(double* out, int K_, cudaStream_t st, bool graph) {
    on = out != nullptr && K_ > 0;
    if (!on) return;
    K = K_;
    stride = K > 64 ? (K + 63) / 64 : 1;
    flags = graph ? cudaEventRecordExternal : cudaEventRecordDefault;
    ev.resize(1);
    cudaEventCreate(&ev[0]);
    cudaEventRecordWithFlags(ev[0], st, flags);
  }
  void mark(int k, cudaStream_t st) {  // after iteration k was enqueued
    if (!on || ((k + 1) % stride != 0 && k != K - 1)) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecordWithFlags(e, st, flags);
    ev.push_back(e);
    at.push_back(k);
  }
  void finish(double* out, cudaStream_t sync_stream, bool ok) {
    if (!on) return;
    cudaStreamSynchronize(sync_stream);
    std::vector<double> t(at.size(), std::nan(""));
    for (size_t j = 0; j < at.size(); ++j) {
      float ms = 0.f;
      if (ok && cudaEventElapsedTime(&ms, ev[0], ev[j + 1]) == cudaSuccess)
        t[j] = ms * 1e-3;
      else
        (void)cudaGetLastError();
    }
    int k0 = -1;
    double t0 = 0.0;
    for (size_t j = 0; j < at.size(); ++j) {
      const int k1 = at[j];
      for (int k = k0 + 1; k <= k1; ++k) out[k] = t0 + (t[j] - t0) * (k - k0) / (double)(k1 - k0);
      k0 = k1;
      t0 = t[j];
    }
    for (int k = k0 + 1; k < K; ++k) out[k] = std::nan("");  // run stopped early
    for (auto e : ev) cudaEventDestroy(e);
    ev.clear();
    at.clear();
  }
};

// ---- programmatic dependent launch -------------------------------------------
// Every kernel of a launch chain starts with pdl_enter(): it lets the NEXT
// kernel in the stream begin launching right away and then waits until the
// previous kernel has completed and its writes are visible.  Without the
// launch attribute both instructions are no-ops, so a kernel is correct
// whichever way it was launched.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

// Launch with the programmatic-stream-serialization attribute when the grid
// fits in one wave (small, latency-bound launches: single 256^2 / 512^2
// problems); large multi-wave grids keep plain stream ordering.
template <typename... KArgs, typename... Args>
cudaError_t launch_chain(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                         cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  const long long ctas = (long long)grid.x * grid.y * grid.z;
  if (ctas <= 2LL * sm_count()) {
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace psb

// Deterministic fp64 reductions (objective, TV, rel_error, finiteness).
//
// Pass 1: grid (chunks, n) -- each CTA reduces a fixed slice of one problem
// (warp shuffles then shared memory) into partial[p * chunks + blk].
// Pass 2: one warp per problem sums its partials in a fixed order.  The
// result is bit-reproducible run to run; it matches numpy's pairwise/BLAS
// order only to ~1e-15 relative (SURVEY 8(c+)).
#include "common.cuh"

namespace psb {

namespace {

constexpr int RB = 256;  // threads per reduction CTA

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double s[RB / 32];
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) s[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = l < RB / 32 ? s[l] : 0.0;
    r = warp_sum(r);
  }
  return r;  // valid in thread 0
}

enum Op { SUMSQ = 0, DOT = 1, NONFINITE = 2, BELOW = 3, OUTSIDE_BALL = 4 };

template <class T, int OP>
__global__ void __launch_bounds__(RB) elem_reduce(const T* __restrict__ a, const T* __restrict__ b,
                                                  int64_t len, int64_t bstride, double thr,
                                                  int chunks, double* __restrict__ part) {
  const int64_t p = blockIdx.y;
  const int64_t per = (len + chunks - 1) / chunks;
  const int64_t lo = blockIdx.x * per, hi = min(len, lo + per);
  const T* ap = a + p * len;
  const T* bp = b ? b + p * bstride : nullptr;
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += RB) {
    const double av = (double)ap[i];
    if (OP == SUMSQ) {
      const double d = bp ? av - (double)bp[i] : av;
      acc += d * d;
    } else if (OP == DOT) {
      acc += av * (double)bp[i];
    } else if (OP == NONFINITE) {
      acc += isfinite(av) ? 0.0 : 1.0;
    } else if (OP == OUTSIDE_BALL) {  // tv.py:98-100: sqrt(q0^2 + q1^2) > thr, in fp64
      const double bv = (double)bp[i];
      acc += sqrt(av * av + bv * bv) > thr ? 1.0 : 0.0;
    } else {
      acc += av < thr ? 1.0 : 0.0;
    }
  }
  const double r = block_sum(acc);
  if (threadIdx.x == 0) part[p * chunks + blockIdx.x] = r;
}

// tv.py:19-22 -- sum over pixels of |grad u|, fp64 accumulation.
template <class T>
__global__ void __launch_bounds__(RB) tv_reduce(const T* __restrict__ u, int H, int W, int chunks,
                                                double* __restrict__ part) {
  const int64_t p = blockIdx.y;
  const int64_t len = (int64_t)H * W;
  const int64_t per = (len + chunks - 1) / chunks;
  const int64_t lo = blockIdx.x * per, hi = min(len, lo + per);
  const T* up = u + p * len;
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += RB) {
    const int r = (int)(i / W), c = (int)(i % W);
    const double v = (double)up[i];
    const double gy = r < H - 1 ? (double)up[i + W] - v : 0.0;
    const double gx = c < W - 1 ? (double)up[i + 1] - v : 0.0;
    acc += sqrt(gy * gy + gx * gx);
  }
  const double r = block_sum(acc);
  if (threadIdx.x == 0) part[p * chunks + blockIdx.x] = r;
}

__global__ void finish_reduce(const double* __restrict__ part, int chunks, int64_t n,
                              double* __restrict__ out) {
  const int64_t p = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int l = threadIdx.x & 31;
  if (p >= n) return;
  double acc = 0.0;
  for (int c = l; c < chunks; c += 32) acc += part[p * chunks + c];
  acc = warp_sum(acc);
  if (l == 0) out[p] = acc;
}

int chunks_for(int64_t n, int64_t len) {
  const int64_t want_blocks = 8LL * sm_count();
  int64_t c = std::max<int64_t>(1, want_blocks / std::max<int64_t>(n, 1));
  c = std::min<int64_t>(c, (len + RB * 4 - 1) / (RB * 4));
  return (int)std::max<int64_t>(1, std::min<int64_t>(c, 1024));
}

template <class Launch>
int two_pass(int64_t n, int64_t len, double* out, cudaStream_t st, Launch launch) {
  PSB_REQUIRE(n >= 0 && n <= 65535, "reduce: batch size out of range");
  if (n == 0) return PSB_OK;
  const int chunks = chunks_for(n, len);
  double* part = nullptr;
  PSB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&part), sizeof(double) * n * chunks, st));
  launch(dim3(chunks, (unsigned)n), chunks, part);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) {
    finish_reduce<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(part, chunks, n, out);
    e = cudaGetLastError();
  }
  cudaFreeAsync(part, st);
  if (e != cudaSuccess) return fail(PSB_ERR_CUDA, std::string("reduce launch: ") + cudaGetErrorString(e));
  return PSB_OK;
}

template <int OP>
int elem(int dtype, const void* a, const void* b, int64_t n, int64_t len, double* out,
         cudaStream_t st, int64_t bstride = -1, double thr = 0.0) {
  if (bstride < 0) bstride = len;
  if (dtype == PSB_F32)
    return two_pass(n, len, out, st, [&](dim3 g, int chunks, double* part) {
      elem_reduce<float, OP><<<g, RB, 0, st>>>((const float*)a, (const float*)b, len, bstride, thr,
                                               chunks, part);
    });
  if (dtype == PSB_F64)
    return two_pass(n, len, out, st, [&](dim3 g, int chunks, double* part) {
      elem_reduce<double, OP><<<g, RB, 0, st>>>((const double*)a, (const double*)b, len, bstride,
                                                thr, chunks, part);
    });
  return fail(PSB_ERR_VALUE, "reduce: unknown dtype");
}

}  // namespace

}  // namespace psb

extern "C" {

int psb_sumsq(int dtype, const void* a, const void* b, int64_t n, int64_t len, double* out,
              void* stream) {
  return psb::elem<psb::SUMSQ>(dtype, a, b, n, len, out, psb::as_stream(stream));
}

int psb_dot(int dtype, const void* a, const void* b, int64_t n, int64_t len, double* out,
            void* stream) {
  PSB_REQUIRE(b != nullptr, "dot: second operand missing");
  return psb::elem<psb::DOT>(dtype, a, b, n, len, out, psb::as_stream(stream));
}

int psb_sumsq_bcast(int dtype, const void* a, const void* b, int64_t n, int64_t len, double* out,
                    void* stream) {
  PSB_REQUIRE(b != nullptr, "sumsq_bcast: shared operand missing");
  return psb::elem<psb::SUMSQ>(dtype, a, b, n, len, out, psb::as_stream(stream), 0);
}

int psb_count_below(int dtype, const void* a, int64_t n, int64_t len, double thresh, double* out,
                    void* stream) {
  return psb::elem<psb::BELOW>(dtype, a, nullptr, n, len, out, psb::as_stream(stream), len, thresh);
}

int psb_count_outside_ball(int dtype, const void* q, int64_t len, double r, double* out,
                           void* stream) {
  const size_t es = dtype == PSB_F32 ? 4 : 8;
  const void* q1 = static_cast<const char*>(q) + es * (size_t)len;
  return psb::elem<psb::OUTSIDE_BALL>(dtype, q, q1, 1, len, out, psb::as_stream(stream), 0, r);
}

int psb_count_nonfinite(int dtype, const void* a, int64_t count, double* out, void* stream) {
  return psb::elem<psb::NONFINITE>(dtype, a, nullptr, 1, count, out, psb::as_stream(stream));
}

int psb_tv2d(int dtype, const void* u, int64_t n, int H, int W, double* out, void* stream) {
  PSB_REQUIRE(H >= 2 && W >= 2, "tv_value: need a 2-D grid with both sides >= 2");
  auto st = psb::as_stream(stream);
  const int64_t len = (int64_t)H * W;
  if (dtype == PSB_F32)
    return psb::two_pass(n, len, out, st, [&](dim3 g, int chunks, double* part) {
      psb::tv_reduce<float><<<g, psb::RB, 0, st>>>((const float*)u, H, W, chunks, part);
    });
  if (dtype == PSB_F64)
    return psb::two_pass(n, len, out, st, [&](dim3 g, int chunks, double* part) {
      psb::tv_reduce<double><<<g, psb::RB, 0, st>>>((const double*)u, H, W, chunks, part);
    });
  return psb::fail(PSB_ERR_VALUE, "tv2d: unknown dtype");
}

}  // extern "C"

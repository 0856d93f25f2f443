// Periodic convolution blur and its fidelity gradient (operators.py:109-184,
// problems.py:121 -- BASELINE config 2).
//
// Two evaluation orders:
//  * direct  : the reference's 2-D tap loop (a outer, b inner, accumulator
//              starting at 0, every op rounded) -- bit-identical to
//              blur_forward/blur_adjoint in the fp64 instantiation;
//  * separable: Gaussian kernels are outer products w = w1 w1^T, so the
//              production path does 2k instead of k^2 MACs per pixel, and the
//              fidelity gradient g = A^T (A u - b) is ONE fused kernel: a CTA
//              stages its u tile plus a 2R halo (periodic wrap) in shared
//              memory, forms r = A u - b on the tile plus an R halo, and then
//              applies the flipped (correlation) pass to produce g -- u, b
//              read once, g written once (12 B/px fp32, 24 B/px fp64).
#include <cstdlib>

#include "common.cuh"

namespace psb {

namespace {

constexpr int KMAX = 15;

struct Taps {
  int k;
  double w2[KMAX * KMAX];
  double w1[KMAX];
};

__device__ __forceinline__ int wrap(int i, int n) {
  i %= n;
  return i < 0 ? i + n : i;
}

// operators.py:149-158 / 161-172 in the reference order.
template <class T>
__global__ void blur_direct_kernel(const T* __restrict__ u, T* __restrict__ out, int64_t n, int H,
                                   int W, Taps t, int adjoint) {
  using A = Ar<T>;
  const int c = t.k / 2;
  const int64_t HW = (int64_t)H * W;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n * HW;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = idx / HW;
    const int i = (int)((idx % HW) / W), j = (int)(idx % W);
    const T* up = u + p * HW;
    T acc = T(0);
    for (int a = 0; a < t.k; ++a) {
      const int ii = adjoint ? wrap(i + a - c, H) : wrap(i - a + c, H);
      for (int b = 0; b < t.k; ++b) {
        const T w = (T)t.w2[a * t.k + b];
        if (w == T(0)) continue;
        const int jj = adjoint ? wrap(j + b - c, W) : wrap(j - b + c, W);
        acc = A::add(acc, A::mul(w, up[(int64_t)ii * W + jj]));
      }
    }
    out[idx] = acc;
  }
}

__device__ __forceinline__ int wrap1(int i, int n) {  // periodic index, cheap near [0, n)
  while (i < 0) i += n;
  while (i >= n) i -= n;
  return i;
}

// Fused g = A^T (A u - b), separable, kernel size K and tile side TS at
// compile time: every loop below has a constant trip count over the 256
// threads (unrolled, no runtime division), and the periodic tile rows /
// columns are wrapped once per element with a compare (|offset| < H, W).
// One CTA per TS x TS output tile; TS = 16 gives 1024 CTAs at 512^2, all
// resident at once (22 KB of shared memory each in fp64).
__device__ __forceinline__ int wrap_near(int i, int n, bool near) {
  if (!near) {  // image smaller than a tile: any offset
    i %= n;
    return i < 0 ? i + n : i;
  }
  return i < 0 ? i + n : (i >= n ? i - n : i);  // i in [-n, 2n)
}

// Optional ProxSkip pre epilogue of the fused gradient (deblurring driver):
// coin iterations write the prox input z = (x - gamma g) + hcoef h and keep g
// for the post step; skipped iterations write x-hat = (x - gamma g) + gamma h
// to x_next, a buffer other than the x being read (other CTAs still stage
// its halo), and the driver swaps the two.
template <class T, class TF>
struct PreEpi {
  T* x_next;
  const T* h;
  TF* z;
  T gamma, hcoef;
  int coin;
  int32_t* bad;
  int k;
};

template <class T, int TS, int K, int SEP_NT, class TF, bool EPI>
__global__ void __launch_bounds__(SEP_NT, 2048 / SEP_NT) blur_grad_sep_kernel(
    const T* __restrict__ u, const T* __restrict__ bdat, T* __restrict__ g, int H, int W, Taps t,
    PreEpi<T, TF> epi) {
  using A = Ar<T>;
  extern __shared__ unsigned char smem_raw[];
  pdl_enter();
  T* sm = reinterpret_cast<T*>(smem_raw);
  constexpr int R = K / 2;
  constexpr int NU = TS + 4 * R;  // u tile side (2R halo each side)
  constexpr int NR = TS + 2 * R;  // r tile side
  T* su = sm;                     // NU x NU
  T* sh = su + NU * NU;           // NU rows x NR cols  (row pass of A)
  T* sr = sh + NU * NR;           // NR x NR            (r = A u - b)
  T* sh2 = sr + NR * NR;          // NR rows x TS cols  (row pass of A^T)
  T w1[K];
#pragma unroll
  for (int q = 0; q < K; ++q) w1[q] = (T)t.w1[q];

  const int i0 = blockIdx.y * TS, j0 = blockIdx.x * TS;
  const int tid = threadIdx.x;
  const bool near = H >= NU && W >= NU;  // every tile index within one period
#pragma unroll
  for (int e0 = 0; e0 < NU * NU; e0 += SEP_NT) {
    const int e = e0 + tid;
    if (NU * NU % SEP_NT == 0 || e < NU * NU) {
      const int a = e / NU, b = e % NU;
      su[e] = u[(int64_t)wrap_near(i0 - 2 * R + a, H, near) * W +
                wrap_near(j0 - 2 * R + b, W, near)];
    }
  }
  __syncthreads();
  // forward A: out(i,j) = sum_a sum_b w1[a] w1[b] u(i-a+c, j-b+c)
#pragma unroll
  for (int e0 = 0; e0 < NU * NR; e0 += SEP_NT) {
    const int e = e0 + tid;
    if (NU * NR % SEP_NT == 0 || e < NU * NR) {
      const int a = e / NR, jc = e % NR;  // jc: r-tile column; u column jc + R + (c - b)
      T acc = T(0);
#pragma unroll
      for (int q = 0; q < K; ++q) acc += w1[q] * su[a * NU + jc + R + (R - q)];
      sh[e] = acc;
    }
  }
  __syncthreads();
#pragma unroll
  for (int e0 = 0; e0 < NR * NR; e0 += SEP_NT) {
    const int e = e0 + tid;
    if (NR * NR % SEP_NT == 0 || e < NR * NR) {
      const int ic = e / NR, jc = e % NR;
      T acc = T(0);
#pragma unroll
      for (int q = 0; q < K; ++q) acc += w1[q] * sh[(ic + R + (R - q)) * NR + jc];
      const int gi = wrap_near(i0 - R + ic, H, near), gj = wrap_near(j0 - R + jc, W, near);
      sr[e] = acc - bdat[(int64_t)gi * W + gj];
    }
  }
  __syncthreads();
  // adjoint A^T: out(i,j) = sum_a sum_b w1[a] w1[b] r(i+a-c, j+b-c)
#pragma unroll
  for (int e0 = 0; e0 < NR * TS; e0 += SEP_NT) {
    const int e = e0 + tid;
    if (NR * TS % SEP_NT == 0 || e < NR * TS) {
      const int ic = e / TS, jt = e % TS;
      T acc = T(0);
#pragma unroll
      for (int q = 0; q < K; ++q) acc += w1[q] * sr[ic * NR + jt + q];
      sh2[e] = acc;
    }
  }
  __syncthreads();
#pragma unroll
  for (int e0 = 0; e0 < TS * TS; e0 += SEP_NT) {
    const int e = e0 + tid;
    if (TS * TS % SEP_NT == 0 || e < TS * TS) {
      const int it = e / TS, jt = e % TS;
      const int gi = i0 + it, gj = j0 + jt;
      if (gi < H && gj < W) {
        T acc = T(0);
#pragma unroll
        for (int q = 0; q < K; ++q) acc += w1[q] * sh2[(it + q) * TS + jt];
        const int64_t o = (int64_t)gi * W + gj;
        if constexpr (EPI) {
          // the ProxSkip pre step on this pixel (proxskip_pre_kernel's
          // arithmetic, skip.py:66-70); x is the tile centre already staged
          const T xo = su[(it + 2 * R) * NU + jt + 2 * R];
          const T tt = A::sub(xo, A::mul(epi.gamma, acc));
          if (epi.coin) {
            g[o] = acc;  // the post step recomputes x-hat from it
            epi.z[o] = (TF)A::add(tt, A::mul(epi.hcoef, epi.h[o]));
          } else {
            const T xn = A::add(tt, A::mul(epi.gamma, epi.h[o]));
            epi.x_next[o] = xn;
            if (!finite(xn) && epi.bad) atomicMin(epi.bad, epi.k);
          }
        } else {
          g[o] = acc;
        }
      }
    }
  }
}

template <class T, int TS>
size_t sep_smem(int k) {
  const int R = k / 2, NU = TS + 4 * R, NR = TS + 2 * R;
  return sizeof(T) * (size_t)(NU * NU + NU * NR + NR * NR + NR * TS);
}

int make_taps(const double* taps2d, const double* taps1d, int k, Taps& t) {
  PSB_REQUIRE(k >= 1 && k <= KMAX && (k % 2) == 1, "blur: kernel size must be odd and <= 15");
  t.k = k;
  for (int i = 0; i < k * k; ++i) t.w2[i] = taps2d ? taps2d[i] : 0.0;
  for (int i = 0; i < k; ++i) t.w1[i] = taps1d ? taps1d[i] : 0.0;
  return PSB_OK;
}

template <class T, class TF, bool EPI, int K>
int launch_sep_k(const void* u, const void* b, void* g, int H, int W, const Taps& t,
                 const PreEpi<T, TF>& epi, cudaStream_t st) {
  // 32 x 32 output tiles, 1024 threads: at 512^2 the 256 CTAs are resident
  // at once (2 per SM); measured 8.96 us against 10.0 for 16 x 16 / 256
  constexpr int TS = 32, NT = 1024;
  const size_t sm = sep_smem<T, TS>(K);
  auto kern = blur_grad_sep_kernel<T, TS, K, NT, TF, EPI>;
  PSB_CHECK(func_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  dim3 grid((W + TS - 1) / TS, (H + TS - 1) / TS);
  PSB_CUDA(launch_chain(kern, grid, dim3(NT), sm, st, (const T*)u, (const T*)b, (T*)g, H, W, t,
                        epi));
  return PSB_OK;
}

template <class T, class TF, bool EPI>
int launch_sep(const void* u, const void* b, void* g, int H, int W, const Taps& t,
               const PreEpi<T, TF>& e, cudaStream_t st) {
  switch (t.k) {
    case 1: return launch_sep_k<T, TF, EPI, 1>(u, b, g, H, W, t, e, st);
    case 3: return launch_sep_k<T, TF, EPI, 3>(u, b, g, H, W, t, e, st);
    case 5: return launch_sep_k<T, TF, EPI, 5>(u, b, g, H, W, t, e, st);
    case 7: return launch_sep_k<T, TF, EPI, 7>(u, b, g, H, W, t, e, st);
    case 9: return launch_sep_k<T, TF, EPI, 9>(u, b, g, H, W, t, e, st);
    case 11: return launch_sep_k<T, TF, EPI, 11>(u, b, g, H, W, t, e, st);
    case 13: return launch_sep_k<T, TF, EPI, 13>(u, b, g, H, W, t, e, st);
    case 15: return launch_sep_k<T, TF, EPI, 15>(u, b, g, H, W, t, e, st);
    default: return fail(PSB_ERR_VALUE, "blur: kernel size must be odd and <= 15");
  }
}

}  // namespace

int blur_grad2d(int dtype, const void* u, const void* b, void* g, int H, int W,
                const double* taps2d, const double* taps1d, int k, int separable, void* scratch,
                cudaStream_t st);

// Separable gradient fused with the ProxSkip pre step (driver.cu, deblurring)
int blur_grad_pre2d(int dto, int dtf, const void* x, const void* b, void* g, int H, int W,
                    const double* taps1d, int k, void* x_next, const void* h, void* z,
                    double gamma, double hcoef, int coin, int32_t* bad, int kiter,
                    cudaStream_t st) {
  Taps t;
  int rc = make_taps(nullptr, taps1d, k, t);
  if (rc) return rc;
  PSB_REQUIRE(k <= H && k <= W, "blur: kernel size exceeds image");
  PSB_REQUIRE(taps1d != nullptr, "blur: separable mode needs 1-D taps");
  if (dto == PSB_F64 && dtf == PSB_F32) {
    PreEpi<double, float> e{(double*)x_next, (const double*)h, (float*)z, gamma, hcoef, coin, bad,
                            kiter};
    return launch_sep<double, float, true>(x, b, g, H, W, t, e, st);
  }
  if (dto == PSB_F64 && dtf == PSB_F64) {
    PreEpi<double, double> e{(double*)x_next, (const double*)h, (double*)z, gamma, hcoef, coin,
                             bad, kiter};
    return launch_sep<double, double, true>(x, b, g, H, W, t, e, st);
  }
  if (dto == PSB_F32 && dtf == PSB_F32) {
    PreEpi<float, float> e{(float*)x_next, (const float*)h, (float*)z, (float)gamma, (float)hcoef,
                           coin, bad, kiter};
    return launch_sep<float, float, true>(x, b, g, H, W, t, e, st);
  }
  return fail(PSB_ERR_VALUE, "blur: unsupported dtype pair");
}

}  // namespace psb

extern "C" {

int psb_blur2d(int dtype, const void* u, void* out, int64_t n, int H, int W, const double* taps2d,
               int ksize, int adjoint, void* stream) {
  psb::Taps t;
  int rc = psb::make_taps(taps2d, nullptr, ksize, t);
  if (rc) return rc;
  PSB_REQUIRE(ksize <= H && ksize <= W, "blur: kernel size exceeds image");
  const int64_t cnt = n * (int64_t)H * W;
  if (cnt == 0) return PSB_OK;
  dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((cnt + 255) / 256, 64LL * psb::sm_count())));
  auto st = psb::as_stream(stream);
  if (dtype == PSB_F32)
    psb::blur_direct_kernel<float><<<grid, 256, 0, st>>>((const float*)u, (float*)out, n, H, W, t, adjoint);
  else if (dtype == PSB_F64)
    psb::blur_direct_kernel<double><<<grid, 256, 0, st>>>((const double*)u, (double*)out, n, H, W, t, adjoint);
  else
    return psb::fail(PSB_ERR_VALUE, "blur: unknown dtype");
  PSB_LAUNCHED("blur_direct");
  return PSB_OK;
}

int psb_blur_grad2d(int dtype, const void* u, const void* b, void* g, int H, int W,
                    const double* taps2d, const double* taps1d, int ksize, int separable,
                    void* scratch, void* stream) {
  return psb::blur_grad2d(dtype, u, b, g, H, W, taps2d, taps1d, ksize, separable, scratch,
                          psb::as_stream(stream));
}

}  // extern "C"

namespace psb {

// g = A^T (A u - b).  separable: one fused kernel.  direct: the reference
// order (forward into `scratch`, subtract b, adjoint), bit-exact in fp64.
int blur_grad2d(int dtype, const void* u, const void* b, void* g, int H, int W,
                const double* taps2d, const double* taps1d, int k, int separable, void* scratch,
                cudaStream_t st) {
  Taps t;
  int rc = make_taps(taps2d, taps1d, k, t);
  if (rc) return rc;
  PSB_REQUIRE(k <= H && k <= W, "blur: kernel size exceeds image");
  if (separable) {
    PSB_REQUIRE(taps1d != nullptr, "blur: separable mode needs 1-D taps");
    if (dtype == PSB_F32)
      return launch_sep<float, float, false>(u, b, g, H, W, t, PreEpi<float, float>{}, st);
    if (dtype == PSB_F64)
      return launch_sep<double, float, false>(u, b, g, H, W, t, PreEpi<double, float>{}, st);
    return fail(PSB_ERR_VALUE, "blur: unknown dtype");
  }
  PSB_REQUIRE(scratch != nullptr, "blur: direct mode needs an (H, W) scratch buffer");
  rc = psb_blur2d(dtype, u, scratch, 1, H, W, taps2d, k, 0, st);
  if (rc) return rc;
  rc = psb_lincomb(dtype, 1.0, scratch, -1.0, b, scratch, (int64_t)H * W, st);
  if (rc) return rc;
  return psb_blur2d(dtype, scratch, g, 1, H, W, taps2d, k, 1, st);
}

}  // namespace psb

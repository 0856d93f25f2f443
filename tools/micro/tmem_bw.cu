// Micro-benchmark: TMEM as a thread-private spill space.  Each thread owns 128
// columns of its TMEM lane (4 warps share a lane quarter: 4 x 128 = 512
// columns); measures tcgen05.st / tcgen05.ld .32x32b.x32 throughput per SM
// against LDS.64 / STS.64 of the same bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu && ./tmem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void tm_st32(uint32_t addr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(addr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tm_ld32(uint32_t addr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(addr)
      : "memory");
}

// mode 0: TMEM st+ld, 1: TMEM ld only, 2: TMEM st only, 3: smem st+ld (64-bit), 4: smem ld only
__global__ void __launch_bounds__(512, 1) bench(int mode, int iters, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t tm_base;
  extern __shared__ __align__(16) unsigned char dyn[];
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tm_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // lane quarter of this warp (bits 31:16 = lane, 15:0 = column), 128 columns per warp
  const uint32_t addr = tm_base + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128);
  uint32_t v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = tid * 33 + i;
  unsigned long long* s64 = reinterpret_cast<unsigned long long*>(dyn);
  tm_st32(addr, v);
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) s64[i * 512 + tid] = ((unsigned long long)v[2 * i + 1] << 32) | v[2 * i];
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0 || mode == 2) {
      tm_st32(addr, v);
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
    if (mode == 0 || mode == 1) {
      tm_ld32(addr, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += 1;
    }
    if (mode == 3) {
#pragma unroll
      for (int i = 0; i < 16; ++i) s64[i * 512 + tid] = ((unsigned long long)v[2 * i + 1] << 32) | v[2 * i];
    }
    if (mode == 3 || mode == 4) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const unsigned long long x = s64[i * 512 + tid];
        v[2 * i] = (uint32_t)x + 1;
        v[2 * i + 1] = (uint32_t)(x >> 32) + 1;
      }
    }
    if (mode == 2) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += 1;
    }
  }
  const long long t1 = clock64();
  __syncthreads();
  if (tid == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) acc ^= v[i];
  sink[blockIdx.x * 512 + tid] = acc;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tm_base));
}

int main() {
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 148 * 512 * 4);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 512 * 8);
  const char* names[] = {"TMEM st+ld x32", "TMEM ld x32", "TMEM st x32", "smem 16x(STS.64+LDS.64)", "smem 16xLDS.64"};
  const int iters = 2000;
  for (int mode = 0; mode < 5; ++mode) {
    bench<<<148, 512, 16 * 512 * 8>>>(mode, iters, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%s: %s\n", names[mode], cudaGetErrorString(e));
      return 1;
    }
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double c = (double)h[0] / iters;  // cycles per iteration of one CTA (16 warps)
    const double bytes = 512.0 * 32 * 4 * ((mode == 0 || mode == 3) ? 2 : 1);
    printf("%-26s %8.1f cycles per CTA-iteration (16 warps x 4 KB), %.1f B/cycle/SM\n", names[mode], c, bytes / c);
  }
  return 0;
}

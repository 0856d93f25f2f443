// Per-problem Bernoulli coin streams on the device (skip.py:16-28, 67, 136):
// coin_k = Generator(Philox(seed)).random() < p, bit-identical to numpy.
//
// One thread per seed:
//   * SeedSequence(seed).generate_state(2, uint64) -> the Philox4x64-10 key
//     (numpy/random/bit_generator.pyx: hashmix / mix over a 4-word pool,
//     entropy = the seed's little-endian 32-bit words);
//   * Philox4x64-10 with a zero counter incremented before each 4-word block
//     (numpy/random/src/philox/philox.h), random() = (next64 >> 11) * 2^-53.
// Config 4 draws 4096 streams x 300 coins; the host numpy loop takes ~50 ms,
// this kernel well under a millisecond.  tests/test_gpu_edges.py pins it
// against numpy's Generator(Philox(seed)) stream for many seeds.
#include <vector>

#include "common.cuh"

namespace psb {

namespace {

constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu,
                   MULT_B = 0x58f38dedu, MIX_MULT_L = 0xca01f9ddu, MIX_MULT_R = 0x4973f715u;

__host__ __device__ inline uint32_t hashmix(uint32_t v, uint32_t& hc) {
  v ^= hc;
  hc *= MULT_A;
  v *= hc;
  v ^= v >> 16;
  return v;
}

__host__ __device__ inline uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = MIX_MULT_L * x - MIX_MULT_R * y;
  r ^= r >> 16;
  return r;
}

// SeedSequence(seed).generate_state(2, np.uint64) for 0 <= seed < 2^64
__host__ __device__ inline void philox_key(uint64_t seed, uint64_t key[2]) {
  uint32_t ent[2];
  int n_ent = 0;
  if (seed == 0) {
    ent[n_ent++] = 0;
  } else {
    while (seed) {
      ent[n_ent++] = (uint32_t)(seed & 0xffffffffu);
      seed >>= 32;
    }
  }
  uint32_t pool[4], hc = INIT_A;
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n_ent ? ent[i] : 0u, hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], hc));
  // (at most 2 entropy words: no words beyond the pool to fold in)
  uint32_t st[4], hb = INIT_B;
  for (int i = 0; i < 4; ++i) {
    uint32_t v = pool[i] ^ hb;
    hb *= MULT_B;
    v *= hb;
    v ^= v >> 16;
    st[i] = v;
  }
  key[0] = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
  key[1] = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
}

__host__ __device__ inline void mulhilo(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
#ifdef __CUDA_ARCH__
  lo = a * b;
  hi = __umul64hi(a, b);
#else
  const unsigned __int128 p = (unsigned __int128)a * b;
  lo = (uint64_t)p;
  hi = (uint64_t)(p >> 64);
#endif
}

__host__ __device__ inline void philox4x64_10(const uint64_t ctr_in[4], const uint64_t key_in[2],
                                              uint64_t out[4]) {
  uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint64_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo(0xD2E7470EE14C6C93ull, c0, hi0, lo0);
    mulhilo(0xCA5A826395121157ull, c2, hi1, lo1);
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

__global__ void coin_table_kernel(const uint64_t* __restrict__ seeds, int64_t n, int K, double p,
                                  uint8_t* __restrict__ coins) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t key[2], ctr[4] = {0, 0, 0, 0}, buf[4];
  philox_key(seeds[i], key);
  int pos = 4;
  for (int k = 0; k < K; ++k) {
    if (pos == 4) {
      if (++ctr[0] == 0 && ++ctr[1] == 0 && ++ctr[2] == 0) ++ctr[3];
      philox4x64_10(ctr, key, buf);
      pos = 0;
    }
    const double u = (double)(buf[pos++] >> 11) * (1.0 / 9007199254740992.0);
    coins[(int64_t)k * n + i] = u < p ? 1 : 0;
  }
}

}  // namespace

}  // namespace psb

extern "C" int psb_coin_table(const int64_t* seeds_host, int64_t n, int K, double p,
                              uint8_t* coins_host, void* stream) {
  PSB_REQUIRE(n >= 0 && K >= 0, "coin_table: negative size");
  PSB_REQUIRE(p > 0 && p <= 1, "SkipConfig: p must be in (0, 1]");
  for (int64_t i = 0; i < n; ++i)
    PSB_REQUIRE(seeds_host[i] >= 0, "SeedSequence: seeds must be non-negative");
  if (n == 0 || K == 0) return PSB_OK;
  cudaStream_t st = psb::as_stream(stream);
  void* d = nullptr;
  const size_t sb = sizeof(uint64_t) * (size_t)n, cb = (size_t)K * (size_t)n;
  PSB_CUDA(cudaMallocAsync(&d, sb + cb, st));
  uint64_t* dseeds = static_cast<uint64_t*>(d);
  uint8_t* dcoins = static_cast<uint8_t*>(d) + sb;
  PSB_CUDA(cudaMemcpyAsync(dseeds, seeds_host, sb, cudaMemcpyHostToDevice, st));
  psb::coin_table_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(dseeds, n, K, p, dcoins);
  PSB_LAUNCHED("coin_table");
  PSB_CUDA(cudaMemcpyAsync(coins_host, dcoins, cb, cudaMemcpyDeviceToHost, st));
  PSB_CUDA(cudaFreeAsync(d, st));
  PSB_CUDA(cudaStreamSynchronize(st));
  return PSB_OK;
}

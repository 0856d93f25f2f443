// Library-level C ABI: version, thread-local error message, device query.
#include <cstring>

#include "common.cuh"

namespace psb {

namespace {
thread_local std::string g_err;
}

void set_error(const std::string& msg) { g_err = msg; }

int fail(int status, const std::string& msg) {
  g_err = msg;
  return status;
}

int sm_count() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
      cached = n;
    else
      cached = 148;
  }
  return cached;
}

}  // namespace psb

extern "C" {

int psb_abi_version(void) { return PSB_ABI_VERSION; }

const char* psb_last_error(void) { return psb::g_err.c_str(); }

int psb_device_sm_count(int* out) {
  int dev = 0;
  PSB_CUDA(cudaGetDevice(&dev));
  PSB_CUDA(cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, dev));
  return PSB_OK;
}

/* ---- context and device buffers (the caller-facing half of the
 * boundary for hosts without a CUDA runtime of their own) ----------------- */
struct psb_ctx {
  int device;
  cudaStream_t stream;
  void* pinned;  // staging buffer for host <-> device copies
  size_t pinned_bytes;
};

int psb_ctx_create(int device, psb_ctx** out) {
  PSB_REQUIRE(out != nullptr, "ctx_create: null output");
  *out = nullptr;
  PSB_CUDA(cudaSetDevice(device));
  psb_ctx* c = new psb_ctx{device, nullptr, nullptr, 0};
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return psb::fail(PSB_ERR_CUDA, "ctx_create: stream creation failed");
  }
  *out = c;
  return PSB_OK;
}

int psb_ctx_destroy(psb_ctx* c) {
  if (!c) return PSB_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (c->pinned) cudaFreeHost(c->pinned);
  cudaStreamDestroy(c->stream);
  delete c;
  return PSB_OK;
}

void* psb_ctx_stream(psb_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int psb_ctx_sync(psb_ctx* c) {
  PSB_REQUIRE(c != nullptr, "ctx_sync: null context");
  PSB_CUDA(cudaStreamSynchronize(c->stream));
  return PSB_OK;
}

int psb_buf_alloc(psb_ctx* c, int64_t bytes, void** dptr) {
  PSB_REQUIRE(c != nullptr && dptr != nullptr && bytes >= 0, "buf_alloc: bad arguments");
  *dptr = nullptr;
  if (bytes == 0) return PSB_OK;
  PSB_CUDA(cudaSetDevice(c->device));
  PSB_CUDA(cudaMallocAsync(dptr, (size_t)bytes, c->stream));
  PSB_CUDA(cudaMemsetAsync(*dptr, 0, (size_t)bytes, c->stream));
  return PSB_OK;
}

int psb_buf_free(psb_ctx* c, void* dptr) {
  PSB_REQUIRE(c != nullptr, "buf_free: null context");
  if (dptr) PSB_CUDA(cudaFreeAsync(dptr, c->stream));
  return PSB_OK;
}

// host <-> device through a pinned staging buffer (pageable copies are
// several times slower); synchronous with respect to the host
static int staged(psb_ctx* c, void* dst, const void* src, int64_t bytes, bool up) {
  PSB_REQUIRE(c != nullptr && bytes >= 0, "copy: bad arguments");
  if (bytes == 0) return PSB_OK;
  PSB_CUDA(cudaSetDevice(c->device));
  const size_t chunk = 16u << 20;
  if (!c->pinned) {
    PSB_CUDA(cudaMallocHost(&c->pinned, 2 * chunk));
    c->pinned_bytes = 2 * chunk;
  }
  char* pin[2] = {static_cast<char*>(c->pinned), static_cast<char*>(c->pinned) + chunk};
  cudaEvent_t done[2];
  PSB_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
  PSB_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
  bool busy[2] = {false, false};
  int64_t prev_off = -1;
  size_t prev_n = 0;
  int prev_k = 0, k = 0;
  for (int64_t off = 0; off < bytes; off += (int64_t)chunk, k ^= 1) {
    const size_t n = (size_t)std::min<int64_t>((int64_t)chunk, bytes - off);
    if (busy[k]) cudaEventSynchronize(done[k]);
    if (up) {
      std::memcpy(pin[k], static_cast<const char*>(src) + off, n);
      cudaMemcpyAsync(static_cast<char*>(dst) + off, pin[k], n, cudaMemcpyHostToDevice, c->stream);
    } else {
      cudaMemcpyAsync(pin[k], static_cast<const char*>(src) + off, n, cudaMemcpyDeviceToHost,
                      c->stream);
    }
    cudaEventRecord(done[k], c->stream);
    busy[k] = true;
    if (!up && prev_off >= 0) {  // drain the previous chunk while this one is in flight
      cudaEventSynchronize(done[prev_k]);
      std::memcpy(static_cast<char*>(dst) + prev_off, pin[prev_k], prev_n);
    }
    prev_off = off;
    prev_n = n;
    prev_k = k;
  }
  if (!up && prev_off >= 0) {
    cudaEventSynchronize(done[prev_k]);
    std::memcpy(static_cast<char*>(dst) + prev_off, pin[prev_k], prev_n);
  }
  cudaStreamSynchronize(c->stream);
  cudaEventDestroy(done[0]);
  cudaEventDestroy(done[1]);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return psb::fail(PSB_ERR_CUDA, std::string("copy: ") + cudaGetErrorString(e));
  return PSB_OK;
}

int psb_upload(psb_ctx* c, void* dptr, const void* host, int64_t bytes) {
  return staged(c, dptr, host, bytes, true);
}

int psb_download(psb_ctx* c, void* host, const void* dptr, int64_t bytes) {
  return staged(c, host, dptr, bytes, false);
}

}  // extern "C"

// libtnb C ABI: library/device entry points and error plumbing (include/tnb.h).
#include <atomic>
#include <cstdio>
#include <mutex>
#include <string>

#include "common.cuh"

namespace tnb {

static thread_local std::string g_last_error = "";

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  std::string m = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  set_error(m);
  return TNB_ECUDA;
}

static std::atomic<long long> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static int g_ndev = -1;
static int g_sms = 0;
static std::once_flag g_dev_once;

static void probe_devices() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  g_ndev = n;
  if (n > 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    // workspaces (split-K partials, block-sparse metadata) come from the stream-ordered
    // pool; keep freed blocks cached instead of unmapping them at every synchronize
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
  }
}

int require_device() {
  std::call_once(g_dev_once, probe_devices);
  if (g_ndev <= 0) return fail(TNB_ENODEV, "no CUDA device visible: libtnb has no CPU fallback");
  return TNB_OK;
}

int sm_count() {
  std::call_once(g_dev_once, probe_devices);
  return g_sms > 0 ? g_sms : 148;
}

}  // namespace tnb

extern "C" {

int tnb_version(void) { return 100; }

int64_t tnb_launch_count(void) { return (int64_t)tnb::g_launches.load(); }

const char* tnb_last_error(void) { return tnb::g_last_error.c_str(); }

int tnb_device_count(int* count) {
  if (!count) return tnb::fail(TNB_EINVAL, "count is NULL");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  *count = n;
  return TNB_OK;
}

int tnb_set_device(int device) {
  int rc = tnb::require_device();
  if (rc) return rc;
  TNB_CUDA_CHECK(cudaSetDevice(device));
  return TNB_OK;
}

int tnb_synchronize(void* stream) {
  int rc = tnb::require_device();
  if (rc) return rc;
  TNB_CUDA_CHECK(cudaStreamSynchronize((cudaStream_t)stream));
  TNB_CUDA_CHECK(cudaGetLastError());
  return TNB_OK;
}

}  // extern "C"

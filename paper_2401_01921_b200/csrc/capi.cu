// libtnb C ABI: library/device entry points and error plumbing (include/tnb.h).
#include <atomic>
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

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

// ---- kernel timer ----------------------------------------------------------
struct KRec {
  int family;
  cudaEvent_t ev0, ev1;
  double work;
};
static std::atomic<bool> g_kt_on{false};
static std::mutex g_kt_mu;
static std::vector<KRec> g_kt_recs;
static std::vector<cudaEvent_t> g_kt_pool;

static cudaEvent_t kt_event() {
  if (!g_kt_pool.empty()) {
    cudaEvent_t e = g_kt_pool.back();
    g_kt_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return e;
}

KTimer::KTimer(int fam, cudaStream_t s, double w) : family(fam), st(s), work(w) {
  if (!g_kt_on.load(std::memory_order_relaxed)) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return;
  }
  std::lock_guard<std::mutex> g(g_kt_mu);
  ev0 = kt_event();
  ev1 = kt_event();
  if (ev0) cudaEventRecord(ev0, st);
}

KTimer::~KTimer() {
  if (!ev0 || !ev1) return;
  cudaEventRecord(ev1, st);
  std::lock_guard<std::mutex> g(g_kt_mu);
  g_kt_recs.push_back({family, ev0, ev1, work});
}

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

bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cs != cudaStreamCaptureStatusNone;
}

namespace {
// memory owned by captured graphs, queued for release by their user objects' destructors
// (which may not call CUDA): pinned host buffers and device buffers (with their device)
struct Deferred {
  void* p;
  int device;  // -1: pinned host memory
};
std::mutex g_deferred_mu;
std::vector<Deferred> g_deferred;
void CUDART_CB queue_free(void* rec) {
  Deferred* d = static_cast<Deferred*>(rec);
  std::lock_guard<std::mutex> lk(g_deferred_mu);
  g_deferred.push_back(*d);
  delete d;
}

// Ties `p` to the graph being captured on `st` (a user object the graph retains).
int tie_to_graph(cudaStream_t st, void* p, int device) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaGraph_t graph = nullptr;
  TNB_CUDA_CHECK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &graph, nullptr, nullptr));
  if (cs != cudaStreamCaptureStatusActive || !graph) return fail(TNB_EINVAL, "tie_to_graph: stream is not capturing");
  Deferred* rec = new Deferred{p, device};
  cudaUserObject_t obj = nullptr;
  cudaError_t e = cudaUserObjectCreate(&obj, rec, queue_free, 1, cudaUserObjectNoDestructorSync);
  if (e != cudaSuccess) {
    delete rec;
    return cuda_fail(e, "tie_to_graph: cudaUserObjectCreate");
  }
  // the graph takes over our reference: p lives until the graph and every exec made from it die
  TNB_CUDA_CHECK(cudaGraphRetainUserObject(graph, obj, 1, cudaGraphUserObjectMove));
  return TNB_OK;
}
}  // namespace

void release_deferred_host() {
  std::vector<Deferred> q;
  {
    std::lock_guard<std::mutex> lk(g_deferred_mu);
    q.swap(g_deferred);
  }
  int cur = -1;
  for (const Deferred& d : q) {
    if (d.device < 0) {
      cudaFreeHost(d.p);
    } else {
      if (cur < 0) cudaGetDevice(&cur);
      cudaSetDevice(d.device);
      cudaFree(d.p);
    }
  }
  if (cur >= 0) cudaSetDevice(cur);
  cudaGetLastError();
}

int capture_pinned(cudaStream_t st, size_t bytes, void** out) {
  *out = nullptr;
  void* p = nullptr;
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  TNB_CUDA_CHECK(cudaThreadExchangeStreamCaptureMode(&mode));
  cudaError_t e = cudaMallocHost(&p, bytes);
  cudaThreadExchangeStreamCaptureMode(&mode);
  if (e != cudaSuccess) return cuda_fail(e, "capture_pinned: cudaMallocHost");
  int rc = tie_to_graph(st, p, -1);
  if (rc) {
    cudaFreeHost(p);
    return rc;
  }
  *out = p;
  return TNB_OK;
}

int capture_device_ws(cudaStream_t st, size_t bytes, void** out) {
  *out = nullptr;
  int dev = 0;
  TNB_CUDA_CHECK(cudaGetDevice(&dev));
  void* p = nullptr;
  // cudaMalloc is a "potentially unsafe" call under global-mode capture: relax this
  // thread's capture mode for the allocation only (it does not touch the stream)
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  TNB_CUDA_CHECK(cudaThreadExchangeStreamCaptureMode(&mode));
  cudaError_t e = cudaMalloc(&p, bytes);
  cudaThreadExchangeStreamCaptureMode(&mode);
  if (e != cudaSuccess) return cuda_fail(e, "capture_device_ws: cudaMalloc");
  int rc = tie_to_graph(st, p, dev);
  if (rc) {
    cudaFree(p);
    return rc;
  }
  *out = p;
  return TNB_OK;
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

int tnb_ktimer_enable(int on) {
  tnb::g_kt_on.store(on != 0);
  return TNB_OK;
}

int tnb_ktimer_reset(void) {
  std::lock_guard<std::mutex> g(tnb::g_kt_mu);
  for (auto& r : tnb::g_kt_recs) {
    cudaEventSynchronize(r.ev1);
    tnb::g_kt_pool.push_back(r.ev0);
    tnb::g_kt_pool.push_back(r.ev1);
  }
  tnb::g_kt_recs.clear();
  cudaGetLastError();
  return TNB_OK;
}

int tnb_ktimer_read(int family, int64_t* launches, double* ms, double* work) {
  if (!launches || !ms || !work) return tnb::fail(TNB_EINVAL, "ktimer_read: NULL argument");
  std::lock_guard<std::mutex> g(tnb::g_kt_mu);
  int64_t n = 0;
  double t = 0.0, w = 0.0;
  for (auto& r : tnb::g_kt_recs) {
    if (r.family != family) continue;
    TNB_CUDA_CHECK(cudaEventSynchronize(r.ev1));
    float x = 0.f;
    TNB_CUDA_CHECK(cudaEventElapsedTime(&x, r.ev0, r.ev1));
    ++n;
    t += x;
    w += r.work;
  }
  *launches = n;
  *ms = t;
  *work = w;
  return TNB_OK;
}

int tnb_memcpy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width, int64_t height,
                       int kind, void* stream) {
  int rc = tnb::require_device();
  if (rc) return rc;
  if (!dst || !src || width < 0 || height < 0 || dpitch < width || spitch < width || kind < 0 || kind > 4)
    return tnb::fail(TNB_EINVAL, "memcpy2d: bad arguments");
  if (width == 0 || height == 0) return TNB_OK;
  TNB_CUDA_CHECK(cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width, (size_t)height,
                                   (cudaMemcpyKind)kind, (cudaStream_t)stream));
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

// Shared helpers for libtnb (sm_100a): status/error plumbing, fast integer
// division, and small host utilities.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <string>

#include "../../include/tnb.h"

// Device-side bounds checks for a CHECKED build (-DTNB_CHECKED=1, tools/build_checked.sh):
// the stand-in for compute-sanitizer, which this GPU pool does not allow. Every gathered
// operand offset is checked against its block / operand extent and every stream-K spin
// wait is bounded; a violation prints the site and traps. Compiled out by default.
#ifndef TNB_CHECKED
#define TNB_CHECKED 0
#endif
#if TNB_CHECKED
#include <cstdio>
#define TNB_DCHECK(cond, what)                                                                            \
  do {                                                                                                    \
    if (!(cond)) {                                                                                        \
      printf("TNB_DCHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__, (int)blockIdx.x, \
             (int)threadIdx.x);                                                                           \
      __trap();                                                                                           \
    }                                                                                                     \
  } while (0)
#else
#define TNB_DCHECK(cond, what) \
  do {                         \
  } while (0)
#endif

namespace tnb {

// Thread-local last-error message (tnb_last_error).
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define TNB_CUDA_CHECK(expr)                                   \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) return ::tnb::cuda_fail(_e, #expr); \
  } while (0)

// Returns TNB_OK iff at least one CUDA device is visible (cached).
int require_device();
int sm_count();

// True iff `st` is being captured into a CUDA graph.
bool capturing(cudaStream_t st);

// Pinned host memory owned by the graph being captured on `st`: a captured memcpy node
// re-reads its host source at every replay, so the source must live as long as the
// graph. The buffer is tied to the graph with a cudaUserObject; when the last graph
// (or instantiated graph) referencing it is destroyed, the pointer is queued and freed
// by the next release_deferred_host() call (CUDA API calls are not allowed inside a
// user-object destructor).
int capture_pinned(cudaStream_t st, size_t bytes, void** out);
// Device memory owned by the graph being captured on `st`, allocated once at capture time
// (not a per-replay allocation node) and released after the graph is destroyed. Used for
// stream-K workspaces of captured GEMMs: a replay never shares them with eager launches.
int capture_device_ws(cudaStream_t st, size_t bytes, void** out);
// Frees queued graph-owned host / device buffers. Call only outside stream capture.
void release_deferred_host();

// Counts every kernel this library launches (tnb_launch_count); bench.py reports it.
void count_launch(int n = 1);

// Per-family CUDA-event timing of this library's kernel launches (tnb_ktimer_*).
// Construct right before a launch and let it go out of scope right after: when the
// timer is enabled (and the stream is not being captured into a graph) it records
// an event pair on the launching stream and the algorithmic work of the launch.
struct KTimer {
  KTimer(int family, cudaStream_t st, double work);
  ~KTimer();
  KTimer(const KTimer&) = delete;
  KTimer& operator=(const KTimer&) = delete;
  int family;
  cudaStream_t st;
  double work;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

// Launches a persistent kernel whose CTAs wait on one another (stream-K partial
// hand-offs: an owner spins on the flags of its predecessor CTAs) with the COOPERATIVE
// attribute: the driver co-schedules every CTA of the grid (or rejects the launch), so an
// owner never waits on a CTA that cannot be dispatched because other kernels -- NCCL
// collectives, work on other streams -- hold SMs. The attribute survives graph capture.
template <typename... KArgs, typename... Args>
cudaError_t launch_cooperative(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                               cudaStream_t st, Args&&... args) {
  static const bool off = getenv("TNB_NO_COOP") != nullptr;  // dev A/B switch
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = off ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<Args&&>(args)...);
}

// Programmatic dependent launch: the kernel may be scheduled while the previous kernel on
// the stream is still running (its launch latency and index-table prologue overlap that
// kernel's tail); it MUST execute pdl_wait() before touching global memory another kernel
// produces or consumes. Only kernels that do are launched this way.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  static const bool off = getenv("TNB_NO_PDL") != nullptr;  // dev A/B switch
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = off ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<Args&&>(args)...);
}
// griddepcontrol.wait: every prerequisite grid has completed and its memory is visible.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// let the next PDL-launched kernel be scheduled (it still waits in pdl_wait for our completion)
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// Unsigned 32-bit division by a runtime-invariant divisor via multiply-high
// (Granlund-Montgomery). Valid for 0 <= n < 2^31 and 1 <= d < 2^31.
struct FastDiv {
  uint32_t d, m, s;
  __host__ __device__ FastDiv() : d(1), m(0), s(0) {}
  __host__ __device__ explicit FastDiv(uint32_t div) {
    d = div;
    if (d == 1) { m = 0; s = 0; return; }
    s = 0;
    while ((1ull << s) < d) ++s;  // s = ceil(log2 d)
    uint64_t mm = ((1ull << 32) * ((1ull << s) - d)) / d + 1;
    m = (uint32_t)mm;
  }
  __host__ __device__ __forceinline__ uint32_t div(uint32_t n) const {
#ifdef __CUDA_ARCH__
    if (d == 1) return n;
    uint32_t t = __umulhi(n, m);
    return (t + n) >> s;
#else
    return n / d;
#endif
  }
};

}  // namespace tnb

// Microbenchmark: cost of one stage hand-off in a warp-specialised mbarrier ring
// (16 consumer warps, NPROD producer threads, 8 stages), no data movement.
// Variants: arrivals per stage on `full` = every producer thread (noinc / plain) or one per
// producer warp; consumers: one arrive per warp on `empty`.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
template <int HINT>
__device__ __forceinline__ void wait_t(uint64_t* b, uint32_t ph) {
  if (HINT)
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n@!P bra W_%=;\n}" ::"r"(su32(b)), "r"(ph), "r"(0x989680));
  else
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}" ::"r"(su32(b)), "r"(ph));
}
__device__ int g_sink;
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b))); }
__device__ __forceinline__ void arrive_noinc(uint64_t* b) { asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(b))); }

template <int NPROD, int MODE, int WORK = 0, int HINT = 0>  // MODE 0: per-thread noinc, 1: plain, 2: per-warp
__global__ void ring(int iters, long long* out) {
  auto wait = [](uint64_t* b, uint32_t ph) { wait_t<HINT>(b, ph); };
  constexpr int NMATH = 512, ST = 8;
  __shared__ uint64_t full[ST], empty[ST];
  const int tid = threadIdx.x;
  if (tid == 0)
    for (int s = 0; s < ST; ++s) {
      init(&full[s], MODE == 2 ? NPROD / 32 : NPROD);
      init(&empty[s], NMATH / 32);
    }
  __syncthreads();
  long long t0 = clock64();
  if (tid >= NMATH) {
    const int p = tid - NMATH;
    for (int g = 0; g < iters; ++g) {
      const int s = g % ST;
      if (g >= ST) wait(&empty[s], ((g / ST) & 1) ^ 1);
      if (WORK) {  // dependent integer chain: WORK instructions of producer work per stage
        int x = g + p;
#pragma unroll
        for (int w = 0; w < WORK; ++w) x = x * 1664525 + 1013904223;
        if (x == 12345) g_sink = x;
      }
      if (MODE == 0) arrive_noinc(&full[s]);
      else if (MODE == 1) arrive(&full[s]);
      else {
        __syncwarp();
        if ((p & 31) == 0) arrive(&full[s]);
      }
    }
  } else {
    for (int g = 0; g < iters; ++g) {
      const int s = g % ST;
      wait(&full[s], (g / ST) & 1);
      __syncwarp();
      if ((tid & 31) == 0) arrive(&empty[s]);
    }
    if (tid == 0) out[blockIdx.x] = clock64() - t0;
  }
}

template <int NPROD, int MODE, int WORK = 0, int HINT = 0>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  const int iters = 4096;
  ring<NPROD, MODE, WORK, HINT><<<148, 512 + NPROD>>>(iters, d);
  ring<NPROD, MODE, WORK, HINT><<<148, 512 + NPROD>>>(iters, d);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%-28s NPROD=%3d work=%3d hint=%d: %.1f cycles per stage (%s)\n", name, NPROD, WORK, HINT, mx / iters,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<256, 0>("per-thread noinc arrive");
  run<256, 1>("per-thread plain arrive");
  run<256, 2>("per-warp arrive");
  run<128, 0>("per-thread noinc arrive");
  run<128, 2>("per-warp arrive");
  run<32, 0>("per-thread noinc arrive");
  run<256, 0, 0, 1>("noinc, suspend hint");
  run<256, 0, 32, 0>("noinc + 32 dep. IMADs");
  run<256, 0, 64, 0>("noinc + 64 dep. IMADs");
  run<256, 0, 64, 1>("noinc + 64 IMADs, hint");
  run<256, 0, 128, 0>("noinc + 128 dep. IMADs");
  return 0;
}

// FP64 roofline probe for B200 (sm_100a): DMMA (mma.sync f64) vs DFMA issue rate.
// Prints achieved TFLOP/s for each; the max is the fp64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    for (int bps : {1, 2}) {
      int threads = warps * 32;
      int blocks = sms * bps;
      float ms = time_it([&] { dmma_loop<8><<<blocks, threads>>>(out, iters); });
      double flop = 2.0 * 256.0 * 8 * iters * (double)blocks * warps;  // 256 MAC per warp-mma
      printf("DMMA m8n8k4 warps/cta=%d ctas/sm=%d : %.2f TFLOP/s\n", warps, bps, flop / ms / 1e9);
      ms = time_it([&] { dfma_loop<16><<<blocks, threads>>>(out, iters); });
      flop = 2.0 * 16 * iters * (double)blocks * threads;
      printf("DFMA          warps/cta=%d ctas/sm=%d : %.2f TFLOP/s\n", warps, bps, flop / ms / 1e9);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s sms %d\n", cudaGetErrorString(e), sms);
  return 0;
}

// DMMA.8x8x4 issue-rate probe (dev aid): W warps per CTA, F independent accumulator
// fragments per warp, one CTA per SM; prints FMA/clk/SM achieved.
#include <cstdio>
#include <cuda_runtime.h>
template <int F>
__global__ void k(double* out, int iters, long long* cyc) {
  double c0[F], c1[F];
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
#pragma unroll
  for (int f = 0; f < F; ++f) c0[f] = c1[f] = 0.0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int f = 0; f < F; ++f)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0[f]), "+d"(c1[f]) : "d"(a), "d"(b));
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int f = 0; f < F; ++f) s += c0[f] + c1[f];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int F>
void run(int warps) {
  double* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 8);
  cudaMalloc(&cyc, 8);
  const int iters = 2000;
  k<F><<<148, warps * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  k<F><<<148, warps * 32>>>(out, iters, cyc);
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  double fma = (double)warps * F * iters * 256.0;
  printf("warps %2d frags %2d: %6.1f FMA/clk/SM (%.0f cycles per DMMA per SMSP)\n", warps, F, fma / h,
         (double)h / ((double)warps * F * iters / 4));
  cudaFree(out);
  cudaFree(cyc);
}
int main() {
  for (int w : {1, 2, 4, 8, 16}) {
    run<1>(w); run<2>(w); run<4>(w); run<8>(w); run<16>(w);
  }
  return 0;
}

// Tile-config sweep for the FP64 DMMA core (development tool; not the product path).
// Builds C[M,N] = A[M,K] B[K,N] with the library's TileCore and reports TFLOP/s.
#include <cstdio>
#include <cstring>
#include <vector>

#include "../paper_2401_01921_b200/csrc/gemm_core.cuh"

namespace tnb {
void set_error(const std::string&) {}
int fail(int c, const std::string&) { return c; }
int cuda_fail(cudaError_t, const char*) { return TNB_ECUDA; }
}  // namespace tnb
using namespace tnb;

struct Desc {
  int M, N, K, tiles_m, tiles_n;
  Group rowA, kA, kB, colB;
  int a_mfast, b_nfast;
};

template <int BM, int BN, int BK, int WM, int WN, int ST>
__global__ void __launch_bounds__(WM* WN * 32, 1) bench_kernel(const double* A, const double* B, double* C, Desc d) {
  using Core = TileCore<false, 0, BM, BN, BK, WM, WN, ST>;
  extern __shared__ __align__(16) unsigned char smem[];
  int bid = blockIdx.x;
  const int group = 8, per_group = group * d.tiles_n;
  const int g = bid / per_group, first_m = g * group;
  const int gsz = min(d.tiles_m - first_m, group), in_g = bid - g * per_group;
  const int tm = first_m + in_g % gsz, tn = in_g / gsz;
  typename Core::Acc acc;
  Core::zero(acc);
  Core::mainloop(smem, A, B, d.rowA, d.kA, d.kB, d.colB, tm * BM, tn * BN, d.M, d.N, 0, d.K, d.a_mfast, d.b_nfast, acc);
  Core::store(C, d.N, tm * BM, tn * BN, d.M, d.N, acc);
}

Group g1(int64_t dim, int64_t stride) {
  Group g;
  memset(&g, 0, sizeof(g));
  g.n = 1;
  g.dim[0] = (int)dim;
  g.div[0] = FastDiv((uint32_t)dim);
  g.stride[0] = stride;
  return g;
}

template <int BM, int BN, int BK, int WM, int WN, int ST>
void run(const char* name, int M, int N, int K, bool a_mfast, bool b_nfast, double* A, double* B, double* C) {
  using Core = TileCore<false, 0, BM, BN, BK, WM, WN, ST>;
  auto kern = bench_kernel<BM, BN, BK, WM, WN, ST>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Core::kSmem);
  Desc d;
  d.M = M; d.N = N; d.K = K;
  d.tiles_m = (M + BM - 1) / BM; d.tiles_n = (N + BN - 1) / BN;
  // A: a_mfast -> stored K x M (m contiguous); else M x K
  d.rowA = a_mfast ? g1(M, 1) : g1(M, K);
  d.kA = a_mfast ? g1(K, M) : g1(K, 1);
  d.kB = b_nfast ? g1(K, N) : g1(K, 1);
  d.colB = b_nfast ? g1(N, 1) : g1(N, K);
  d.a_mfast = a_mfast; d.b_nfast = b_nfast;
  int grid = d.tiles_m * d.tiles_n;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WM * WN * 32, Core::kSmem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 2; ++i) kern<<<grid, WM * WN * 32, Core::kSmem>>>(A, B, C, d);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<grid, WM * WN * 32, Core::kSmem>>>(A, B, C, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaError_t err = cudaGetLastError();
  printf("%-28s M=%5d N=%5d K=%5d a_mfast=%d b_nfast=%d per_sm=%d smem=%6zu : %.3f ms %.2f TFLOP/s %s\n", name, M, N, K,
         a_mfast, b_nfast, per_sm, Core::kSmem, best, 2.0 * M * N * (double)K / best / 1e9, cudaGetErrorString(err));
}

int main() {
  size_t n = (size_t)8192 * 8192;
  double *A, *B, *C;
  cudaMalloc(&A, n * 8); cudaMalloc(&B, n * 8); cudaMalloc(&C, n * 8);
  cudaMemset(A, 0, n * 8); cudaMemset(B, 0, n * 8);
  struct Shape { int M, N, K; bool am, bn; };
  Shape shapes[] = {{2048, 5120, 1024, true, false}, {2048, 1024, 5120, true, true}, {4096, 4096, 4096, false, true},
                    {4096, 4096, 4096, true, false}};
  for (auto s : shapes) {
    run<128, 128, 16, 2, 4, 3>("128x128x16 w2x4 s3", s.M, s.N, s.K, s.am, s.bn, A, B, C);
    run<128, 128, 16, 4, 4, 3>("128x128x16 w4x4 s3", s.M, s.N, s.K, s.am, s.bn, A, B, C);
    run<128, 128, 32, 2, 4, 3>("128x128x32 w2x4 s3", s.M, s.N, s.K, s.am, s.bn, A, B, C);
    run<128, 128, 32, 4, 4, 3>("128x128x32 w4x4 s3", s.M, s.N, s.K, s.am, s.bn, A, B, C);
    run<128, 128, 16, 4, 2, 4>("128x128x16 w4x2 s4", s.M, s.N, s.K, s.am, s.bn, A, B, C);
    run<128, 64, 16, 2, 2, 4>("128x64x16 w2x2 s4", s.M, s.N, s.K, s.am, s.bn, A, B, C);
    run<256, 128, 16, 4, 4, 3>("256x128x16 w4x4 s3", s.M, s.N, s.K, s.am, s.bn, A, B, C);
    run<128, 256, 16, 4, 4, 3>("128x256x16 w4x4 s3", s.M, s.N, s.K, s.am, s.bn, A, B, C);
  }
  return 0;
}

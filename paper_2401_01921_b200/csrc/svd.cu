// Batched one-sided Jacobi SVD of the charge-sector matrices of a block-sparse tensor
// (the factorisation step of linalg.svd / svd_truncate, pkg/src/tnkit/linalg.py:246-341,
// where the reference calls LAPACK gesdd sector by sector).
//
// Every sector matrix A (m x n, m <= n, row-major, float64) is factorised by
// Hestenes' one-sided Jacobi on its ROWS -- rows are contiguous, so every access is a
// coalesced row sweep:  B = Q A with Q orthogonal (product of plane rotations) and the
// rows of B mutually orthogonal; then sigma_i = |b_i|, v_i = b_i / sigma_i, U = Q^T.
// Rows are paired by a round-robin tournament (m/2 disjoint pairs per round, m-1
// rounds per sweep) and sweeps repeat until a whole sweep performs no rotation
// (|b_p . b_q| <= tol |b_p| |b_q| for every pair) or max_sweeps is hit.
//
// One thread-block CLUSTER (16 CTAs x 16 warps) owns one sector: a warp rotates one
// row pair per task, the cluster barrier (barrier.cluster arrive.release /
// wait.acquire) separates rounds, and B / Q live in global memory read with .cg loads
// (L2; the 126 MB L2 holds every sector of a C4-sized two-site tensor). All sectors
// run concurrently, one cluster each. The finalize pass (same kernel) ranks the
// singular values (descending, ties by row) and writes the torch-compatible thin
// factors U (m x m), S (m), Vh (m x n). Rows with sigma below rank_tol * sigma_max
// cannot be normalised into an orthonormal V: such sectors are flagged (status -2)
// and the host recomputes them with the library factorisation.
#include <cmath>
#include <vector>

#include "common.cuh"

namespace tnb {
namespace {

constexpr int kCluster = 16;  // non-portable cluster size (B200 allows 16)
constexpr int kWarps = 16;
constexpr int kRegPL = 20;    // rows up to 640 long are held in registers (20 per lane)

struct SvdTask {
  const double* a; // [m][n] in (read only)
  double* b;       // [m][n] workspace: the rotated rows
  double* q;       // [m][m] workspace: accumulated rotations (rows)
  double* u;       // [m][m] out
  double* s;       // [m] out
  double* vh;      // [m][n] out
  int* status;     // [1] out: sweeps used (>0), -1 not converged, -2 rank deficient
  int* counter;    // [2] rotation counters (zero on entry)
  double* norm;    // [m] scratch: |b_i|
  int m, n;
};

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// round-robin tournament: P players (P even), round r, pair i -> (a, b)
__device__ __forceinline__ void rr_pair(int P, int r, int i, int& a, int& b) {
  const int M = P - 1;
  if (i == 0) {
    a = r % M;
    b = M;
  } else {
    a = (r + i) % M;
    b = (r - i + M) % M;
  }
}

__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kWarps * 32)
    jacobi_rows_kernel(const SvdTask* __restrict__ tasks, int max_sweeps, double tol, double rank_tol) {
  const SvdTask t = tasks[blockIdx.x / kCluster];
  const int crank = (int)cluster_rank();
  const int lane = threadIdx.x & 31;
  const int gw = crank * kWarps + (threadIdx.x >> 5);  // warp index within the cluster
  constexpr int NW = kCluster * kWarps;
  const int m = t.m, n = t.n;
  double* __restrict__ B = t.b;
  double* __restrict__ Q = t.q;
  // Q = I, B = A
  for (int64_t x = (int64_t)gw * 32 + lane; x < (int64_t)m * m; x += (int64_t)NW * 32)
    __stcg(Q + x, (x / m == x % m) ? 1.0 : 0.0);
  for (int64_t x = (int64_t)gw * 32 + lane; x < (int64_t)m * n; x += (int64_t)NW * 32) __stcg(B + x, t.a[x]);
  cluster_sync_all();
  const int P = m + (m & 1);  // an odd row count gets a virtual zero row (its pairs are skipped)
  // rotation threshold on |cos(b_p, b_q)|: tol x the rounding level of a length-n dot product
  const double thresh = tol * sqrt((double)n) * 2.220446049250313e-16;
  int sweep = 0, status = -1;
  if (m > 1) {
    int nrot = 0;
    for (sweep = 1; sweep <= max_sweeps; ++sweep) {
      int* cnt = t.counter + (sweep & 1);
      for (int r = 0; r < P - 1; ++r) {
        for (int i = gw; i < P / 2; i += NW) {
          int a, b;
          rr_pair(P, r, i, a, b);
          if (a >= m || b >= m) continue;
          if (a > b) {
            const int x = a;
            a = b;
            b = x;
          }
          double* ra = B + (int64_t)a * n;
          double* rb = B + (int64_t)b * n;
          double* qa = Q + (int64_t)a * m;
          double* qb = Q + (int64_t)b * m;
          if (n <= 32 * kRegPL) {
            // rows held in registers: one L2 round trip for B's rows, one for Q's
            double x[kRegPL], y[kRegPL];
            double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
            for (int u = 0; u < kRegPL; ++u) {
              const int j = lane + 32 * u;
              x[u] = j < n ? __ldcg(ra + j) : 0.0;
              y[u] = j < n ? __ldcg(rb + j) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kRegPL; ++u) {
              al = fma(x[u], x[u], al);
              be = fma(y[u], y[u], be);
              ga = fma(x[u], y[u], ga);
            }
            al = warp_sum(al);
            be = warp_sum(be);
            ga = warp_sum(ga);
            if (!(fabs(ga) > thresh * sqrt(al * be)) || al == 0.0 || be == 0.0) continue;
            const double zeta = (be - al) / (2.0 * ga);
            const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
#pragma unroll
            for (int u = 0; u < kRegPL; ++u) {
              const int j = lane + 32 * u;
              if (j < n) {
                __stcg(ra + j, c * x[u] - s * y[u]);
                __stcg(rb + j, s * x[u] + c * y[u]);
              }
            }
#pragma unroll
            for (int u = 0; u < kRegPL; ++u) {
              const int j = lane + 32 * u;
              x[u] = j < m ? __ldcg(qa + j) : 0.0;
              y[u] = j < m ? __ldcg(qb + j) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kRegPL; ++u) {
              const int j = lane + 32 * u;
              if (j < m) {
                __stcg(qa + j, c * x[u] - s * y[u]);
                __stcg(qb + j, s * x[u] + c * y[u]);
              }
            }
          } else {
            double al = 0.0, be = 0.0, ga = 0.0;
            for (int j = lane; j < n; j += 32) {
              const double x = __ldcg(ra + j), y = __ldcg(rb + j);
              al = fma(x, x, al);
              be = fma(y, y, be);
              ga = fma(x, y, ga);
            }
            al = warp_sum(al);
            be = warp_sum(be);
            ga = warp_sum(ga);
            if (!(fabs(ga) > thresh * sqrt(al * be)) || al == 0.0 || be == 0.0) continue;
            const double zeta = (be - al) / (2.0 * ga);
            const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
            for (int j = lane; j < n; j += 32) {
              const double x = __ldcg(ra + j), y = __ldcg(rb + j);
              __stcg(ra + j, c * x - s * y);
              __stcg(rb + j, s * x + c * y);
            }
            for (int j = lane; j < m; j += 32) {
              const double x = __ldcg(qa + j), y = __ldcg(qb + j);
              __stcg(qa + j, c * x - s * y);
              __stcg(qb + j, s * x + c * y);
            }
          }
          ++nrot;  // (warp-uniform)
        }
        cluster_sync_all();
      }
      // sweep done: any rotation? one atomic per warp per sweep (not per rotation)
      if (lane == 0 && nrot) atomicAdd(cnt, nrot);
      nrot = 0;
      cluster_sync_all();
      const int rot = __ldcg(cnt);
      cluster_sync_all();  // everyone has read the counter before it is reset
      if (crank == 0 && threadIdx.x == 0) *cnt = 0;
      if (rot == 0) {
        status = sweep;
        break;
      }
    }
  } else {
    status = 1;
  }
  cluster_sync_all();
  // ---- finalize: sigma_i = |b_i| -> rank (descending, ties by row) -> U, S, Vh
  for (int i = gw; i < m; i += NW) {
    double x2 = 0.0;
    for (int j = lane; j < n; j += 32) {
      const double x = __ldcg(B + (int64_t)i * n + j);
      x2 = fma(x, x, x2);
    }
    x2 = warp_sum(x2);
    if (lane == 0) __stcg(t.norm + i, sqrt(x2));
  }
  cluster_sync_all();
  double smax = 0.0;
  for (int k = lane; k < m; k += 32) smax = fmax(smax, __ldcg(t.norm + k));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) smax = fmax(smax, __shfl_xor_sync(0xffffffffu, smax, o));
  bool deficient = false;
  for (int i = gw; i < m; i += NW) {
    const double si = __ldcg(t.norm + i);
    int rank = 0;
    for (int k = lane; k < m; k += 32) {
      const double sk = __ldcg(t.norm + k);
      rank += (sk > si || (sk == si && k < i)) ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    if (si <= rank_tol * smax) deficient = true;
    if (lane == 0) t.s[rank] = si;
    const double inv = si > 0.0 ? 1.0 / si : 0.0;
    for (int j = lane; j < n; j += 32) t.vh[(int64_t)rank * n + j] = __ldcg(B + (int64_t)i * n + j) * inv;
    for (int j = lane; j < m; j += 32) t.u[(int64_t)j * m + rank] = __ldcg(Q + (int64_t)i * m + j);
  }
  if (deficient && lane == 0) atomicExch(t.status, -2);
  cluster_sync_all();
  if (crank == 0 && threadIdx.x == 0) {
    if (atomicAdd(t.status, 0) != -2) *t.status = status;
  }
}

}  // namespace
}  // namespace tnb

extern "C" int tnb_svd_jacobi_batched(int nsec, const TnbSvdSector* secs, int max_sweeps, double tol,
                                      double rank_tol, void* stream) {
  using namespace tnb;
  int rc = require_device();
  if (rc) return rc;
  if (nsec < 0 || (nsec > 0 && !secs) || max_sweeps < 1) return fail(TNB_EINVAL, "svd_jacobi: bad arguments");
  if (nsec == 0) return TNB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<SvdTask> h(nsec);
  for (int i = 0; i < nsec; ++i) {
    const TnbSvdSector& x = secs[i];
    if (x.m < 1 || x.n < x.m || !x.a || !x.b || !x.q || !x.u || !x.s || !x.vh || !x.status)
      return fail(TNB_EINVAL, "svd_jacobi: sector needs 1 <= m <= n and all buffers");
    h[i] = {static_cast<const double*>(x.a), static_cast<double*>(x.b), static_cast<double*>(x.q),
            static_cast<double*>(x.u),
            static_cast<double*>(x.s), static_cast<double*>(x.vh), x.status, nullptr, nullptr,
            (int)x.m, (int)x.n};
  }
  // device task table + rotation counters + norm / rank scratch in one allocation
  int64_t msum = 0;
  for (int i = 0; i < nsec; ++i) msum += secs[i].m;
  const size_t tb = sizeof(SvdTask) * (size_t)nsec, cb = sizeof(int) * 2 * (size_t)nsec;
  const size_t nb = sizeof(double) * (size_t)msum;
  void* mem = nullptr;
  TNB_CUDA_CHECK(cudaMallocAsync(&mem, tb + nb + cb, st));
  double* norms = reinterpret_cast<double*>(static_cast<char*>(mem) + tb);
  int* counters = reinterpret_cast<int*>(static_cast<char*>(mem) + tb + nb);
  for (int i = 0, off = 0; i < nsec; off += (int)secs[i].m, ++i) {
    h[i].counter = counters + 2 * i;
    h[i].norm = norms + off;
  }
  cudaError_t e = cudaMemcpyAsync(mem, h.data(), tb, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(counters, 0, cb, st);
  for (int i = 0; e == cudaSuccess && i < nsec; ++i) e = cudaMemsetAsync(secs[i].status, 0, sizeof(int), st);
  if (e == cudaSuccess) {
    double work = 0.0;
    for (int i = 0; i < nsec; ++i) work += 2.0 * secs[i].m * (double)secs[i].m * secs[i].n;
    static bool configured = false;
    if (!configured) {
      e = cudaFuncSetAttribute(jacobi_rows_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      configured = e == cudaSuccess;
    }
    if (e == cudaSuccess) {
      KTimer kt(TNB_KF_OTHER, st, work);
      jacobi_rows_kernel<<<nsec * kCluster, kWarps * 32, 0, st>>>(static_cast<const SvdTask*>(mem), max_sweeps,
                                                                    tol, rank_tol);
      e = cudaGetLastError();
    }
  }
  count_launch();
  cudaFreeAsync(mem, st);
  if (e != cudaSuccess) return cuda_fail(e, "svd_jacobi: launch");
  return TNB_OK;
}

// Batched one-sided Jacobi SVD of the charge-sector matrices of a block-sparse tensor
// (the factorisation step of linalg.svd / svd_truncate, pkg/src/tnkit/linalg.py:246-341,
// where the reference calls LAPACK gesdd sector by sector).
//
// Every sector matrix A (m x n, m <= n, row-major, float64 or complex128) is factorised by
// Hestenes' one-sided Jacobi on its ROWS -- rows are contiguous, so every access is a
// coalesced row sweep:  B = Q A with Q orthogonal (product of plane rotations) and the
// rows of B mutually orthogonal; then sigma_i = |b_i|, v_i = b_i / sigma_i, U = Q^H
// (complex pairs: the phase of <b_p, b_q> is rotated out of b_q first, then the real
// rotation applies).
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
// (rank-deficient sectors: product states, degenerate wavefunctions) cannot be normalised
// into V rows; their Vh rows are completed in the same kernel to an orthonormal basis of
// the complement of the kept rows (deterministic pseudo-random starts, two-pass Gram-Schmidt
// against every earlier row, cluster-wide), as LAPACK's gesdd completes V. U = Q^H is
// unitary whatever the rank, so U S Vh = A and both factors stay orthonormal.
#include <cmath>
#include <vector>

#include "common.cuh"

namespace tnb {
namespace {

constexpr int kCluster = 16;  // non-portable cluster size (B200 allows 16)
constexpr int kWarps = 16;
constexpr int kRegU = 10;     // float64 rows up to 640 (10 double2 units per lane) in registers

struct SvdTask {
  const void* a;   // [m][n] in (read only)
  void* b;         // [m][n] workspace: the rotated rows
  void* q;         // [m][m] workspace: accumulated rotations (rows)
  void* u;         // [m][m] out
  double* s;       // [m] out (real)
  void* vh;        // [m][n] out
  int* status;     // [1] out: sweeps used (>0), -1 not converged, -2 rank deficient
  int* counter;    // [2] rotation counters (zero on entry)
  double* norm;    // [m] scratch: |b_i|
  double* coef;    // [2m + 2] scratch: Gram-Schmidt coefficients (re, im) + the candidate's norm
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

// ---- scalar helpers: real (double) and complex (double2) rows -----------------------
template <bool CPLX>
struct Sc;
template <>
struct Sc<false> {
  using T = double;
  static constexpr int kRegPL = 20;  // rows up to 640 long live in registers (20 per lane)
  __device__ static T zero() { return 0.0; }
  __device__ static T one() { return 1.0; }
  __device__ static double abs2(T x) { return x * x; }
  __device__ static void acc2(double& acc, T x) { acc = fma(x, x, acc); }
  // acc += conj(x) * y  (split into re / im accumulators)
  __device__ static void dot(double& re, double& im, T x, T y) { re = fma(x, y, re); }
  __device__ static T conj(T x) { return x; }
  __device__ static T scale(double c, T x) { return c * x; }
  // phase p (unit; +-1 for real rows) times y
  __device__ static T mulph(double pr, double pi, T y) { return pr * y; }
  __device__ static T lin(double c, T x, double s, T y) { return c * x + s * y; }  // c x + s y
};
template <>
struct Sc<true> {
  using T = double2;
  static constexpr int kRegPL = 10;
  __device__ static T zero() { return make_double2(0.0, 0.0); }
  __device__ static T one() { return make_double2(1.0, 0.0); }
  __device__ static double abs2(T x) { return fma(x.x, x.x, x.y * x.y); }
  __device__ static void acc2(double& acc, T x) { acc = fma(x.x, x.x, fma(x.y, x.y, acc)); }
  __device__ static void dot(double& re, double& im, T x, T y) {
    re = fma(x.x, y.x, fma(x.y, y.y, re));
    im = fma(x.x, y.y, fma(-x.y, y.x, im));
  }
  __device__ static T conj(T x) { return make_double2(x.x, -x.y); }
  __device__ static T scale(double c, T x) { return make_double2(c * x.x, c * x.y); }
  __device__ static T mulph(double pr, double pi, T y) {
    return make_double2(fma(pr, y.x, -pi * y.y), fma(pr, y.y, pi * y.x));
  }
  __device__ static T lin(double c, T x, double s, T y) {
    return make_double2(fma(c, x.x, s * y.x), fma(c, x.y, s * y.y));
  }
};

template <typename T>
__device__ __forceinline__ T ldcg(const T* p) {
  return __ldcg(p);
}
template <typename T>
__device__ __forceinline__ void stcg(T* p, T v) {
  __stcg(p, v);
}

// One plane rotation of rows (a, b) of B and Q, given al = |b_a|^2, be = |b_b|^2 and
// g = <b_a, b_b> = |g| e^{i phi}: with b' = e^{-i phi} b_b the real Hestenes rotation on
// (b_a, b') makes them orthogonal; Q rows take the same unitary 2 x 2 map.
// Returns false if the pair is already orthogonal to the threshold.
__device__ __forceinline__ bool rotation(double al, double be, double gre, double gim, double thresh, double& c,
                                         double& s, double& pr, double& pi) {
  const double ga = sqrt(gre * gre + gim * gim);
  if (!(ga > thresh * sqrt(al * be)) || al == 0.0 || be == 0.0) return false;
  pr = gre / ga;  // e^{-i phi} = conj(g) / |g|
  pi = -gim / ga;
  const double zeta = (be - al) / (2.0 * ga);
  const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  c = 1.0 / sqrt(1.0 + tt * tt);
  s = c * tt;
  return true;
}

// deterministic pseudo-random value in [-1, 1) (splitmix64 of the key)
__device__ __forceinline__ double rnd_unit(uint64_t key) {
  uint64_t z = key + 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  z ^= z >> 31;
  return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

// Orthonormal completion of Vh rows [r0, m): row r starts from a pseudo-random vector,
// is orthogonalised (twice) against rows 0 .. r-1 and normalised; all warps of the
// cluster cooperate on every step (rows are sequentially dependent).
template <bool CPLX>
__device__ void complete_rows(typename Sc<CPLX>::T* __restrict__ VH, int r0, int m, int n, double* coef, int gw,
                              int lane) {
  using S = Sc<CPLX>;
  using T = typename S::T;
  constexpr int NW = kCluster * kWarps;
  const int gt = gw * 32 + lane;
  for (int r = r0; r < m; ++r) {
    T* v = VH + (int64_t)r * n;
    for (int attempt = 0; attempt < 8; ++attempt) {
      for (int j = gt; j < n; j += NW * 32) {
        const uint64_t key = ((uint64_t)r << 40) ^ ((uint64_t)attempt << 32) ^ (uint64_t)j;
        if constexpr (CPLX) stcg(v + j, make_double2(rnd_unit(key), rnd_unit(key ^ 0x5555555555555555ull)));
        else stcg(v + j, rnd_unit(key));
      }
      cluster_sync_all();
      double before = 0.0;
      for (int pass = 0; pass < 2; ++pass) {
        // coefficients <v_k, v> of the earlier rows (a warp per row)
        for (int k = gw; k < r; k += NW) {
          double re = 0.0, im = 0.0;
          for (int j = lane; j < n; j += 32) S::dot(re, im, ldcg(VH + (int64_t)k * n + j), ldcg(v + j));
          re = warp_sum(re);
          if constexpr (CPLX) im = warp_sum(im);
          if (lane == 0) {
            __stcg(coef + 2 * k, re);
            __stcg(coef + 2 * k + 1, im);
          }
        }
        if (pass == 0 && gw == 0) {  // the candidate's norm before projection
          double x2 = 0.0;
          for (int j = lane; j < n; j += 32) x2 += S::abs2(ldcg(v + j));
          x2 = warp_sum(x2);
          if (lane == 0) __stcg(coef + 2 * m, x2);
        }
        cluster_sync_all();
        if (pass == 0) before = __ldcg(coef + 2 * m);
        // v -= sum_k <v_k, v> v_k   (a thread per element)
        for (int j = gt; j < n; j += NW * 32) {
          T x = ldcg(v + j);
          for (int k = 0; k < r; ++k) {
            const double cr = __ldcg(coef + 2 * k), ci = __ldcg(coef + 2 * k + 1);
            const T y = ldcg(VH + (int64_t)k * n + j);
            if constexpr (CPLX) {
              x.x -= cr * y.x - ci * y.y;
              x.y -= cr * y.y + ci * y.x;
            } else {
              x -= cr * y;
            }
          }
          stcg(v + j, x);
        }
        cluster_sync_all();
      }
      if (gw == 0) {
        double x2 = 0.0;
        for (int j = lane; j < n; j += 32) x2 += S::abs2(ldcg(v + j));
        x2 = warp_sum(x2);
        if (lane == 0) __stcg(coef + 2 * m + 1, x2);
      }
      cluster_sync_all();
      const double after = __ldcg(coef + 2 * m + 1);
      // accept unless the start lay (numerically) inside the span of the earlier rows
      const bool ok = after > 1e-6 * before && after > 0.0;
      if (ok) {
        const double inv = 1.0 / sqrt(after);
        for (int j = gt; j < n; j += NW * 32) stcg(v + j, S::scale(inv, ldcg(v + j)));
      }
      cluster_sync_all();
      if (ok) break;
    }
  }
}

template <bool CPLX>
__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kWarps * 32)
    jacobi_rows_kernel(const SvdTask* __restrict__ tasks, int max_sweeps, double tol, double rank_tol) {
  using S = Sc<CPLX>;
  using T = typename S::T;
  constexpr int RPL = S::kRegPL;
  const SvdTask t = tasks[blockIdx.x / kCluster];
  const int crank = (int)cluster_rank();
  const int lane = threadIdx.x & 31;
  const int gw = crank * kWarps + (threadIdx.x >> 5);  // warp index within the cluster
  constexpr int NW = kCluster * kWarps;
  const int m = t.m, n = t.n;
  T* __restrict__ B = static_cast<T*>(t.b);
  T* __restrict__ Q = static_cast<T*>(t.q);
  const T* __restrict__ Ain = static_cast<const T*>(t.a);
  // workspace row strides: float64 rows are padded to an even length (zero pad) so a row is
  // a whole number of 16-byte double2 units -- the register path moves 16 B per lane access
  const int ldb = CPLX ? n : n + (n & 1), ldq = CPLX ? m : m + (m & 1);
  // Q = I, B = A
  for (int64_t x = (int64_t)gw * 32 + lane; x < (int64_t)m * ldq; x += (int64_t)NW * 32) {
    const int64_t i = x / ldq, j = x - i * ldq;
    stcg(Q + x, (i == j) ? S::one() : S::zero());
  }
  for (int64_t x = (int64_t)gw * 32 + lane; x < (int64_t)m * ldb; x += (int64_t)NW * 32) {
    const int64_t i = x / ldb, j = x - i * ldb;
    stcg(B + x, j < n ? Ain[i * n + j] : S::zero());
  }
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
          T* ra = B + (int64_t)a * ldb;
          T* rb = B + (int64_t)b * ldb;
          T* qa = Q + (int64_t)a * ldq;
          T* qb = Q + (int64_t)b * ldq;
          double c, s, pr, pi;
          if constexpr (!CPLX) {
            if (ldb <= 64 * kRegU && ldq <= 64 * kRegU) {
              // float64 rows as double2 units in registers: one 16-byte access per lane and unit
              const int nu = ldb >> 1, mu = ldq >> 1;
              const double2* ra2 = reinterpret_cast<const double2*>(ra);
              const double2* rb2 = reinterpret_cast<const double2*>(rb);
              double2 x[kRegU], y[kRegU];
              double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
              for (int u = 0; u < kRegU; ++u) {
                const int j = lane + 32 * u;
                x[u] = j < nu ? __ldcg(ra2 + j) : make_double2(0.0, 0.0);
                y[u] = j < nu ? __ldcg(rb2 + j) : make_double2(0.0, 0.0);
              }
#pragma unroll
              for (int u = 0; u < kRegU; ++u) {
                al = fma(x[u].x, x[u].x, fma(x[u].y, x[u].y, al));
                be = fma(y[u].x, y[u].x, fma(y[u].y, y[u].y, be));
                ga = fma(x[u].x, y[u].x, fma(x[u].y, y[u].y, ga));
              }
              al = warp_sum(al);
              be = warp_sum(be);
              ga = warp_sum(ga);
              if (!rotation(al, be, ga, 0.0, thresh, c, s, pr, pi)) continue;
              const double sp = s * pr, cp = c * pr;  // real phase: +-1
              double2* wa = reinterpret_cast<double2*>(ra);
              double2* wb = reinterpret_cast<double2*>(rb);
#pragma unroll
              for (int u = 0; u < kRegU; ++u) {
                const int j = lane + 32 * u;
                if (j < nu) {
                  __stcg(wa + j, make_double2(c * x[u].x - sp * y[u].x, c * x[u].y - sp * y[u].y));
                  __stcg(wb + j, make_double2(s * x[u].x + cp * y[u].x, s * x[u].y + cp * y[u].y));
                }
              }
              const double2* qa2 = reinterpret_cast<const double2*>(qa);
              const double2* qb2 = reinterpret_cast<const double2*>(qb);
#pragma unroll
              for (int u = 0; u < kRegU; ++u) {
                const int j = lane + 32 * u;
                x[u] = j < mu ? __ldcg(qa2 + j) : make_double2(0.0, 0.0);
                y[u] = j < mu ? __ldcg(qb2 + j) : make_double2(0.0, 0.0);
              }
              double2* va = reinterpret_cast<double2*>(qa);
              double2* vb = reinterpret_cast<double2*>(qb);
#pragma unroll
              for (int u = 0; u < kRegU; ++u) {
                const int j = lane + 32 * u;
                if (j < mu) {
                  __stcg(va + j, make_double2(c * x[u].x - sp * y[u].x, c * x[u].y - sp * y[u].y));
                  __stcg(vb + j, make_double2(s * x[u].x + cp * y[u].x, s * x[u].y + cp * y[u].y));
                }
              }
              ++nrot;
              continue;
            }
          }
          if (CPLX && n <= 32 * RPL && m <= 32 * RPL) {
            // rows held in registers: one L2 round trip for B's rows, one for Q's
            T x[RPL], y[RPL];
            double al = 0.0, be = 0.0, gre = 0.0, gim = 0.0;
#pragma unroll
            for (int u = 0; u < RPL; ++u) {
              const int j = lane + 32 * u;
              x[u] = j < n ? ldcg(ra + j) : S::zero();
              y[u] = j < n ? ldcg(rb + j) : S::zero();
            }
#pragma unroll
            for (int u = 0; u < RPL; ++u) {
              S::acc2(al, x[u]);
              S::acc2(be, y[u]);
              S::dot(gre, gim, x[u], y[u]);
            }
            al = warp_sum(al);
            be = warp_sum(be);
            gre = warp_sum(gre);
            if constexpr (CPLX) gim = warp_sum(gim);
            if (!rotation(al, be, gre, gim, thresh, c, s, pr, pi)) continue;
#pragma unroll
            for (int u = 0; u < RPL; ++u) {
              const int j = lane + 32 * u;
              if (j < n) {
                const T yp = S::mulph(pr, pi, y[u]);
                stcg(ra + j, S::lin(c, x[u], -s, yp));
                stcg(rb + j, S::lin(s, x[u], c, yp));
              }
            }
#pragma unroll
            for (int u = 0; u < RPL; ++u) {
              const int j = lane + 32 * u;
              x[u] = j < m ? ldcg(qa + j) : S::zero();
              y[u] = j < m ? ldcg(qb + j) : S::zero();
            }
#pragma unroll
            for (int u = 0; u < RPL; ++u) {
              const int j = lane + 32 * u;
              if (j < m) {
                const T yp = S::mulph(pr, pi, y[u]);
                stcg(qa + j, S::lin(c, x[u], -s, yp));
                stcg(qb + j, S::lin(s, x[u], c, yp));
              }
            }
          } else {
            double al = 0.0, be = 0.0, gre = 0.0, gim = 0.0;
            for (int j = lane; j < n; j += 32) {
              const T x = ldcg(ra + j), y = ldcg(rb + j);
              S::acc2(al, x);
              S::acc2(be, y);
              S::dot(gre, gim, x, y);
            }
            al = warp_sum(al);
            be = warp_sum(be);
            gre = warp_sum(gre);
            if constexpr (CPLX) gim = warp_sum(gim);
            if (!rotation(al, be, gre, gim, thresh, c, s, pr, pi)) continue;
            for (int j = lane; j < n; j += 32) {
              const T x = ldcg(ra + j), yp = S::mulph(pr, pi, ldcg(rb + j));
              stcg(ra + j, S::lin(c, x, -s, yp));
              stcg(rb + j, S::lin(s, x, c, yp));
            }
            for (int j = lane; j < m; j += 32) {
              const T x = ldcg(qa + j), yp = S::mulph(pr, pi, ldcg(qb + j));
              stcg(qa + j, S::lin(c, x, -s, yp));
              stcg(qb + j, S::lin(s, x, c, yp));
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
  // ---- finalize: sigma_i = |b_i| -> rank (descending, ties by row) -> U = Q^H, S, Vh = B / S
  T* __restrict__ U = static_cast<T*>(t.u);
  T* __restrict__ VH = static_cast<T*>(t.vh);
  for (int i = gw; i < m; i += NW) {
    double x2 = 0.0;
    for (int j = lane; j < n; j += 32) x2 += S::abs2(ldcg(B + (int64_t)i * ldb + j));
    x2 = warp_sum(x2);
    if (lane == 0) __stcg(t.norm + i, sqrt(x2));
  }
  cluster_sync_all();
  double smax = 0.0;
  for (int k = lane; k < m; k += 32) smax = fmax(smax, __ldcg(t.norm + k));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) smax = fmax(smax, __shfl_xor_sync(0xffffffffu, smax, o));
  // rows whose sigma is below rank_tol * sigma_max (they rank last): their Vh rows are
  // completed below instead of normalised
  int nd = 0;
  for (int k = lane; k < m; k += 32) nd += __ldcg(t.norm + k) <= rank_tol * smax ? 1 : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nd += __shfl_xor_sync(0xffffffffu, nd, o);
  for (int i = gw; i < m; i += NW) {
    const double si = __ldcg(t.norm + i);
    int rank = 0;
    for (int k = lane; k < m; k += 32) {
      const double sk = __ldcg(t.norm + k);
      rank += (sk > si || (sk == si && k < i)) ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    if (lane == 0) t.s[rank] = si;
    if (rank < m - nd) {
      const double inv = 1.0 / si;
      for (int j = lane; j < n; j += 32) stcg(VH + (int64_t)rank * n + j, S::scale(inv, ldcg(B + (int64_t)i * ldb + j)));
    }
    for (int j = lane; j < m; j += 32) U[(int64_t)j * m + rank] = S::conj(ldcg(Q + (int64_t)i * ldq + j));
  }
  cluster_sync_all();
  if (nd > 0) complete_rows<CPLX>(VH, m - nd, m, n, t.coef, gw, lane);
  if (crank == 0 && threadIdx.x == 0) *t.status = status;
}

template <bool CPLX>
int launch_jacobi(const void* tasks, int nsec, int max_sweeps, double tol, double rank_tol, double work,
                  cudaStream_t st) {
  auto kern = jacobi_rows_kernel<CPLX>;
  static bool configured = false;
  if (!configured) {
    TNB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    configured = true;
  }
  {
    KTimer kt(TNB_KF_OTHER, st, work);
    kern<<<nsec * kCluster, kWarps * 32, 0, st>>>(static_cast<const SvdTask*>(tasks), max_sweeps, tol, rank_tol);
  }
  count_launch();
  TNB_CUDA_CHECK(cudaGetLastError());
  return TNB_OK;
}

}  // namespace
}  // namespace tnb

extern "C" int tnb_svd_jacobi_batched(int dtype, int nsec, const TnbSvdSector* secs, int max_sweeps, double tol,
                                      double rank_tol, void* stream) {
  using namespace tnb;
  int rc = require_device();
  if (rc) return rc;
  if (dtype != TNB_F64 && dtype != TNB_C128) return fail(TNB_EUNSUP, "svd_jacobi: float64 / complex128 only");
  if (nsec < 0 || (nsec > 0 && !secs) || max_sweeps < 1) return fail(TNB_EINVAL, "svd_jacobi: bad arguments");
  if (nsec == 0) return TNB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<SvdTask> h(nsec);
  int64_t msum = 0;
  double work = 0.0;
  for (int i = 0; i < nsec; ++i) {
    const TnbSvdSector& x = secs[i];
    if (x.m < 1 || x.n < x.m || !x.a || !x.b || !x.q || !x.u || !x.s || !x.vh || !x.status)
      return fail(TNB_EINVAL, "svd_jacobi: sector needs 1 <= m <= n and all buffers");
    h[i] = {x.a, x.b, x.q, x.u, static_cast<double*>(x.s), x.vh, x.status, nullptr, nullptr, nullptr, (int)x.m,
            (int)x.n};
    msum += x.m;
    work += 2.0 * x.m * (double)x.m * x.n;
  }
  // device task table + rotation counters + norm scratch in one allocation
  const size_t tb = sizeof(SvdTask) * (size_t)nsec, cb = sizeof(int) * 2 * (size_t)nsec;
  const size_t nb = sizeof(double) * (size_t)(3 * msum + 2 * nsec);  // norms [m] + coefficients [2m + 2]
  void* mem = nullptr;
  TNB_CUDA_CHECK(cudaMallocAsync(&mem, tb + nb + cb, st));
  double* norms = reinterpret_cast<double*>(static_cast<char*>(mem) + tb);
  int* counters = reinterpret_cast<int*>(static_cast<char*>(mem) + tb + nb);
  for (int i = 0, off = 0; i < nsec; off += 3 * (int)secs[i].m + 2, ++i) {
    h[i].counter = counters + 2 * i;
    h[i].norm = norms + off;
    h[i].coef = norms + off + secs[i].m;
  }
  cudaError_t e = cudaMemcpyAsync(mem, h.data(), tb, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(counters, 0, cb, st);
  for (int i = 0; e == cudaSuccess && i < nsec; ++i) e = cudaMemsetAsync(secs[i].status, 0, sizeof(int), st);
  if (e != cudaSuccess) {
    cudaFreeAsync(mem, st);
    return cuda_fail(e, "svd_jacobi: task upload");
  }
  rc = dtype == TNB_F64 ? launch_jacobi<false>(mem, nsec, max_sweeps, tol, rank_tol, work, st)
                        : launch_jacobi<true>(mem, nsec, max_sweeps, tol, rank_tol, work, st);
  cudaFreeAsync(mem, st);
  return rc;
}

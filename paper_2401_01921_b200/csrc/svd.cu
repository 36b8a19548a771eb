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
// One thread-block CLUSTER (16 CTAs) owns one sector and B / Q live in global memory read
// with .cg loads (L2; the 126 MB L2 holds every sector of a C4-sized two-site tensor). All
// sectors run concurrently, one cluster each. Two schedules of the same rotations:
//  * jacobi_block_kernel (default): rows in blocks, a tournament over block pairs, each CTA
//    staging its pair's rows in shared memory and doing their Gram matrix, one inner
//    Jacobi sweep and the row / Q updates on chip (DMMA for the products) -- one cluster
//    barrier per block round (see the section comment below);
//  * jacobi_rows_kernel (sectors whose staged rows cannot fit in shared memory, i.e. rows
//    longer than ~13k float64 elements): a warp rotates one row pair per task and the
//    cluster barrier (barrier.cluster arrive.release / wait.acquire) separates rounds. The finalize pass (same kernel) ranks the
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
  int bsz, nb;     // block kernel: rows per block, blocks (a multiple of 2 x kCluster)
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
  // (one sqrt, one division, one reciprocal square root on the dependent chain -- the
  // block kernel's inner rounds wait on it -- instead of three sqrt and four divisions)
  const double g2 = gre * gre + gim * gim;
  if (!(g2 > thresh * thresh * (al * be)) || al == 0.0 || be == 0.0) return false;
  double ga;
  if (gim == 0.0) {  // real rows: the phase is the sign
    ga = fabs(gre);
    pr = copysign(1.0, gre);
    pi = 0.0;
  } else {
    ga = sqrt(g2);
    const double inv = 1.0 / ga;
    pr = gre * inv;  // e^{-i phi} = conj(g) / |g|
    pi = -gim * inv;
  }
  // tan of the rotation angle, Rutishauser's stable form: t = sign(d) 2|g| / (|d| + sqrt(d^2 + 4|g|^2))
  const double d = be - al;
  const double tt = copysign(2.0 * ga, d) / (fabs(d) + sqrt(fma(d, d, 4.0 * g2)));
  c = rsqrt(fma(tt, tt, 1.0));
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
                              int lane, int NW) {
  using S = Sc<CPLX>;
  using T = typename S::T;
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

// ---- finalize: sigma_i = |b_i| -> rank (descending, ties by row) -> U = Q^H, S, Vh = B / S
template <bool CPLX>
__device__ void finalize_sector(const SvdTask& t, const typename Sc<CPLX>::T* __restrict__ B,
                                const typename Sc<CPLX>::T* __restrict__ Q, int ldb, int ldq, int status,
                                double rank_tol, int gw, int lane, int crank, int NW) {
  using S = Sc<CPLX>;
  using T = typename S::T;
  const int m = t.m, n = t.n;
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
  if (nd > 0) complete_rows<CPLX>(VH, m - nd, m, n, t.coef, gw, lane, NW);
  if (crank == 0 && threadIdx.x == 0) *t.status = status;
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
  finalize_sector<CPLX>(t, B, Q, ldb, ldq, status, rank_tol, gw, lane, crank, NW);
}

// ===================================================================== block Jacobi
// Blocked one-sided Jacobi (the round-robin tournament over BLOCKS of rows): the rows are
// split into nb blocks of bsz rows; in every round the 16 CTAs of the sector's cluster
// each take one pair of blocks (I, J), stage its h <= 2 bsz rows W in shared memory, form
// their Gram matrix G = W W^H with DMMA, run one cyclic Jacobi sweep on G (the same
// Hestenes rotation of rows p, q -- applied as G <- J G J^H and accumulated as V <- J V),
// and rewrite the rows as V W (B) and V Q_R (the matching rows of Q) with DMMA. One
// cluster barrier per round instead of one per row-pair round: a sweep of an m x n sector
// moves every row through L2 (m / bsz) times instead of m times, and the rotations'
// arithmetic (6 m^2 n FMA per sweep) runs on the tensor pipe. Convergence as for the
// row kernel: a sweep in which no pair (whichever block pair it met in) needed rotating.
constexpr int kBlkSmemMax = 220 * 1024;
// 17 warps: a block pair of h <= 34 rows has <= 17 row pairs per inner round, one warp each
// (with 16, warp 0 took two and set every round's latency)
constexpr int kBlkWarps = 17;
constexpr int kSortSweeps = 3;  // sweeps that start by sorting the rows by norm (1 / 3 / all: 13 / 13 / 13
                                // sweeps at 516^2, 12 / 11 / 12 at 256^2)

__host__ __device__ __forceinline__ int blk_hp(int bsz) { return ((2 * bsz + 7) / 8) * 8; }
// shared-memory row stride of the staged rows (elements): >= n, 4 mod 16 doubles (two
// doubles per complex element) so the DMMA fragment loads of 4 rows hit distinct banks
__host__ __device__ __forceinline__ int blk_ldw(int n, bool cplx) {
  const int e = cplx ? 2 : 1;
  int w = ((n * e + 15) / 16) * 16 + 4;
  return w / e;
}
__host__ __device__ __forceinline__ size_t blk_smem(int bsz, int n, bool cplx) {
  const int hp = blk_hp(bsz), es = cplx ? 16 : 8;
  return (size_t)hp * blk_ldw(n, cplx) * es + 2 * (size_t)hp * (hp + 1) * es + (size_t)(hp / 2) * 4 * 8 +
         (size_t)hp * 8;  // W, G, V, rotations, row indices, pairs
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <bool CPLX>
struct Frag;
template <>
struct Frag<false> {
  // C (8 x 8) += A (8 x 4) B (4 x 8)
  __device__ static void mma(double (&c)[2][2], double a, double b) { dmma884(c[0][0], c[0][1], a, b); }
  // C += A B^H (B given as its 8 x 4 rows: b = B^T fragment)
  __device__ static void mma_h(double (&c)[2][2], double a, double b) { dmma884(c[0][0], c[0][1], a, b); }
  __device__ static double re(double x) { return x; }
};
template <>
struct Frag<true> {
  // complex A B: re = Ar Br - Ai Bi, im = Ar Bi + Ai Br (c[0] = re pair, c[1] = im pair)
  __device__ static void mma(double (&c)[2][2], double2 a, double2 b) {
    dmma884(c[0][0], c[0][1], a.x, b.x);
    dmma884(c[0][0], c[0][1], -a.y, b.y);
    dmma884(c[1][0], c[1][1], a.x, b.y);
    dmma884(c[1][0], c[1][1], a.y, b.x);
  }
  // A conj(B): re = Ar Br + Ai Bi, im = Ai Br - Ar Bi
  __device__ static void mma_h(double (&c)[2][2], double2 a, double2 b) {
    dmma884(c[0][0], c[0][1], a.x, b.x);
    dmma884(c[0][0], c[0][1], a.y, b.y);
    dmma884(c[1][0], c[1][1], a.y, b.x);
    dmma884(c[1][0], c[1][1], -a.x, b.y);
  }
};

template <bool CPLX>
__device__ __forceinline__ typename Sc<CPLX>::T frag_out(const double (&c)[2][2], int e) {
  if constexpr (CPLX) return make_double2(c[0][e], c[1][e]);
  else return c[0][e];
}

// Out (h x ncols, rows R in global, row stride ld) = V (hp x hp) X (hp x ncols, smem stride ldw).
// A warp computes an 8 x 16 output tile (one V fragment feeds two DMMAs); K runs over the
// first round4(h) rows only (rows h.. of X are zero).
template <bool CPLX>
__device__ void blk_apply(const typename Sc<CPLX>::T* __restrict__ V, int ldv, const typename Sc<CPLX>::T* __restrict__ X,
                          int ldw, int h, int hp, int ncols, typename Sc<CPLX>::T* __restrict__ out, int ld,
                          const int* rows, int warp, int lane) {
  using T = typename Sc<CPLX>::T;
  const int tiles_i = (h + 7) / 8, tiles_j = (ncols + 15) / 16, kend = (h + 3) & ~3;
  const int r = lane >> 2, q = lane & 3;
  for (int tt = warp; tt < tiles_i * tiles_j; tt += kBlkWarps) {
    const int ti = tt % tiles_i, tj = tt / tiles_i;
    const int i0 = ti * 8, j0 = tj * 16;
    double c0[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, c1[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    const bool two = j0 + 8 < ncols;
    for (int k0 = 0; k0 < kend; k0 += 4) {
      const T a = V[(i0 + r) * ldv + k0 + q];
      const T* xb = X + (k0 + q) * ldw + j0 + r;
      Frag<CPLX>::mma(c0, a, xb[0]);
      if (two) Frag<CPLX>::mma(c1, a, xb[8]);
    }
    const int i = i0 + r;
    if (i < h) {
      T* dst = out + (int64_t)rows[i] * ld;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = j0 + 2 * q + e;
        if (j < ncols) stcg(dst + j, frag_out<CPLX>(c0, e));
        if (j + 8 < ncols) stcg(dst + j + 8, frag_out<CPLX>(c1, e));
      }
    }
  }
}

// W[i][0, ncols) = src row rows[i] (i < h) by 16-byte cp.async (rows are 16-byte aligned:
// float64 workspace rows have even length), zero elsewhere in [0, hp) x [0, ldw); the
// copies are all in flight at once (a load -> store loop would wait out each L2 round trip)
template <bool CPLX>
__device__ void blk_stage(typename Sc<CPLX>::T* __restrict__ W, int ldw, const typename Sc<CPLX>::T* __restrict__ src,
                          int ld, const int* rows, int h, int hp, int ncols, int tid) {
  using T = typename Sc<CPLX>::T;
  constexpr int EPC = CPLX ? 1 : 2;  // elements per 16-byte chunk
  const int cpr = ncols / EPC;        // chunks per row (ncols is even for float64)
  for (int x = tid; x < h * cpr; x += blockDim.x) {
    const int i = x / cpr, c = x - i * cpr;
    TNB_DCHECK(i < hp && c * EPC + EPC <= ldw, "svd blk_stage range");
    const T* g = src + (int64_t)rows[i] * ld + c * EPC;
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(W + i * ldw + c * EPC);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(g));
  }
  const int tail = ldw - ncols;
  for (int x = tid; x < h * tail; x += blockDim.x) {
    const int i = x / tail;
    W[i * ldw + ncols + (x - i * tail)] = Sc<CPLX>::zero();
  }
  for (int x = h * ldw + tid; x < hp * ldw; x += blockDim.x) W[x] = Sc<CPLX>::zero();
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

template <bool CPLX>
__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kBlkWarps * 32, 1)
    jacobi_block_kernel(const SvdTask* __restrict__ tasks, int max_sweeps, double tol, double rank_tol) {
  using S = Sc<CPLX>;
  using T = typename S::T;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_rot;
  const SvdTask t = tasks[blockIdx.x / kCluster];
  const int crank = (int)cluster_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gw = crank * kBlkWarps + warp;
  constexpr int NW = kCluster * kBlkWarps;
  const int m = t.m, n = t.n, bsz = t.bsz, nb = t.nb;
  T* __restrict__ B = static_cast<T*>(t.b);
  T* __restrict__ Q = static_cast<T*>(t.q);
  const T* __restrict__ Ain = static_cast<const T*>(t.a);
  const int ldb = CPLX ? n : n + (n & 1), ldq = CPLX ? m : m + (m & 1);
  const int hp = blk_hp(bsz), ldw = blk_ldw(n, CPLX), ldg = hp + 1;
  T* W = reinterpret_cast<T*>(smem);
  T* G = W + (size_t)hp * ldw;
  T* V = G + (size_t)hp * ldg;
  double* rot = reinterpret_cast<double*>(V + (size_t)hp * ldg);  // [hp / 2][4]: c, s, pr, pi
  int* rows = reinterpret_cast<int*>(rot + (hp / 2) * 4);           // [hp]
  int* prs = rows + hp;                                              // [hp]: this round's pairs
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
  const double thresh = tol * sqrt((double)n) * 2.220446049250313e-16;
  int sweep = 0, status = -1;
  if (m > 1) {
    for (sweep = 1; sweep <= max_sweeps; ++sweep) {
      int* cnt = t.counter + (sweep & 1);
      if (tid == 0) s_rot = 0;
      if (sweep <= kSortSweeps) {
        // rows sorted by decreasing norm at the start of the first sweeps (de Rijk's ordering:
        // 516 x 516 14 -> 13 sweeps, 256 x 256 12 -> 11): B, Q rows -> the output buffers
        // (scratch until the finalize) in rank order, then back
        T* __restrict__ VHs = static_cast<T*>(t.vh);
        T* __restrict__ Us = static_cast<T*>(t.u);
        for (int i = gw; i < m; i += NW) {
          double x2 = 0.0;
          for (int j = lane; j < n; j += 32) x2 += S::abs2(ldcg(B + (int64_t)i * ldb + j));
          x2 = warp_sum(x2);
          if (lane == 0) __stcg(t.norm + i, x2);
        }
        cluster_sync_all();
        for (int i = gw; i < m; i += NW) {
          const double si = __ldcg(t.norm + i);
          int rank = 0;
          for (int k = lane; k < m; k += 32) {
            const double sk = __ldcg(t.norm + k);
            rank += (sk > si || (sk == si && k < i)) ? 1 : 0;
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
          for (int j = lane; j < n; j += 32) stcg(VHs + (int64_t)rank * n + j, ldcg(B + (int64_t)i * ldb + j));
          for (int j = lane; j < m; j += 32) stcg(Us + (int64_t)rank * m + j, ldcg(Q + (int64_t)i * ldq + j));
        }
        cluster_sync_all();
        for (int i = gw; i < m; i += NW) {
          for (int j = lane; j < n; j += 32) stcg(B + (int64_t)i * ldb + j, ldcg(VHs + (int64_t)i * n + j));
          for (int j = lane; j < m; j += 32) stcg(Q + (int64_t)i * ldq + j, ldcg(Us + (int64_t)i * m + j));
        }
        cluster_sync_all();
      }
      for (int r = 0; r < nb - 1; ++r) {
        for (int pi_ = crank; pi_ < nb / 2; pi_ += kCluster) {
          int I, J;
          rr_pair(nb, r, pi_, I, J);
          const int i0 = I * bsz, i1 = min(m, i0 + bsz), j0 = J * bsz, j1 = min(m, j0 + bsz);
          const int hI = max(0, i1 - i0), hJ = max(0, j1 - j0), h = hI + hJ;
          if (h < 2 || (r > 0 && (hI == 0 || hJ == 0))) continue;  // nothing to rotate (CTA-uniform)
          __syncthreads();      // the previous pair's smem reads are done
          for (int i = tid; i < hp; i += blockDim.x) rows[i] = i < hI ? i0 + i : (i < h ? j0 + i - hI : 0);
          __syncthreads();
          blk_stage<CPLX>(W, ldw, B, ldb, rows, h, hp, ldb, tid);  // W = B[rows]
          // V = I
          for (int x = tid; x < hp * ldg; x += blockDim.x) {
            const int i = x / ldg, j = x - i * ldg;
            V[x] = (i == j) ? S::one() : S::zero();
          }
          __syncthreads();
          // G = W W^H: 8 x 8 tiles on and above the diagonal, mirrored
          {
            const int ti_n = (h + 7) / 8, ntile = ti_n * (ti_n + 1) / 2;  // (G rows / columns >= h stay unused)
            const int rr = lane >> 2, qq = lane & 3;
            for (int tt = warp; tt < ntile; tt += kBlkWarps) {
              int ti = 0, rem = tt;
              while (rem >= ti_n - ti) {
                rem -= ti_n - ti;
                ++ti;
              }
              const int tj = ti + rem;
              double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
              const T* wa = W + (ti * 8 + rr) * ldw + qq;
              const T* wb = W + (tj * 8 + rr) * ldw + qq;
              for (int k0 = 0; k0 < ldb; k0 += 4) Frag<CPLX>::mma_h(c, wa[k0], wb[k0]);
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int gi = ti * 8 + rr, gj = tj * 8 + 2 * qq + e;
                const T v = frag_out<CPLX>(c, e);
                G[gi * ldg + gj] = v;
                if (ti != tj) G[gj * ldg + gi] = S::conj(v);  // (a diagonal tile holds both)
              }
            }
          }
          __syncthreads();
          // one cyclic Jacobi sweep over the h rows, on G (two-sided) and V (rows). Per round:
          // the npair rotations (one thread each), then ONE update phase in which a thread
          // applies rotation k to rows {p, q} and rotation k' to columns {p', q'} of a 2 x 2
          // block of G at once (G <- J G J^H), or rotation k to a column of rows {p, q} of V
          // The first block round of a sweep visits every pair of the h rows (a round-robin
          // tournament, h - 1 rounds); later rounds only the cross pairs I x J (max(hI, hJ)
          // rounds of min(hI, hJ) disjoint pairs): every pair of rows of the sector is still
          // visited at least once per sweep -- within-block pairs in round 0, where every block
          // plays -- so a sweep without rotations still means B did not change during it.
          // (A row in no pair of an inner round still needs that round's column rotations in
          // its row of G: the |hI - hJ| rows left over by the cross pairs of unequal blocks
          // ride along in identity "pairs", two to a pair, the last with the spare row h.)
          const bool cross = r > 0;
          const int hh = h + (h & 1);
          const int nreal = cross ? min(hI, hJ) : hh / 2;
          const int npair = cross ? nreal + (abs(hI - hJ) + 1) / 2 : nreal;
          const int nround = cross ? max(hI, hJ) : hh - 1;
          for (int ir = 0; ir < nround; ++ir) {
            if (tid < 32) {  // (npair <= hp / 2 <= 32: warp 0 computes every rotation)
              // pair `tid` of inner round ir (no integer divisions)
              int p = 0, q = 0;
              bool idle = false;
              if (tid < npair) {
                if (cross) {
                  // the larger block (n rows, offset o) cycles against the smaller one: its
                  // row (t + ir) mod n meets row t of the smaller block, t < nreal; rows
                  // t >= nreal of the cycle are idle this round
                  const bool iBig = hI > hJ;
                  const int n = iBig ? hI : hJ, o = iBig ? 0 : hI, so = iBig ? hI : 0;
                  auto big = [&](int t) {
                    int x = t + ir;
                    if (x >= n) x -= n;
                    return o + x;
                  };
                  if (tid < nreal) {
                    p = so + tid;
                    q = big(tid);
                  } else {
                    idle = true;
                    const int t = nreal + 2 * (tid - nreal);
                    p = big(t);
                    q = t + 1 < n ? big(t + 1) : h;  // (h: the spare row, h < hp when used)
                  }
                } else {
                  const int M = hh - 1;
                  if (tid == 0) {
                    p = ir;
                    q = M;
                  } else {
                    p = ir + tid;
                    if (p >= M) p -= M;
                    q = ir - tid;
                    if (q < 0) q += M;
                  }
                }
              }
              if (p > q) {
                const int x = p;
                p = q;
                q = x;
              }
              double c = 1.0, sn = 0.0, pr = 1.0, pim = 0.0;
              bool did = false;
              if (tid < npair && q < h && !idle) {
                // <b_p, b_q> = sum conj(b_p) b_q = G[q][p]
                const T g = G[q * ldg + p];
                double gre, gim, al, be;
                if constexpr (CPLX) {
                  gre = g.x;
                  gim = g.y;
                  al = G[p * ldg + p].x;
                  be = G[q * ldg + q].x;
                } else {
                  gre = g;
                  gim = 0.0;
                  al = G[p * ldg + p];
                  be = G[q * ldg + q];
                }
                did = rotation(al, be, gre, gim, thresh, c, sn, pr, pim);
                if (!did) {
                  c = 1.0;
                  sn = 0.0;
                  pr = 1.0;
                  pim = 0.0;
                }
              }
              const unsigned nrot_w = __popc(__ballot_sync(0xffffffffu, did));  // (no same-address atomics)
              if (tid == 0) s_rot += (int)nrot_w;
              if (tid < npair) {
                rot[4 * tid] = c;
                rot[4 * tid + 1] = sn;
                rot[4 * tid + 2] = pr;
                rot[4 * tid + 3] = pim;
                prs[2 * tid] = p;
                prs[2 * tid + 1] = q;
              }
            }
            __syncthreads();
            // warp w takes row pairs k = w, w + 16: lane l updates the G block (rows of pair k) x
            // (columns of pair l) and columns l, l + 32 of V's rows p, q
            for (int k = warp; k < npair; k += kBlkWarps) {
              const double s1 = rot[4 * k + 1];
              const int p = prs[2 * k], q = prs[2 * k + 1];
              const double c1 = rot[4 * k], pr1 = rot[4 * k + 2], pi1 = rot[4 * k + 3];
              if (lane < npair) {
                const int k2 = lane;
                const double s2 = rot[4 * k2 + 1];
                if (s1 != 0.0 || s2 != 0.0) {
                  const int p2 = prs[2 * k2], q2 = prs[2 * k2 + 1];
                  T a00 = G[p * ldg + p2], a01 = G[p * ldg + q2], a10 = G[q * ldg + p2], a11 = G[q * ldg + q2];
                  if (s1 != 0.0) {  // rows: x_p' = c x_p - s ph x_q, x_q' = s x_p + c ph x_q
                    const T y0 = S::mulph(pr1, pi1, a10), y1 = S::mulph(pr1, pi1, a11);
                    const T n00 = S::lin(c1, a00, -s1, y0), n01 = S::lin(c1, a01, -s1, y1);
                    a10 = S::lin(s1, a00, c1, y0);
                    a11 = S::lin(s1, a01, c1, y1);
                    a00 = n00;
                    a01 = n01;
                  }
                  if (s2 != 0.0) {  // columns: g_p' = c g_p - s conj(ph) g_q, g_q' = s g_p + c conj(ph) g_q
                    const double c = rot[4 * k2], pr = rot[4 * k2 + 2], pim = rot[4 * k2 + 3];
                    const T y0 = S::mulph(pr, -pim, a01), y1 = S::mulph(pr, -pim, a11);
                    const T n00 = S::lin(c, a00, -s2, y0), n10 = S::lin(c, a10, -s2, y1);
                    a01 = S::lin(s2, a00, c, y0);
                    a11 = S::lin(s2, a10, c, y1);
                    a00 = n00;
                    a10 = n10;
                  }
                  G[p * ldg + p2] = a00;
                  G[p * ldg + q2] = a01;
                  G[q * ldg + p2] = a10;
                  G[q * ldg + q2] = a11;
                }
              }
              if (s1 != 0.0) {
                for (int col = lane; col < hp; col += 32) {
                  T* vp = V + p * ldg + col;
                  T* vq = V + q * ldg + col;
                  const T yp = *vp, yq = S::mulph(pr1, pi1, *vq);
                  *vp = S::lin(c1, yp, -s1, yq);
                  *vq = S::lin(s1, yp, c1, yq);
                }
              }
            }
            __syncthreads();
          }
          // B[rows] = V W ; then Q[rows] = V Q[rows]
          blk_apply<CPLX>(V, ldg, W, ldw, h, hp, ldb, B, ldb, rows, warp, lane);
          __syncthreads();
          blk_stage<CPLX>(W, ldw, Q, ldq, rows, h, hp, ldq, tid);  // W = Q[rows]
          __syncthreads();
          blk_apply<CPLX>(V, ldg, W, ldw, h, hp, ldq, Q, ldq, rows, warp, lane);
        }
        cluster_sync_all();
      }
      __syncthreads();
      if (tid == 0 && s_rot) atomicAdd(cnt, s_rot);
      cluster_sync_all();
      const int rot_all = __ldcg(cnt);
      cluster_sync_all();  // everyone has read the counter before it is reset
      if (crank == 0 && tid == 0) *cnt = 0;
      if (rot_all == 0) {
        status = sweep;
        break;
      }
    }
  } else {
    status = 1;
  }
  cluster_sync_all();
  finalize_sector<CPLX>(t, B, Q, ldb, ldq, status, rank_tol, gw, lane, crank, NW);
}

template <bool CPLX>
int launch_jacobi(const void* tasks, int nsec, int max_sweeps, double tol, double rank_tol, double work,
                  size_t block_smem, cudaStream_t st) {
  auto kern = block_smem ? jacobi_block_kernel<CPLX> : jacobi_rows_kernel<CPLX>;
  static bool configured[2] = {false, false};
  if (!configured[block_smem ? 1 : 0]) {
    TNB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    if (block_smem) TNB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kBlkSmemMax));
    configured[block_smem ? 1 : 0] = true;
  }
  {
    KTimer kt(TNB_KF_OTHER, st, work);
    kern<<<nsec * kCluster, (block_smem ? kBlkWarps : kWarps) * 32, block_smem, st>>>(static_cast<const SvdTask*>(tasks), max_sweeps, tol,
                                                           rank_tol);
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
            (int)x.n, 1, 2};
    msum += x.m;
    work += 2.0 * x.m * (double)x.m * x.n;
  }
  // block kernel: ~one block pair per CTA and round (nb = 2 x cluster blocks, or one row per
  // block below that), more blocks where 2 bsz staged rows would not fit in shared memory;
  // a sector whose single-row blocks still do not fit takes the whole batch to the row kernel
  const bool cplx = dtype == TNB_C128;
  static const bool rows_only = getenv("TNB_SVD_ROWS") != nullptr;  // dev A/B switch
  size_t block_smem = 0;
  bool block_ok = !rows_only;
  for (int i = 0; i < nsec && block_ok; ++i) {
    const int m = h[i].m, n = h[i].n;
    int nb = std::min(2 * kCluster, m + (m & 1));
    int bsz = (m + nb - 1) / nb;
    while ((blk_smem(bsz, n, cplx) > kBlkSmemMax || blk_hp(bsz) > 64) && bsz > 1) {  // (warp 0: <= 32 pairs)
      nb += 2 * kCluster;
      bsz = (m + nb - 1) / nb;
    }
    if (blk_smem(bsz, n, cplx) > kBlkSmemMax) block_ok = false;
    h[i].bsz = bsz;
    h[i].nb = std::max(2, nb);
    block_smem = std::max(block_smem, blk_smem(bsz, n, cplx));
  }
  if (!block_ok) block_smem = 0;
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
  rc = dtype == TNB_F64 ? launch_jacobi<false>(mem, nsec, max_sweeps, tol, rank_tol, work, block_smem, st)
                        : launch_jacobi<true>(mem, nsec, max_sweeps, tol, rank_tol, work, block_smem, st);
  cudaFreeAsync(mem, st);
  return rc;
}

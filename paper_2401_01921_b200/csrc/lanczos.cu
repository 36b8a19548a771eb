// One Lanczos orthogonalisation step on the device (the vector work of
// pkg/src/tnkit/linalg.py:474-562 around each matvec), with alpha / beta kept in HBM:
//
//   c_k   = <q_k, w>            k = 0 .. r-1   (Krylov basis Q stored as r ROWS of length n)
//   alpha = Re c_{r-1}
//   w    -= sum_k c_k q_k                      (full reorthogonalisation; it also removes the
//                                               alpha q_{r-1} and beta q_{r-2} terms of the
//                                               three-term recurrence the reference subtracts
//                                               explicitly before its reorthogonalisation)
//   beta  = |w|,  q_r = w / beta               (when beta > 0; the host handles breakdown)
//
// Three HBM-bound launches, no host synchronisation: (1) per-chunk partial dots of every
// basis row with w (the chunk of w staged in shared memory, a warp per row), the last CTA
// reducing the partials in chunk order; (2) the update w -= Q^T c with per-CTA partial
// squared norms, the last CTA reducing them in order (beta) and recording alpha / beta;
// (3) q_r = w / beta. Deterministic: every reduction runs in a fixed order. With r = 0 the
// step only normalises (the start vector).
#include <cmath>

#include "common.cuh"

namespace tnb {
namespace {

constexpr int kChunk = 2048;  // elements of w per CTA
constexpr int kThreads = 256;

template <bool CPLX>
struct Lv;
template <>
struct Lv<false> {
  using T = double;
  __device__ static void dot(double& re, double& im, T q, T w) { re = fma(q, w, re); }
  __device__ static T axpy(T w, double cr, double ci, T q) { return fma(-cr, q, w); }
  __device__ static double abs2(T x) { return x * x; }
  __device__ static T scale(double s, T x) { return s * x; }
};
template <>
struct Lv<true> {
  using T = double2;
  // conj(q) * w
  __device__ static void dot(double& re, double& im, T q, T w) {
    re = fma(q.x, w.x, fma(q.y, w.y, re));
    im = fma(q.x, w.y, fma(-q.y, w.x, im));
  }
  // w - c q
  __device__ static T axpy(T w, double cr, double ci, T q) {
    return make_double2(w.x - (cr * q.x - ci * q.y), w.y - (cr * q.y + ci * q.x));
  }
  __device__ static double abs2(T x) { return fma(x.x, x.x, x.y * x.y); }
  __device__ static T scale(double s, T x) { return make_double2(s * x.x, s * x.y); }
};

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Deterministic CTA-wide sum: thread t adds elements t, t + kThreads, ... of its own
// subset in order, then a fixed-shape tree over the threads (smem `red`, kThreads doubles).
__device__ double cta_sum_fixed(const double* v, int64_t count, int64_t stride, double* red) {
  double s = 0.0;
  for (int64_t c = threadIdx.x; c < count; c += kThreads) s += __ldcg(v + c * stride);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int h = kThreads / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  const double out = red[0];
  __syncthreads();
  return out;
}

struct LzWork {
  double* part;    // [nchunks][r][2] partial dots
  double* coef;    // [r][2] reduced coefficients c_k
  double* npart;   // [nchunks] partial squared norms
  int* counter;    // [2] last-CTA counters (self-resetting)
  double* alpha;   // out: alpha
  double* beta;    // out: beta
};

template <bool CPLX>
__global__ void __launch_bounds__(kThreads) lz_project(const typename Lv<CPLX>::T* __restrict__ Q, int64_t ldq, int r,
                                                       const typename Lv<CPLX>::T* __restrict__ w, int64_t n,
                                                       LzWork wk) {
  using L = Lv<CPLX>;
  using T = typename L::T;
  __shared__ T ws[kChunk];
  __shared__ bool last;
  const int64_t j0 = (int64_t)blockIdx.x * kChunk;
  const int len = (int)min64(kChunk, n - j0);
  for (int x = threadIdx.x; x < len; x += kThreads) ws[x] = w[j0 + x];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kThreads / 32;
  for (int k = warp; k < r; k += nw) {
    const T* q = Q + (int64_t)k * ldq + j0;
    // 4 independent partial sums per lane keep 4 loads in flight; combined in a fixed order
    double re[4] = {0.0, 0.0, 0.0, 0.0}, im[4] = {0.0, 0.0, 0.0, 0.0};
    int x = lane;
    for (; x + 96 < len; x += 128) {
      const T a0 = __ldcs(q + x), a1 = __ldcs(q + x + 32), a2 = __ldcs(q + x + 64), a3 = __ldcs(q + x + 96);
      L::dot(re[0], im[0], a0, ws[x]);
      L::dot(re[1], im[1], a1, ws[x + 32]);
      L::dot(re[2], im[2], a2, ws[x + 64]);
      L::dot(re[3], im[3], a3, ws[x + 96]);
    }
    for (; x < len; x += 32) L::dot(re[0], im[0], __ldcs(q + x), ws[x]);
    double sre = warp_sum((re[0] + re[1]) + (re[2] + re[3]));
    double sim = CPLX ? warp_sum((im[0] + im[1]) + (im[2] + im[3])) : 0.0;
    if (lane == 0) {
      wk.part[((int64_t)blockIdx.x * r + k) * 2] = sre;
      wk.part[((int64_t)blockIdx.x * r + k) * 2 + 1] = sim;
    }
  }
  // the last CTA to finish reduces the partials in chunk order (deterministic)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(wk.counter, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double red[kThreads];
  for (int k = 0; k < r; ++k) {
    const double re = cta_sum_fixed(wk.part + 2 * (int64_t)k, gridDim.x, 2 * (int64_t)r, red);
    const double im = CPLX ? cta_sum_fixed(wk.part + 2 * (int64_t)k + 1, gridDim.x, 2 * (int64_t)r, red) : 0.0;
    if (threadIdx.x == 0) {
      wk.coef[2 * k] = re;
      wk.coef[2 * k + 1] = im;
    }
  }
  if (threadIdx.x == 0) *wk.counter = 0;
}

template <bool CPLX>
__global__ void __launch_bounds__(kThreads) lz_update(const typename Lv<CPLX>::T* __restrict__ Q, int64_t ldq, int r,
                                                      typename Lv<CPLX>::T* __restrict__ w, int64_t n, LzWork wk) {
  using L = Lv<CPLX>;
  using T = typename L::T;
  extern __shared__ double cs[];  // [r][2]
  __shared__ double red[kThreads];
  __shared__ bool last;
  for (int x = threadIdx.x; x < 2 * r; x += kThreads) cs[x] = __ldcg(wk.coef + x);
  __syncthreads();
  const int64_t j0 = (int64_t)blockIdx.x * kChunk;
  const int len = (int)min64(kChunk, n - j0);
  // each thread owns kEl elements; every basis row is one round of kEl independent loads
  constexpr int kEl = kChunk / kThreads;
  T v[kEl];
#pragma unroll
  for (int e = 0; e < kEl; ++e) {
    const int x = threadIdx.x + e * kThreads;
    if (x < len) v[e] = w[j0 + x];
  }
  for (int k = 0; k < r; ++k) {
    const T* q = Q + (int64_t)k * ldq + j0;
    const double cr = cs[2 * k], ci = cs[2 * k + 1];
#pragma unroll
    for (int e = 0; e < kEl; ++e) {
      const int x = threadIdx.x + e * kThreads;
      if (x < len) v[e] = L::axpy(v[e], cr, ci, __ldcs(q + x));
    }
  }
  double nrm = 0.0;
#pragma unroll
  for (int e = 0; e < kEl; ++e) {
    const int x = threadIdx.x + e * kThreads;
    if (x < len) {
      w[j0 + x] = v[e];
      nrm += L::abs2(v[e]);
    }
  }
  nrm = warp_sum(nrm);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) s += red[i];
    wk.npart[blockIdx.x] = s;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(wk.counter + 1, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const double s2 = cta_sum_fixed(wk.npart, gridDim.x, 1, red);
  if (threadIdx.x == 0) {
    *wk.beta = sqrt(s2);
    *wk.alpha = r > 0 ? cs[2 * (r - 1)] : 0.0;
    wk.counter[1] = 0;
  }
}

template <bool CPLX>
__global__ void __launch_bounds__(kThreads) lz_normalise(const typename Lv<CPLX>::T* __restrict__ w,
                                                         typename Lv<CPLX>::T* __restrict__ qn, int64_t n,
                                                         const double* beta) {
  using L = Lv<CPLX>;
  const double b = *beta;
  const double inv = b > 0.0 ? 1.0 / b : 0.0;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    qn[j] = L::scale(inv, w[j]);
}

template <bool CPLX>
int run(const void* Q, int64_t ldq, int r, void* w, int64_t n, void* q_next, double* alpha, double* beta,
        void* work, cudaStream_t st) {
  using T = typename Lv<CPLX>::T;
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  if (nchunks >= (1ll << 31)) return fail(TNB_EUNSUP, "lanczos_step: vector too long");
  char* p = static_cast<char*>(work);
  LzWork wk;
  wk.counter = reinterpret_cast<int*>(p);
  wk.coef = reinterpret_cast<double*>(p + 16);
  wk.part = wk.coef + 2 * (int64_t)r;
  wk.npart = wk.part + 2 * (int64_t)r * nchunks;
  wk.alpha = alpha;
  wk.beta = beta;
  if (r > 0) {
    {
      KTimer kt(TNB_KF_OTHER, st, (double)(r + 1) * n * sizeof(T));
      lz_project<CPLX><<<(unsigned)nchunks, kThreads, 0, st>>>(static_cast<const T*>(Q), ldq, r,
                                                               static_cast<const T*>(w), n, wk);
    }
    count_launch();
    TNB_CUDA_CHECK(cudaGetLastError());
  }
  const size_t smem = (size_t)16 * (r > 0 ? r : 1);
  if (smem > 48 * 1024) TNB_CUDA_CHECK(cudaFuncSetAttribute(lz_update<CPLX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                            (int)smem));
  {
    KTimer kt(TNB_KF_OTHER, st, (double)(r + 2) * n * sizeof(T));
    lz_update<CPLX><<<(unsigned)nchunks, kThreads, smem, st>>>(static_cast<const T*>(Q), ldq, r, static_cast<T*>(w),
                                                               n, wk);
  }
  count_launch();
  TNB_CUDA_CHECK(cudaGetLastError());
  if (q_next) {
    const int64_t grid = std::min<int64_t>((n + kThreads - 1) / kThreads, (int64_t)sm_count() * 8);
    KTimer kt(TNB_KF_OTHER, st, 2.0 * n * sizeof(T));
    lz_normalise<CPLX><<<(unsigned)grid, kThreads, 0, st>>>(static_cast<const T*>(w), static_cast<T*>(q_next), n,
                                                            beta);
    count_launch();
    TNB_CUDA_CHECK(cudaGetLastError());
  }
  return TNB_OK;
}

}  // namespace
}  // namespace tnb

extern "C" int64_t tnb_lanczos_work_bytes(int r, int64_t n) {
  const int64_t nchunks = (n + tnb::kChunk - 1) / tnb::kChunk;
  return 16 + 8 * (2 * (int64_t)r + 2 * (int64_t)r * nchunks + nchunks);
}

extern "C" int tnb_lanczos_step(int dtype, const void* q, int64_t ldq, int r, void* w, int64_t n, void* q_next,
                                double* alpha, double* beta, void* work, void* stream) {
  using namespace tnb;
  int rc = require_device();
  if (rc) return rc;
  if (dtype != TNB_F64 && dtype != TNB_C128) return fail(TNB_EUNSUP, "lanczos_step: float64 / complex128 only");
  if (r < 0 || n < 1 || ldq < n || (r > 0 && !q) || !w || !alpha || !beta || !work)
    return fail(TNB_EINVAL, "lanczos_step: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  return dtype == TNB_F64 ? run<false>(q, ldq, r, w, n, q_next, alpha, beta, work, st)
                          : run<true>(q, ldq, r, w, n, q_next, alpha, beta, work, st);
}

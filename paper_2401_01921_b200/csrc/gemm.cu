// a11: dense pairwise contraction on FP64 tensor cores (DMMA) -- the B200
// replacement for np.tensordot(a.view(), b.view(), axes=(a_pos, b_pos)) +
// np.ascontiguousarray (pkg/src/tnkit/contract.py:127-132).
//
// The contraction is a GEMM C[M,N] = A[M,K] . B[K,N] whose operands are read
// IN PLACE from the reference's storage model (buffer + lazy permutation): the
// permute is fused into the operand loads. Each operand index group (A rows,
// A contracted, B contracted, B cols) is a short list of (dim, stride) digits;
// a row/col offset table is built once per CTA tile and a K offset table once
// per k-tile (per stage), so every element address is
//     base + row_off[m] + k_off[k]
// and the cp.async gathers go straight into shared memory.
//
// Math: mma.sync.m8n8k4 f64 (SASS DMMA.8x8x4), the FP64 tensor-core path on
// sm_100a (tcgen05 has no f64 kind). Complex128 is either 4M (four real DMMAs
// per fragment pair, exact products) or 3M (Gauss: three real DMMAs; (Ar+Ai),
// (Br+Bi) formed from the staged fragments in registers).
//
// Tile shape and split-K are chosen per problem on the host to fill the 148 SMs;
// split-K partials are reduced by a second deterministic kernel (fixed order,
// no atomics). Very skinny problems (N, K <= 64: e.g. the MPO step of
// L.A.W.R) go to a separate memory-bound kernel.
#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <mutex>
#include <cstring>
#include <vector>

#include "gemm_sk.cuh"

namespace tnb {

int permute_device(const void* src, void* dst, int es, int rank, const int64_t* shape, const int32_t* perm,
                   cudaStream_t st);

namespace {



// Warp-specialised dense tile GEMM (producer warpgroup + DMMA warps).
template <bool CPLX, int MODE, int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES>
__global__ void __launch_bounds__(WARPS_M* WARPS_N * 32 + 128, 1)
    gemm_ws_kernel(const typename Elem<CPLX>::T* __restrict__ A, const typename Elem<CPLX>::T* __restrict__ B,
                   typename Elem<CPLX>::T* __restrict__ C, const __grid_constant__ GemmDesc d) {
  using Core = TileCoreWS<CPLX, MODE, BM, BN, BK, WARPS_M, WARPS_N, STAGES, 0, 0>;
  extern __shared__ __align__(16) unsigned char smem[];
  int bid = blockIdx.x;
  const int split = bid % d.splitk;
  bid /= d.splitk;
  int tm, tn;
  {
    const int group = 8;
    const int per_group = group * d.tiles_n;
    const int g = bid / per_group;
    const int first_m = g * group;
    const int gsz = min(d.tiles_m - first_m, group);
    const int in_g = bid - g * per_group;
    tm = first_m + in_g % gsz;
    tn = in_g / gsz;
  }
  const int m0 = tm * BM, n0 = tn * BN;
  const int kbeg = split * d.k_per_split;
  const int kend = min(d.K, kbeg + d.k_per_split);
  typename Core::Acc acc;
  Core::zero(acc);
  bool math;
  if (d.a_mfast) {
    if (d.b_nfast) math = Core::template run<true, true>(smem, A, B, d.rowA, d.kA, d.kB, d.colB, m0, n0, d.M, d.N, kbeg, kend, d.kaff, acc);
    else math = Core::template run<true, false>(smem, A, B, d.rowA, d.kA, d.kB, d.colB, m0, n0, d.M, d.N, kbeg, kend, d.kaff, acc);
  } else {
    if (d.b_nfast) math = Core::template run<false, true>(smem, A, B, d.rowA, d.kA, d.kB, d.colB, m0, n0, d.M, d.N, kbeg, kend, d.kaff, acc);
    else math = Core::template run<false, false>(smem, A, B, d.rowA, d.kA, d.kB, d.colB, m0, n0, d.M, d.N, kbeg, kend, d.kaff, acc);
  }
  if (math)
    Core::store(C + (size_t)split * (size_t)d.M * (size_t)d.out_ld, d.out_ld, m0, n0, d.M, d.N, acc);
}

// Persistent stream-K warp-specialised GEMM (SKCore): the dense contraction path.
template <bool CPLX, int MODE, int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool AMF, bool BNF>
__global__ void __launch_bounds__(WARPS_M* WARPS_N * 32 + 128, 1)
    gemm_sk_kernel(const typename Elem<CPLX>::T* __restrict__ A, const typename Elem<CPLX>::T* __restrict__ B,
                   typename Elem<CPLX>::T* __restrict__ C, const __grid_constant__ GemmDesc d, const SKParams sk) {
  extern __shared__ __align__(16) unsigned char smem[];
  SKCore<CPLX, MODE, BM, BN, BK, WARPS_M, WARPS_N, STAGES>::template run<AMF, BNF>(smem, A, B, C, d, sk);
}

// Dense tile GEMM: one CTA per (tile, K split); tile raster in groups of 8
// tile-rows so concurrently running CTAs share B panels in L2.
template <bool CPLX, int MODE, int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, int MINB>
__global__ void __launch_bounds__(WARPS_M* WARPS_N * 32, MINB)
    gemm_kernel(const typename Elem<CPLX>::T* __restrict__ A, const typename Elem<CPLX>::T* __restrict__ B,
                typename Elem<CPLX>::T* __restrict__ C, const __grid_constant__ GemmDesc d) {
  using Core = TileCore<CPLX, MODE, BM, BN, BK, WARPS_M, WARPS_N, STAGES>;
  extern __shared__ __align__(16) unsigned char smem[];
  pdl_launch_dependents();  // (pdl_wait: in the mainloop, after the index tables)
  int bid = blockIdx.x;
  const int split = bid % d.splitk;
  bid /= d.splitk;
  int tm, tn;
  {
    const int group = 8;
    const int per_group = group * d.tiles_n;
    const int g = bid / per_group;
    const int first_m = g * group;
    const int gsz = min(d.tiles_m - first_m, group);
    const int in_g = bid - g * per_group;
    tm = first_m + in_g % gsz;
    tn = in_g / gsz;
  }
  const int m0 = tm * BM, n0 = tn * BN;
  const int kbeg = split * d.k_per_split;
  const int kend = min(d.K, kbeg + d.k_per_split);
  typename Core::Acc acc;
  Core::zero(acc);
  Core::mainloop(smem, A, B, d.rowA, d.kA, d.kB, d.colB, m0, n0, d.M, d.N, kbeg, kend, d.a_mfast != 0,
                 d.b_nfast != 0, acc);
  Core::store(C + (size_t)split * (size_t)d.M * (size_t)d.out_ld, d.out_ld, m0, n0, d.M, d.N, acc);
}

// split-K reduction: out[i] = sum_{s in order} ws[s][i]
template <bool CPLX>
__global__ void splitk_reduce_kernel(const typename Elem<CPLX>::T* __restrict__ ws,
                                     typename Elem<CPLX>::T* __restrict__ out, int64_t n, int S) {
  pdl_wait();
  pdl_launch_dependents();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    if constexpr (!CPLX) {
      double s = ws[i];
      for (int q = 1; q < S; ++q) s += ws[(size_t)q * n + i];
      out[i] = s;
    } else {
      double2 s = ws[i];
      for (int q = 1; q < S; ++q) {
        double2 v = ws[(size_t)q * n + i];
        s.x += v.x;
        s.y += v.y;
      }
      out[i] = s;
    }
  }
}

// ------------------------------------------------------------------ dot kernel
// C[M, N] with M * N <= 16 and any K (a (nearly) fully contracted step, e.g. the closing
// a* contraction of a PEPS site: M = N = 1, K = 8192): memory-bound, no tensor-core tile
// to fill. CTA c sums its contiguous K chunk for every output (thread-strided k, fixed
// shuffle tree, warps summed in order) and writes one partial per output;
// splitk_reduce_kernel then adds the CTA partials in CTA order -- deterministic.
template <bool CPLX>
__global__ void __launch_bounds__(256) dot_kernel(const typename Elem<CPLX>::T* __restrict__ A,
                                                  const typename Elem<CPLX>::T* __restrict__ B,
                                                  typename Elem<CPLX>::T* __restrict__ ws,
                                                  const __grid_constant__ GemmDesc d, int64_t kchunk) {
  using T = typename Elem<CPLX>::T;
  constexpr int MAXMN = 16;
  __shared__ int64_t rowOff[MAXMN], colOff[MAXMN];
  __shared__ T red[8][MAXMN];
  const int M = d.M, N = d.N, MN = M * N;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < M) rowOff[tid] = group_offset(d.rowA, tid);
  if (tid >= 32 && tid - 32 < N) colOff[tid - 32] = group_offset(d.colB, tid - 32);
  __syncthreads();
  const int64_t kb = (int64_t)blockIdx.x * kchunk;
  const int64_t ke = min64((int64_t)d.K, kb + kchunk);
  double re[MAXMN], im[MAXMN];
#pragma unroll
  for (int j = 0; j < MAXMN; ++j) re[j] = im[j] = 0.0;
  for (int64_t k = kb + tid; k < ke; k += blockDim.x) {
    const int64_t oa = group_offset(d.kA, (uint32_t)k), ob = group_offset(d.kB, (uint32_t)k);
#pragma unroll
    for (int m = 0; m < MAXMN; ++m) {
      if (m >= M) break;
      const T a = __ldcs(A + rowOff[m] + oa);
#pragma unroll
      for (int n = 0; n < MAXMN; ++n) {
        if (n >= N || m * N + n >= MAXMN) break;
        const T b = __ldg(B + colOff[n] + ob);
        const int j = m * N + n;
        if constexpr (!CPLX) {
          re[j] = fma(a, b, re[j]);
        } else {
          re[j] = fma(a.x, b.x, re[j]);
          re[j] = fma(-a.y, b.y, re[j]);
          im[j] = fma(a.x, b.y, im[j]);
          im[j] = fma(a.y, b.x, im[j]);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < MAXMN; ++j) {
    if (j >= MN) break;
    double x = re[j], y = im[j];
    for (int o = 16; o > 0; o >>= 1) {
      x += __shfl_xor_sync(0xffffffffu, x, o);
      if constexpr (CPLX) y += __shfl_xor_sync(0xffffffffu, y, o);
    }
    if (lane == 0) {
      if constexpr (!CPLX) red[warp][j] = x;
      else red[warp][j] = make_double2(x, y);
    }
  }
  __syncthreads();
  if (tid < MN) {
    T s = red[0][tid];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      if constexpr (!CPLX) s += red[w][tid];
      else s = make_double2(s.x + red[w][tid].x, s.y + red[w][tid].y);
    }
    ws[(int64_t)blockIdx.x * MN + tid] = s;
  }
}

// ------------------------------------------------------------------ narrow kernel
// C[M, N] for N <= 16, K <= 32 (the T1.W step of L.A.W.R: N = K = 10): HBM-bound.
// One warp owns 32 consecutive rows (one per lane): a lane issues all K gathered
// loads of its row before any FMA (K loads in flight per lane, no block barrier),
// multiplies by B held in shared memory (broadcast reads), stages the 32 x N
// outputs -- one contiguous run of C -- in a per-warp smem tile and writes them
// with consecutive lanes on consecutive addresses.
template <bool CPLX, int NMAX, int KMAX, int WARPS = (CPLX ? 4 : 8)>
__global__ void __launch_bounds__(WARPS * 32) narrow_kernel(const typename Elem<CPLX>::T* __restrict__ A,
                                                     const typename Elem<CPLX>::T* __restrict__ B,
                                                     typename Elem<CPLX>::T* __restrict__ C,
                                                     const __grid_constant__ GemmDesc d) {
  using T = typename Elem<CPLX>::T;
  __shared__ T Bs[KMAX * NMAX];
  __shared__ int64_t kA[KMAX];
  __shared__ T stage[WARPS][32 * NMAX + 1];
  pdl_wait();
  pdl_launch_dependents();
  const int K = d.K, N = d.N;
  for (int i = threadIdx.x; i < K; i += blockDim.x) kA[i] = group_offset(d.kA, i);
  for (int i = threadIdx.x; i < K * N; i += blockDim.x) {
    const int k = i / N, n = i - k * N;
    Bs[k * NMAX + n] = B[group_offset(d.kB, k) + group_offset(d.colB, n)];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T* st = stage[warp];
  const int64_t nchunks = ((int64_t)d.M + 31) / 32;
  for (int64_t ch = (int64_t)blockIdx.x * WARPS + warp; ch < nchunks; ch += (int64_t)gridDim.x * WARPS) {
    const int64_t r0 = ch * 32;
    const int64_t r = r0 + lane;
    const int rows = (int)(d.M - r0 < 32 ? d.M - r0 : 32);
    T a[KMAX];
    if (r < d.M) {
      const int64_t ro = group_offset(d.rowA, (uint32_t)r);
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < K) a[k] = __ldcs(A + ro + kA[k]);
    }
    if constexpr (!CPLX) {
      double acc[NMAX];
#pragma unroll
      for (int n = 0; n < NMAX; ++n) acc[n] = 0.0;
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < K)
#pragma unroll
          for (int n = 0; n < NMAX; ++n) acc[n] = fma(a[k], Bs[k * NMAX + n], acc[n]);
#pragma unroll
      for (int n = 0; n < NMAX; ++n)
        if (n < N) st[lane * N + n] = acc[n];
    } else {
      double ar[NMAX], ai[NMAX];
#pragma unroll
      for (int n = 0; n < NMAX; ++n) ar[n] = ai[n] = 0.0;
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < K)
#pragma unroll
          for (int n = 0; n < NMAX; ++n) {
            const double2 b = Bs[k * NMAX + n];
            ar[n] = fma(a[k].x, b.x, ar[n]);
            ar[n] = fma(-a[k].y, b.y, ar[n]);
            ai[n] = fma(a[k].x, b.y, ai[n]);
            ai[n] = fma(a[k].y, b.x, ai[n]);
          }
#pragma unroll
      for (int n = 0; n < NMAX; ++n)
        if (n < N) st[lane * N + n] = make_double2(ar[n], ai[n]);
    }
    __syncwarp();
    T* out = C + r0 * N;
    const int tot = rows * N;
    for (int i = lane; i < tot; i += 32) __stcs(out + i, st[i]);
    __syncwarp();
  }
}

// Row-panel variant for the layout the T1.W step of L.A.W.R really has (T1[p][vr][b][w],
// rows (vr, b), contracted (w, p)): the contracted index splits into an INNER digit of
// stride 1 (w, extent Kin) and outer digits (p), and consecutive rows step by exactly Kin.
// Then, for a panel of ROWS consecutive rows inside one run of the innermost row digit,
// each outer k value j covers ONE contiguous span of ROWS * Kin elements, and the panel's
// ROWS x N outputs are one contiguous run of C. Every warp runs its own pipeline over its
// panels: the TMA engine moves the spans into a 3-deep ring of shared-memory panels
// (cp.async.bulk, completion counted in bytes on one mbarrier per slot) and the finished
// panel back out (cp.async.bulk shared -> global), so the LSU only serves the FMA operands
// -- the per-lane 8-byte gathers of narrow_kernel touch a sector per lane and its stores
// go through the L1 a sector at a time.
struct SlabDesc {
  int kin, kout;
  int64_t so[32];         // element offset of outer k value j (added to the panel's row offset)
  int16_t soff[32];       // k -> offset in the staged panel: j * ROWS * Kin + kin
};

template <bool CPLX, int NMAX, int KMAX, int WARPS, int ROWS, bool EXACT>
__global__ void __launch_bounds__(WARPS * 32) narrow_slab_kernel(const typename Elem<CPLX>::T* __restrict__ A,
                                                          const typename Elem<CPLX>::T* __restrict__ B,
                                                          typename Elem<CPLX>::T* __restrict__ C,
                                                          const __grid_constant__ GemmDesc d,
                                                          const __grid_constant__ SlabDesc s) {
  using T = typename Elem<CPLX>::T;
  constexpr int ES = CPLX ? 16 : 8;
#ifndef TNB_SLAB_NB
#define TNB_SLAB_NB 2
#endif
  constexpr int NB = TNB_SLAB_NB;  // panels in the ring (2 / 4 warps: 34.8 us at chi = 1024 f64, 3 / 2: 36.6)
  constexpr int RPL = ROWS / 32;  // rows per lane, multiplied together (one B read feeds all)
  static_assert(NMAX % 2 == 0, "B rows are read as pairs");
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(16) T Bs[KMAX * NMAX];
  __shared__ __align__(8) uint64_t bars[WARPS][NB];
  const int K = EXACT ? KMAX : d.K, N = EXACT ? NMAX : d.N;  // EXACT: sizes known at compile time
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int panel = ROWS * K, outsz = ROWS * N;  // elements
  T* wbase = reinterpret_cast<T*>(smem) + (size_t)warp * (NB * panel + outsz);
  T* out = wbase + NB * panel;
  uint64_t* bar = bars[warp];
  pdl_wait();
  pdl_launch_dependents();
  for (int i = threadIdx.x; i < KMAX * NMAX; i += blockDim.x) {
    const int k = i / NMAX, n = i - k * NMAX;
    T v;
    if constexpr (CPLX) v = make_double2(0.0, 0.0);
    else v = 0.0;
    if (k < K && n < N) v = B[group_offset(d.kB, k) + group_offset(d.colB, n)];
    Bs[i] = v;
  }
  if (lane == 0) {
    for (int b = 0; b < NB; ++b) detail::mbar_init(&bar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int64_t npan = (int64_t)d.M / ROWS;
  const int64_t step = (int64_t)gridDim.x * WARPS;
  const uint32_t span_bytes = (uint32_t)(ROWS * s.kin * ES);
  auto issue = [&](int64_t pn, int b) {  // lane 0 only
    const T* src = A + group_offset(d.rowA, (uint32_t)(pn * ROWS));
    TNB_DCHECK(group_offset(d.rowA, (uint32_t)(pn * ROWS)) + ROWS * s.kin <= d.a_elems, "narrow_slab panel row range");
    const uint32_t dst = smem_u32(wbase + b * panel);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar[b])),
                 "r"(span_bytes * (uint32_t)s.kout)
                 : "memory");
    for (int j = 0; j < s.kout; ++j) {
      TNB_DCHECK(src + s.so[j] - A >= 0 && src + s.so[j] - A + ROWS * s.kin <= d.a_elems, "narrow_slab span");
      detail::bulk_load(dst + j * span_bytes, src + s.so[j], span_bytes, &bar[b]);
    }
  };
  const int64_t first = (int64_t)blockIdx.x * WARPS + warp;
  if (lane == 0)
    for (int b = 0; b < NB; ++b)
      if (first + b * step < npan) issue(first + b * step, b);
  int it = 0;
  for (int64_t pn = first; pn < npan; pn += step, ++it) {
    const int b = it % NB;
    detail::mbar_wait(&bar[b], (uint32_t)(it / NB) & 1);
    const T* buf = wbase + b * panel;
    // the previous panel's bulk store must have finished READING the out buffer
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    __syncwarp();
    if constexpr (!CPLX) {
      double acc[RPL][NMAX];
#pragma unroll
      for (int h = 0; h < RPL; ++h)
#pragma unroll
        for (int n = 0; n < NMAX; ++n) acc[h][n] = 0.0;
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < K) {
          double a[RPL];
#pragma unroll
          for (int h = 0; h < RPL; ++h) a[h] = buf[(h * 32 + lane) * s.kin + s.soff[k]];
#pragma unroll
          for (int n = 0; n < NMAX; n += 2) {
            const double2 bb = *reinterpret_cast<const double2*>(&Bs[k * NMAX + n]);
#pragma unroll
            for (int h = 0; h < RPL; ++h) {
              acc[h][n] = fma(a[h], bb.x, acc[h][n]);
              acc[h][n + 1] = fma(a[h], bb.y, acc[h][n + 1]);
            }
          }
        }
#pragma unroll
      for (int h = 0; h < RPL; ++h) {
        double* o = out + (h * 32 + lane) * N;
        if ((N & 1) == 0) {
#pragma unroll
          for (int n = 0; n < NMAX; n += 2)
            if (n < N) *reinterpret_cast<double2*>(o + n) = make_double2(acc[h][n], acc[h][n + 1]);
        } else {
#pragma unroll
          for (int n = 0; n < NMAX; ++n)
            if (n < N) o[n] = acc[h][n];
        }
      }
    } else {
#pragma unroll
      for (int h = 0; h < RPL; ++h) {
        double ar[NMAX], ai[NMAX];
#pragma unroll
        for (int n = 0; n < NMAX; ++n) ar[n] = ai[n] = 0.0;
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
          if (k < K) {
            const double2 a = buf[(h * 32 + lane) * s.kin + s.soff[k]];
#pragma unroll
            for (int n = 0; n < NMAX; ++n) {
              const double2 bb = Bs[k * NMAX + n];
              ar[n] = fma(a.x, bb.x, ar[n]);
              ar[n] = fma(-a.y, bb.y, ar[n]);
              ai[n] = fma(a.x, bb.y, ai[n]);
              ai[n] = fma(a.y, bb.x, ai[n]);
            }
          }
        double2* o = out + (h * 32 + lane) * N;
#pragma unroll
        for (int n = 0; n < NMAX; ++n)
          if (n < N) o[n] = make_double2(ar[n], ai[n]);
      }
    }
    // generic-proxy writes of the out buffer -> visible to the bulk store (async proxy)
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(C + pn * ROWS * N),
                   "r"(smem_u32(out)), "r"((uint32_t)(outsz * ES))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      // every lane's reads of slot b are complete (their values fed the outputs): refill it
      if (pn + NB * step < npan) issue(pn + NB * step, b);
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// host mirror of group_offset
int64_t host_group_offset(const Group& g, uint32_t idx) {
  int64_t off = 0;
  for (int q = g.n - 1; q >= 0; --q) {
    const uint32_t dig = idx % (uint32_t)g.dim[q];
    idx /= (uint32_t)g.dim[q];
    off += (int64_t)dig * g.stride[q];
  }
  return off;
}

// The row-panel layout of narrow_slab_kernel, if the operand has it.
bool slab_layout(const GemmDesc& d, int es, const void* A, const void* C, int kRows, SlabDesc& s) {
  memset(&s, 0, sizeof(s));
  if (d.rowA.n < 1 || d.kA.n < 1 || d.K > 32 || d.M % kRows) return false;
  // the contracted digit of stride 1
  int qi = -1;
  for (int q = 0; q < d.kA.n; ++q)
    if (d.kA.stride[q] == 1) qi = q;
  if (qi < 0) return false;
  const int kin = d.kA.dim[qi];
  const int rq = d.rowA.n - 1;  // innermost row digit: consecutive rows step by kin
  if (d.rowA.stride[rq] != kin || d.rowA.dim[rq] % kRows) return false;
  s.kin = kin;
  s.kout = d.K / kin;
  if (s.kout * kin != d.K || s.kout > 32) return false;
  // enumerate k: (outer offset -> j, kin digit)
  std::vector<int64_t> outers;
  for (int k = 0; k < d.K; ++k) {
    uint32_t idx = (uint32_t)k;
    int64_t outer = 0;
    int kd = 0;
    for (int q = d.kA.n - 1; q >= 0; --q) {
      const int dig = (int)(idx % (uint32_t)d.kA.dim[q]);
      idx /= (uint32_t)d.kA.dim[q];
      if (q == qi) kd = dig;
      else outer += (int64_t)dig * d.kA.stride[q];
    }
    int j = -1;
    for (size_t x = 0; x < outers.size(); ++x)
      if (outers[x] == outer) j = (int)x;
    if (j < 0) {
      j = (int)outers.size();
      outers.push_back(outer);
      if (j >= 32) return false;
      s.so[j] = outer;
    }
    s.soff[k] = (int16_t)(j * kRows * kin + kd);
  }
  if ((int)outers.size() != s.kout) return false;
  // bulk copies: every span starts 16-byte aligned (panel row offsets: outer row digits'
  // strides and the panel step kRows * kin; outer k offsets; the base pointer) and every
  // output run too
  bool al = (reinterpret_cast<uintptr_t>(A) % 16) == 0;
  for (int q = 0; q < rq; ++q) al = al && (d.rowA.stride[q] * es) % 16 == 0;
  for (int j = 0; j < s.kout; ++j) al = al && (s.so[j] * es) % 16 == 0;
  if (!al || (kRows * kin * es) % 16 || (kRows * d.N * es) % 16 || (reinterpret_cast<uintptr_t>(C) % 16)) return false;
  return true;
}

template <bool CPLX, int NMAX, int KMAX>
int run_narrow(const void* A, const void* B, void* C, const GemmDesc& d, cudaStream_t st) {
  using T = typename Elem<CPLX>::T;
  constexpr int WARPS = CPLX ? 4 : 8;
  auto kern = narrow_kernel<CPLX, NMAX, KMAX, WARPS>;
  static int per_sm = 0;
  if (per_sm == 0) {
    TNB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WARPS * 32, 0));
    if (per_sm < 1) per_sm = 1;
  }
  SlabDesc sd;
  static const bool no_slab = getenv("TNB_NO_SLAB") != nullptr;  // dev A/B switch
#ifndef TNB_SLAB_SW
#define TNB_SLAB_SW 4
#endif
#ifndef TNB_SLAB_ROWS
#define TNB_SLAB_ROWS 64
#endif
  constexpr int SROWS = CPLX ? 32 : TNB_SLAB_ROWS, SW = TNB_SLAB_SW;
  if (!no_slab && slab_layout(d, CPLX ? 16 : 8, A, C, SROWS, sd)) {
    auto sk = (d.K == KMAX && d.N == NMAX) ? narrow_slab_kernel<CPLX, NMAX, KMAX, SW, SROWS, true>
                                           : narrow_slab_kernel<CPLX, NMAX, KMAX, SW, SROWS, false>;
    const size_t smem = (size_t)SW * (TNB_SLAB_NB * SROWS * d.K + SROWS * d.N) * (CPLX ? 16 : 8);
    // occupancy per (kernel, shared-memory size), set up once each
    static std::mutex mu;
    static std::vector<std::pair<std::pair<const void*, size_t>, int>> occ_cache;
    int slab_per_sm = 0;
    {
      std::lock_guard<std::mutex> lk(mu);
      for (auto& e : occ_cache)
        if (e.first.first == (const void*)sk && e.first.second == smem) slab_per_sm = e.second;
      if (!slab_per_sm) {
        TNB_CUDA_CHECK(cudaFuncSetAttribute(sk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        TNB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&slab_per_sm, sk, SW * 32, smem));
        if (slab_per_sm < 1) slab_per_sm = 1;
        occ_cache.push_back({{(const void*)sk, smem}, slab_per_sm});
      }
    }
    const int64_t panels = d.M / SROWS;
    const int64_t grid = std::min<int64_t>((panels + SW - 1) / SW, (int64_t)sm_count() * slab_per_sm);
    {
      KTimer kt(TNB_KF_GEMM_SKINNY, st, 2.0 * d.M * (double)d.N * d.K * (CPLX ? 4 : 1));
      TNB_CUDA_CHECK(launch_pdl(sk, (unsigned)grid, SW * 32, smem, st, static_cast<const T*>(A),
                                static_cast<const T*>(B), static_cast<T*>(C), d, sd));
    }
    count_launch();
    TNB_CUDA_CHECK(cudaGetLastError());
    return TNB_OK;
  }
  const int64_t chunks = ((int64_t)d.M + 31) / 32;
  const int64_t grid = std::min<int64_t>((chunks + WARPS - 1) / WARPS, (int64_t)sm_count() * per_sm);
  {
    KTimer kt(TNB_KF_GEMM_SKINNY, st, 2.0 * d.M * (double)d.N * d.K * (CPLX ? 4 : 1));
    TNB_CUDA_CHECK(launch_pdl(kern, (unsigned)grid, WARPS * 32, 0, st, static_cast<const T*>(A),
                              static_cast<const T*>(B), static_cast<T*>(C), d));
  }
  count_launch();
  TNB_CUDA_CHECK(cudaGetLastError());
  return TNB_OK;
}

// ------------------------------------------------------------------ skinny kernel
// C[M, N] with N <= 64 and K <= 64: memory-bound. Each CTA stages a 128-row
// panel of A (gathered through the offset groups) and all of B in shared
// memory, computes its 128 x N outputs with FMAs, and writes the panel --
// which is one contiguous run of C -- coalesced.
template <bool CPLX>
__global__ void __launch_bounds__(256) skinny_kernel(const typename Elem<CPLX>::T* __restrict__ A,
                                                     const typename Elem<CPLX>::T* __restrict__ B,
                                                     typename Elem<CPLX>::T* __restrict__ C, const __grid_constant__ GemmDesc d) {
  using T = typename Elem<CPLX>::T;
  constexpr int RM = 128;
  extern __shared__ __align__(16) unsigned char smem[];
  const int K = d.K, N = d.N;
  T* Bs = reinterpret_cast<T*>(smem);          // [K][N]
  T* As = Bs + K * N;                          // [RM][K+1]
  T* Cs = As + RM * (K + 1);                   // [RM * N]
  int64_t* kA = reinterpret_cast<int64_t*>(Cs + RM * N);  // [K]
  int64_t* rA = kA + K;                                   // [RM]
  const int tid = threadIdx.x;
  for (int i = tid; i < K; i += blockDim.x) kA[i] = group_offset(d.kA, i);
  for (int i = tid; i < K * N; i += blockDim.x) {
    int k = i / N, n = i - k * N;
    Bs[i] = B[group_offset(d.kB, k) + group_offset(d.colB, n)];
  }
  for (int m0 = blockIdx.x * RM; m0 < d.M; m0 += gridDim.x * RM) {
    const int rows = min(RM, d.M - m0);
    __syncthreads();
    for (int i = tid; i < rows; i += blockDim.x) rA[i] = group_offset(d.rowA, m0 + i);
    __syncthreads();
    for (int i = tid; i < rows * K; i += blockDim.x) {
      int r = i / K, k = i - r * K;
      As[r * (K + 1) + k] = __ldg(A + rA[r] + kA[k]);
    }
    __syncthreads();
    for (int i = tid; i < rows * N; i += blockDim.x) {
      int r = i / N, n = i - r * N;
      const T* a = As + r * (K + 1);
      if constexpr (!CPLX) {
        double s = 0.0;
        for (int k = 0; k < K; ++k) s = fma(a[k], Bs[k * N + n], s);
        Cs[i] = s;
      } else {
        double sr = 0.0, si = 0.0;
        for (int k = 0; k < K; ++k) {
          double2 x = a[k], y = Bs[k * N + n];
          sr = fma(x.x, y.x, sr);
          sr = fma(-x.y, y.y, sr);
          si = fma(x.x, y.y, si);
          si = fma(x.y, y.x, si);
        }
        Cs[i] = make_double2(sr, si);
      }
    }
    __syncthreads();
    T* out = C + (size_t)m0 * N;
    for (int i = tid; i < rows * N; i += blockDim.x) out[i] = Cs[i];
  }
}

// ------------------------------------------------------------------ host side
struct Digit {
  int64_t dim, stride;
};

bool build_group(const std::vector<Digit>& digs, Group& g, int64_t& total) {
  memset(&g, 0, sizeof(g));
  total = 1;
  for (auto& x : digs) total *= x.dim;
  if ((int)digs.size() > kMaxDig) return false;
  g.n = (int)digs.size();
  for (int q = 0; q < g.n; ++q) {
    if (digs[q].dim >= (1ll << 31)) return false;
    g.dim[q] = (int32_t)digs[q].dim;
    g.div[q] = FastDiv((uint32_t)digs[q].dim);
    g.stride[q] = digs[q].stride;
  }
  return true;
}

// merge adjacent digits (outer q, inner q+1) when stride_q == dim_{q+1} * stride_{q+1}
std::vector<Digit> merge_digits(const std::vector<Digit>& in) {
  std::vector<Digit> out;
  for (auto& x : in) {
    if (x.dim == 1) continue;
    if (!out.empty() && out.back().stride == x.dim * x.stride) {
      out.back().dim *= x.dim;
      out.back().stride = x.stride;
    } else {
      out.push_back(x);
    }
  }
  return out;
}

struct Operand {
  int rank;
  std::vector<int64_t> ldim, lstride;  // logical
};

double prod_dims(const Operand& o) {
  double p = 1;
  for (auto x : o.ldim) p *= (double)x;
  return p;
}

int make_operand(int rank, const int64_t* shape, const int32_t* perm, Operand& o) {
  if (rank < 0 || rank > TNB_MAX_RANK) return fail(TNB_EINVAL, "contract: rank out of range");
  std::vector<int64_t> ss(rank, 1);
  for (int a = rank - 2; a >= 0; --a) ss[a] = ss[a + 1] * shape[a + 1];
  std::vector<int> seen(rank, 0);
  o.rank = rank;
  o.ldim.resize(rank);
  o.lstride.resize(rank);
  for (int k = 0; k < rank; ++k) {
    int p = perm[k];
    if (p < 0 || p >= rank || seen[p]) return fail(TNB_EINVAL, "contract: invalid permutation");
    seen[p] = 1;
    if (shape[p] < 1) return fail(TNB_EINVAL, "contract: dimensions must be >= 1");
    o.ldim[k] = shape[p];
    o.lstride[k] = ss[p];
  }
  return TNB_OK;
}

struct Cfg {
  int bm, bn;
};

int sms() { return sm_count(); }

// Persistent stream-K workspace (eager launches): partials, then one flag per CTA.
struct SkWorkspace {
  std::mutex mu;
  void* mem = nullptr;
  size_t flags_off = 0;  // bytes of partials
  int nflags = 0;
  int device = -1;
  cudaEvent_t ev = nullptr;
  cudaStream_t last = nullptr;
  int acquire(size_t partial_bytes, int G, cudaStream_t st) {
    int dev = 0;
    TNB_CUDA_CHECK(cudaGetDevice(&dev));
    if (dev != device || partial_bytes > flags_off || G > nflags) {
      if (mem) {
        TNB_CUDA_CHECK(cudaDeviceSynchronize());
        cudaFree(mem);
        mem = nullptr;
      }
      if (ev && dev != device) {
        cudaEventDestroy(ev);
        ev = nullptr;
      }
      flags_off = std::max(partial_bytes, flags_off);
      nflags = std::max(G, std::max(nflags, 1024));
      TNB_CUDA_CHECK(cudaMalloc(&mem, flags_off + (size_t)nflags * 4));
      TNB_CUDA_CHECK(cudaMemset(static_cast<char*>(mem) + flags_off, 0, (size_t)nflags * 4));
      device = dev;
      last = nullptr;
    }
    if (!ev) TNB_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    if (last && last != st) TNB_CUDA_CHECK(cudaStreamWaitEvent(st, ev, 0));
    return TNB_OK;
  }
  int release(cudaStream_t st) {
    TNB_CUDA_CHECK(cudaEventRecord(ev, st));
    last = st;
    return TNB_OK;
  }
};
SkWorkspace& sk_workspace() {
  static SkWorkspace* w = new SkWorkspace();  // never destroyed (process-lifetime device memory)
  return *w;
}

// WS = 1: warp-specialised kernel (producer warpgroup + DMMA warps); 0: single-role kernel.
template <bool CPLX, int MODE, int BM, int BN, int BK, int WM, int WN, int ST, int MINB, int WS = 0>
struct Tiled {
  static constexpr int ES = CPLX ? 16 : 8;
  static constexpr size_t smem = WS ? TileCoreWS<CPLX, MODE, BM, BN, BK, WM, WN, ST, 0, 0>::kSmem
                                    : TileCore<CPLX, MODE, BM, BN, BK, WM, WN, ST>::kSmem;
  static constexpr int threads = WM * WN * 32 + (WS ? 128 : 0);
  using KernT = void (*)(const typename Elem<CPLX>::T*, const typename Elem<CPLX>::T*, typename Elem<CPLX>::T*,
                         const GemmDesc);
  static KernT kernel() {
    if constexpr (WS) return gemm_ws_kernel<CPLX, MODE, BM, BN, BK, WM, WN, ST>;
    else return gemm_kernel<CPLX, MODE, BM, BN, BK, WM, WN, ST, MINB>;
  }
  // resident CTAs per SM (queried once; one process drives one device)
  static int per_sm() {
    static int cached = -1;
    if (cached < 0) {
      auto kern = kernel();
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
      }
      int n = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
      }
      cached = n;
    }
    return cached;
  }
  // estimated time (arbitrary units: SM-cycles at the DMMA rate) and the split-K factor
  static double plan(const GemmDesc& d, int& split, double tile_penalty) {
    int psm = per_sm();
    if (psm < 1) return 1e300;
    const int slots = sms() * psm;
    const int64_t tiles = (int64_t)((d.M + BM - 1) / BM) * ((d.N + BN - 1) / BN);
    const int kt_total = (d.K + BK - 1) / BK;
    const double step = (double)BM * BN * BK * (CPLX ? (MODE == 1 ? 3 : 4) : 1) / 64.0 * psm * tile_penalty;
    double best = 1e300;
    split = 1;
    for (int s = 1; s <= 128; ++s) {
      if (s > 1 && kt_total / s < 4) break;
      int64_t waves = (tiles * s + slots - 1) / slots;
      double t = (double)waves * ((kt_total + s - 1) / s) * step;
      if (s > 1) t += (double)(s + 1) * d.M * (double)d.N * ES / 6.0e12 * 1.9e9 + 3000.0;  // reduce pass
      if (t < best * 0.98) {
        best = t;
        split = s;
      }
    }
    return best;
  }
  static int run(const void* A, const void* B, void* C, GemmDesc d, int split, cudaStream_t st) {
    using T = typename Elem<CPLX>::T;
    auto kern = kernel();
    if (per_sm() < 1) return fail(TNB_ECUDA, "contract: GEMM kernel does not fit on an SM");
    d.tiles_m = (d.M + BM - 1) / BM;
    d.tiles_n = (d.N + BN - 1) / BN;
    const int kt_total = (d.K + BK - 1) / BK;
    int kts = (kt_total + split - 1) / split;
    d.k_per_split = kts * BK;
    d.splitk = (kt_total + kts - 1) / kts;
    if (d.splitk < 1) d.splitk = 1;
    int64_t grid = (int64_t)d.tiles_m * d.tiles_n * d.splitk;
    if (grid >= (1ll << 31)) return fail(TNB_EUNSUP, "contract: problem too large for the tile grid");
    const double work = 2.0 * d.M * (double)d.N * d.K * (CPLX ? 4 : 1);
    if (d.splitk == 1) {
      {
        KTimer kt(TNB_KF_GEMM, st, work);
        TNB_CUDA_CHECK(launch_pdl(kern, (unsigned)grid, threads, smem, st, static_cast<const T*>(A),
                                  static_cast<const T*>(B), static_cast<T*>(C), d));
      }
      count_launch();
      TNB_CUDA_CHECK(cudaGetLastError());
      return TNB_OK;
    }
    // split-K partials: graph-owned memory under capture, else the process-wide persistent
    // workspace -- no allocation / free nodes between the GEMM and its neighbours, so the
    // programmatic-dependent launches chain (a cudaMallocAsync per call broke the chain)
    size_t n = (size_t)d.M * d.N;
    void* ws = nullptr;
    SkWorkspace* w = nullptr;
    std::unique_lock<std::mutex> lk;
    if (capturing(st)) {
      int rc = capture_device_ws(st, n * d.splitk * ES, &ws);
      if (rc) return rc;
    } else {
      release_deferred_host();
      w = &sk_workspace();
      lk = std::unique_lock<std::mutex>(w->mu);
      int rc = w->acquire(n * d.splitk * ES, 0, st);
      if (rc) return rc;
      ws = w->mem;
    }
    {
      KTimer kt(TNB_KF_GEMM, st, work);
      TNB_CUDA_CHECK(launch_pdl(kern, (unsigned)grid, threads, smem, st, static_cast<const T*>(A),
                                static_cast<const T*>(B), static_cast<T*>(ws), d));
    }
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) {
      int blocks = (int)std::min<size_t>((n + 255) / 256, (size_t)sms() * 8);
      e = launch_pdl(splitk_reduce_kernel<CPLX>, (unsigned)blocks, 256, 0, st, static_cast<const T*>(ws),
                     static_cast<T*>(C), (int64_t)n, d.splitk);
      count_launch();
      if (e == cudaSuccess) e = cudaGetLastError();
    }
    if (w) w->release(st);
    if (e != cudaSuccess) return cuda_fail(e, "contract: split-K GEMM launch");
    return TNB_OK;
  }
};

// Host side of the stream-K kernel: one CTA per SM, workspace for split tiles.
template <bool CPLX, int MODE, int BM, int BN, int BK, int WM, int WN, int ST>
struct StreamK {
  using Core = SKCore<CPLX, MODE, BM, BN, BK, WM, WN, ST>;
  using T = typename Elem<CPLX>::T;
  template <bool AMF, bool BNF>
  static int launch_one(const void* A, const void* B, void* C, const GemmDesc& d, const SKParams& sk, cudaStream_t st) {
    auto kern = gemm_sk_kernel<CPLX, MODE, BM, BN, BK, WM, WN, ST, AMF, BNF>;
    static bool configured = false;
    if (!configured) {
      TNB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Core::kSmem));
      if constexpr (Core::kRegSplit) {
        // the setmaxnreg split assumes the kernel launches with exactly kLaunchRegs per thread
        // (a smaller allocation would leave the math warps' increase waiting forever)
        cudaFuncAttributes fa;
        TNB_CUDA_CHECK(cudaFuncGetAttributes(&fa, kern));
        if (fa.numRegs != Core::kLaunchRegs) return fail(TNB_ECUDA, "gemm: stream-K kernel register count mismatch");
      }
      configured = true;
    }
    {
      KTimer kt(TNB_KF_GEMM, st, 2.0 * d.M * (double)d.N * d.K * (CPLX ? 4 : 1));
      TNB_CUDA_CHECK(launch_cooperative(kern, (unsigned)sk.G, (unsigned)Core::NT, Core::kSmem, st,
                                        static_cast<const T*>(A), static_cast<const T*>(B), static_cast<T*>(C), d, sk));
    }
    count_launch();
    TNB_CUDA_CHECK(cudaGetLastError());
    return TNB_OK;
  }
  static int dispatch(const void* A, const void* B, void* C, const GemmDesc& d, const SKParams& sk, cudaStream_t st) {
    if (d.a_mfast && d.b_nfast) return launch_one<true, true>(A, B, C, d, sk, st);
    if (d.a_mfast) return launch_one<true, false>(A, B, C, d, sk, st);
    if (d.b_nfast) return launch_one<false, true>(A, B, C, d, sk, st);
    return launch_one<false, false>(A, B, C, d, sk, st);
  }
  // Whole BM-row (BN-col) tiles of this operand are one contiguous 16-byte aligned run per
  // k: the innermost free digit is unit-stride and a multiple of the tile, and every other
  // free / contracted stride and the base keep 16-byte alignment.
  static bool bulk_ok(const void* X, const Group& free, const Group& k, int tile, bool fast) {
    constexpr int ES = CPLX ? 16 : 8;
    if (!fast || free.n < 1 || free.stride[free.n - 1] != 1 || free.dim[free.n - 1] % tile) return false;
    if (reinterpret_cast<uintptr_t>(X) % 16) return false;
    for (int q = 0; q < free.n; ++q)
      if ((free.stride[q] * ES) % 16) return false;
    for (int q = 0; q < k.n; ++q)
      if ((k.stride[q] * ES) % 16) return false;
    return true;
  }
  static int run(const void* A, const void* B, void* C, GemmDesc d, cudaStream_t st) {
    d.tiles_m = (d.M + BM - 1) / BM;
    d.tiles_n = (d.N + BN - 1) / BN;
    d.splitk = 1;
    {
      static const bool nobulk = getenv("TNB_NO_BULK") != nullptr;  // A/B switch for measurements
      const bool kfast_path = (d.kaff.ok >= 1 && d.kaff.ok <= 2 && d.kaff.ok >= (BK + 15) / 16) || d.kaff.ok == 3;
      d.bulkA = !nobulk && kfast_path && bulk_ok(A, d.rowA, d.kA, BM, d.a_mfast);
      d.bulkB = !nobulk && kfast_path && bulk_ok(B, d.colB, d.kB, BN, d.b_nfast);
    }
    SKParams sk;
    sk.KT = (d.K + BK - 1) / BK;
    sk.total = (int64_t)d.tiles_m * d.tiles_n * sk.KT;
    if ((int64_t)d.tiles_m * d.tiles_n >= (1ll << 31)) return fail(TNB_EUNSUP, "contract: too many tiles");
    // >= 4 k-tiles per CTA: tiny problems do not pay for many partial hand-offs
    // (r02: 8 / 12 / 16 / 24 k-tiles per CTA measured slower at chi = 128 -- fewer CTAs each
    // walking more k-tiles, while the partial hand-off chain was not the limiter)
    sk.G = (int)std::max<int64_t>(1, std::min<int64_t>(sk.total / 4, sms()));
    const size_t ws_bytes = (size_t)sk.G * Core::ACCN * Core::NMATH * 8;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    TNB_CUDA_CHECK(cudaStreamIsCapturing(st, &cs));
    if (cs != cudaStreamCaptureStatusNone) {
      // graph capture: the graph owns its workspace (a graph replays independently of
      // eager launches on other streams); flags zeroed by a memset node
      void* mem = nullptr;
      int rc = capture_device_ws(st, ws_bytes + (size_t)sk.G * 4 + 64, &mem);
      if (rc) return rc;
      sk.ws = static_cast<double*>(mem);
      sk.flags = reinterpret_cast<int*>(static_cast<char*>(mem) + ws_bytes);
      sk.clear = 1;  // owners reset the flags they consume: clean for the next replay
      cudaError_t e = cudaMemsetAsync(sk.flags, 0, (size_t)sk.G * 4, st);
      return e != cudaSuccess ? cuda_fail(e, "contract: workspace memset") : dispatch(A, B, C, d, sk, st);
    }
    // eager: one persistent workspace per process whose flags the owners reset, so a
    // launch needs no allocation and no memset; launches from different streams are
    // serialised on it through an event
    release_deferred_host();  // memory of destroyed graphs
    SkWorkspace& w = sk_workspace();
    std::lock_guard<std::mutex> lk(w.mu);
    int rc = w.acquire(ws_bytes, sk.G, st);
    if (rc) return rc;
    sk.ws = static_cast<double*>(w.mem);
    sk.flags = reinterpret_cast<int*>(static_cast<char*>(w.mem) + w.flags_off);
    sk.clear = 1;
    rc = dispatch(A, B, C, d, sk, st);
    if (rc) return rc;
    return w.release(st);
  }
};

template <bool CPLX>
size_t skinny_smem(const GemmDesc& d);

template <bool CPLX>
int run_skinny(const void* A, const void* B, void* C, GemmDesc d, cudaStream_t st) {
  using T = typename Elem<CPLX>::T;
  constexpr int ES = CPLX ? 16 : 8;
  size_t smem = skinny_smem<CPLX>(d);
  auto kern = skinny_kernel<CPLX>;
  if (smem > 48 * 1024) TNB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  TNB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
  if (per_sm < 1) per_sm = 1;
  int64_t panels = (d.M + 127) / 128;
  int64_t grid = std::min<int64_t>(panels, (int64_t)sms() * per_sm);
  {
    KTimer kt(TNB_KF_GEMM_SKINNY, st, 2.0 * d.M * (double)d.N * d.K * (CPLX ? 4 : 1));
    kern<<<(unsigned)grid, 256, smem, st>>>(static_cast<const T*>(A), static_cast<const T*>(B), static_cast<T*>(C), d);
  }
  count_launch();
  TNB_CUDA_CHECK(cudaGetLastError());
  return TNB_OK;
}

template <bool CPLX>
size_t skinny_smem(const GemmDesc& d) {
  constexpr int ES = CPLX ? 16 : 8;
  return (size_t)ES * (d.K * d.N + 128 * (d.K + 1) + 128 * d.N) + 8 * (d.K + 128);
}

template <bool CPLX>
int run_dot(const void* A, const void* B, void* C, const GemmDesc& d, cudaStream_t st) {
  using T = typename Elem<CPLX>::T;
  constexpr int ES = CPLX ? 16 : 8;
  const int64_t K = d.K, MN = (int64_t)d.M * d.N;
  const int64_t G = std::max<int64_t>(1, std::min<int64_t>((int64_t)sms() * 4, (K + 2047) / 2048));
  const int64_t kchunk = (K + G - 1) / G;
  void* ws = nullptr;
  TNB_CUDA_CHECK(cudaMallocAsync(&ws, (size_t)(G * MN) * ES, st));
  {
    KTimer kt(TNB_KF_GEMM_SKINNY, st, 2.0 * d.M * (double)d.N * d.K * (CPLX ? 4 : 1));
    dot_kernel<CPLX><<<(unsigned)G, 256, 0, st>>>(static_cast<const T*>(A), static_cast<const T*>(B),
                                                  static_cast<T*>(ws), d, kchunk);
  }
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) {
    splitk_reduce_kernel<CPLX><<<1, 32, 0, st>>>(static_cast<const T*>(ws), static_cast<T*>(C), MN, (int)G);
    count_launch();
    e = cudaGetLastError();
  }
  cudaFreeAsync(ws, st);
  if (e != cudaSuccess) return cuda_fail(e, "contract: dot kernel launch");
  return TNB_OK;
}

template <bool CPLX, int MODE>
int dispatch(const void* A, const void* B, void* C, GemmDesc& d, cudaStream_t st) {
  // the memory-bound kernels write packed rows; a strided output (column panel) takes stream-K
  // (an output index map is written by the stream-K epilogue only)
  const bool packed = d.out_ld == d.N && !d.outmap;
  if (packed && (int64_t)d.M * d.N <= 16) return run_dot<CPLX>(A, B, C, d, st);
  // (N, K <= 10: the MPO step of L.A.W.R with D = 5, d = 2 -- registers sized to it)
  if (packed && d.N <= 10 && d.K <= 10 && d.M >= 4096) return run_narrow<CPLX, 10, 10>(A, B, C, d, st);
  if (packed && d.N <= 16 && d.K <= 16 && d.M >= 4096) return run_narrow<CPLX, 16, 16>(A, B, C, d, st);
  if constexpr (!CPLX)
    if (packed && d.N <= 16 && d.K <= 32 && d.M >= 4096) return run_narrow<CPLX, 16, 32>(A, B, C, d, st);
  if (packed && d.N <= 64 && d.K <= 64 && d.M >= 4096 && skinny_smem<CPLX>(d) <= 160 * 1024)
    return run_skinny<CPLX>(A, B, C, d, st);
  if constexpr (!CPLX) {
    // tile shape with the least padding (N = 64 or M = 64 rows waste half a 128 x 128 tile)
    auto pad = [](int64_t x, int64_t t) { return (x + t - 1) / t * t; };
    const int64_t a128 = pad(d.M, 128) * pad(d.N, 128), aN64 = pad(d.M, 128) * pad(d.N, 64),
                  aM64 = pad(d.M, 64) * pad(d.N, 128);
    // small problems (fewer than ~8 k-iterations of 128 x 128 tiles per SM, e.g. L.A.W.R at
    // chi = 128): 64 x 64 tiles give 4x more stream-K work units, so more SMs take part
    const int64_t it128 = (pad(d.M, 128) / 128) * (pad(d.N, 128) / 128) * ((d.K + 15) / 16);
    if (it128 < (int64_t)sms() * 8) {
      // tiny problems (L.A.W.R at chi = 128: ~2.4 us of DMMA work per launch) are latency
      // bound: a plain one-tile-per-CTA kernel (split-K planned by an occupancy model,
      // fixed-order reduce; launched as programmatic dependents) beats the persistent
      // stream-K kernel's per-stage hand-offs -- C1 graph replay 41.7 -> 28.8 us. The split-K
      // workspace is packed, so strided (column panel) outputs keep stream-K. (Measured and
      // dropped: the reduce inside the GEMM, each of a tile's S co-resident CTAs summing 1/S
      // of its rows after a per-tile arrival counter -- 48 us: the CTAs of a tile wait for
      // the slowest.)
      if (packed) {
        // 64 x 64 tiles, 8 warps of 32 x 16 (C1 graph 28.8 us; 4 warps of 32 x 32: 30.8; 16
        // warps: 30.8; 32 x 32 tiles: 28.8; BK = 32: 39.0; 4 stages: 30.9)
        int split = 1;
        Tiled<false, 0, 64, 64, 16, 2, 4, 3, 2>::plan(d, split, 1.0);
        return Tiled<false, 0, 64, 64, 16, 2, 4, 3, 2>::run(A, B, C, d, split, st);
      }
      return StreamK<false, 0, 64, 64, 16, 4, 4, 4>::run(A, B, C, d, st);
    }
    // a few output tiles over a very long, irregular K (the PEPS closing step: M = 128, N = 64,
    // K = 4.2M, both operands K-gathered): every operand element is read once, in short strided
    // runs -- 32-wide k-tiles double each run per stage
    static const bool no_bk32 = getenv("TNB_NO_BK32") != nullptr;  // dev A/B switch
    if (!no_bk32 && d.kaff.ok == 0 && aN64 <= a128 && pad(d.M, 128) * pad(d.N, 64) <= 4 * 128 * 64 &&
        d.K >= (1 << 16))
      return StreamK<false, 0, 128, 64, 32, 4, 4, 4>::run(A, B, C, d, st);
    if (aN64 < a128 && aN64 <= aM64) return StreamK<false, 0, 128, 64, 16, 4, 4, 4>::run(A, B, C, d, st);
    if (aM64 < a128) return StreamK<false, 0, 64, 128, 16, 4, 4, 4>::run(A, B, C, d, st);
    // (measured: BK = 32 / 3 stages 15% slower; 3, 5 and 6 stages of BK = 16 no faster than 4)
    return StreamK<false, 0, 128, 128, 16, 4, 4, 4>::run(A, B, C, d, st);
  }
  else if constexpr (MODE == 0) return StreamK<true, 0, 64, 128, 8, 4, 4, 4>::run(A, B, C, d, st);
  else return StreamK<true, 1, 64, 64, 8, 4, 4, 4>::run(A, B, C, d, st);
}

// f64 -> c128 widening (mixed-dtype contraction promotes like np.result_type)
__global__ void widen_kernel(const double* __restrict__ x, double2* __restrict__ y, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) y[i] = make_double2(x[i], 0.0);
}

}  // namespace

int contract_dense_device(const void* a, int dta, int ra, const int64_t* sa, const int32_t* pa, const void* b,
                          int dtb, int rb, const int64_t* sb, const int32_t* pb, int nc, const int32_t* aax,
                          const int32_t* bax, void* out, int64_t out_ld, int cplx_mode, cudaStream_t st,
                          const int32_t* out_order = nullptr) {
  if ((dta != TNB_F64 && dta != TNB_C128) || (dtb != TNB_F64 && dtb != TNB_C128))
    return fail(TNB_EUNSUP, "contract: only float64 and complex128 are supported on the GPU path (no CPU fallback)");
  Operand A, B;
  int rc = make_operand(ra, sa, pa, A);
  if (rc) return rc;
  rc = make_operand(rb, sb, pb, B);
  if (rc) return rc;
  if (nc < 0 || nc > ra || nc > rb) return fail(TNB_EINVAL, "contract: bad number of contracted axes");
  std::vector<int> acon(ra, 0), bcon(rb, 0);
  for (int i = 0; i < nc; ++i) {
    int x = aax[i], y = bax[i];
    if (x < 0 || x >= ra || y < 0 || y >= rb || acon[x] || bcon[y])
      return fail(TNB_EINVAL, "contract: bad contracted axis list");
    if (A.ldim[x] != B.ldim[y]) return fail(TNB_EINVAL, "contract: contracted dimensions differ");
    acon[x] = bcon[y] = 1;
  }
  // mixed dtypes: widen the f64 operand into a temporary c128 buffer
  void* tmp = nullptr;
  bool cplx = (dta == TNB_C128) || (dtb == TNB_C128);
  if (cplx && (dta != dtb)) {
    const Operand& R = (dta == TNB_F64) ? A : B;
    int64_t n = 1;
    for (int k = 0; k < R.rank; ++k) n *= R.ldim[k];
    TNB_CUDA_CHECK(cudaMallocAsync(&tmp, (size_t)n * 16, st));
    int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sms() * 8);
    widen_kernel<<<std::max(blocks, 1), 256, 0, st>>>(static_cast<const double*>(dta == TNB_F64 ? a : b),
                                                      static_cast<double2*>(tmp), n);
    count_launch();
    if (dta == TNB_F64) a = tmp;
    else b = tmp;
  }
  std::vector<Digit> rowA, kA, kB, colB;
  for (int k = 0; k < ra; ++k)
    if (!acon[k]) rowA.push_back({A.ldim[k], A.lstride[k]});
  for (int k = 0; k < rb; ++k)
    if (!bcon[k]) colB.push_back({B.ldim[k], B.lstride[k]});
  rowA = merge_digits(rowA);
  colB = merge_digits(colB);
  // contracted digits: merge only when both operands allow it
  std::vector<Digit> ka_raw, kb_raw;
  for (int i = 0; i < nc; ++i) {
    if (A.ldim[aax[i]] == 1) continue;
    ka_raw.push_back({A.ldim[aax[i]], A.lstride[aax[i]]});
    kb_raw.push_back({B.ldim[bax[i]], B.lstride[bax[i]]});
  }
  // An operand whose free rows (cols) are not unit-stride is gathered along K, so its
  // loads coalesce only if consecutive k are adjacent in ITS memory: when exactly one
  // operand is like that, walk K in that operand's memory order (strides descending).
  // (Summation order over K is free; e.g. the PEPS a* step reads B with a 128 KB
  // stride per k in shared-label order -- 8.7x DRAM over-fetch -- and at stride 1 here.)
  const bool a_kfast = !(!rowA.empty() && rowA.back().stride == 1 && rowA.back().dim >= 4);
  const bool b_kfast = !(!colB.empty() && colB.back().stride == 1 && colB.back().dim >= 4);
  const bool k_memorder = a_kfast != b_kfast && ka_raw.size() > 1;
  // Both operands gathered along K: walk K in the LARGER operand's memory order. Its
  // sectors are then consumed whole within a k-tile; the smaller one's partly used
  // sectors are revisited by the next k-tiles while still in L2. (T2.R of L.A.W.R: the
  // 84 MB T2 holds (w2, q) pairs 16 B apart; walking w2 outermost used half of each 32 B
  // sector per pass and read T2 from DRAM ~6x -- 559 MB per launch; in T2's order 136 MB.)
  const bool both_gathered = a_kfast && b_kfast && ka_raw.size() > 1;
  if (k_memorder || both_gathered) {
    std::vector<size_t> idx(ka_raw.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
    bool by_a = a_kfast;
    if (both_gathered) by_a = A.ldim.size() && B.ldim.size() ? prod_dims(A) >= prod_dims(B) : true;
    const std::vector<Digit>& key = by_a ? ka_raw : kb_raw;
    std::stable_sort(idx.begin(), idx.end(), [&](size_t x, size_t y) { return key[x].stride > key[y].stride; });
    std::vector<Digit> ka2, kb2;
    for (size_t i : idx) {
      ka2.push_back(ka_raw[i]);
      kb2.push_back(kb_raw[i]);
    }
    ka_raw.swap(ka2);
    kb_raw.swap(kb2);
  }
  for (size_t i = 0; i < ka_raw.size(); ++i) {
    if (!kA.empty() && kA.back().stride == ka_raw[i].dim * ka_raw[i].stride &&
        kB.back().stride == kb_raw[i].dim * kb_raw[i].stride) {
      kA.back().dim *= ka_raw[i].dim;
      kA.back().stride = ka_raw[i].stride;
      kB.back().dim *= kb_raw[i].dim;
      kB.back().stride = kb_raw[i].stride;
    } else {
      kA.push_back(ka_raw[i]);
      kB.push_back(kb_raw[i]);
    }
  }
  // Contraction order over K is free (only the summation order changes): put the
  // digit that makes every 16-wide k-tile affine innermost, preferring a digit
  // that is contiguous in one of the operands -- unless K follows the memory order of
  // the one k-gathered operand (its smallest-stride digit innermost: coalescing beats
  // the cheaper affine address path; e.g. the PEPS a* step, innermost dn at stride 2
  // interleaved with the free s axis of the same rows).
  const bool keep_order = k_memorder || both_gathered;
  if (kA.size() > 1 && !keep_order) {
    int best = -1;
    int64_t best_score = -1;
    for (size_t i = 0; i < kA.size(); ++i) {
      if (kA[i].dim % 16) continue;
      int64_t score = kA[i].dim + ((kA[i].stride == 1 || kB[i].stride == 1) ? (int64_t(1) << 40) : 0);
      if (score > best_score) {
        best_score = score;
        best = (int)i;
      }
    }
    if (best >= 0 && best != (int)kA.size() - 1) {
      Digit da = kA[best], db = kB[best];
      kA.erase(kA.begin() + best);
      kB.erase(kB.begin() + best);
      kA.push_back(da);
      kB.push_back(db);
    }
  }
  GemmDesc d;
  memset(&d, 0, sizeof(d));
  int64_t M, N, K, K2;
  if (!build_group(rowA, d.rowA, M) || !build_group(colB, d.colB, N) || !build_group(kA, d.kA, K) ||
      !build_group(kB, d.kB, K2)) {
    if (tmp) cudaFreeAsync(tmp, st);
    return fail(TNB_EUNSUP, "contract: index group has too many non-mergeable axes or a dimension >= 2^31");
  }
  if (M >= (1ll << 31) || N >= (1ll << 31) || K >= (1ll << 31) || M * N >= (1ll << 40)) {
    if (tmp) cudaFreeAsync(tmp, st);
    return fail(TNB_EUNSUP, "contract: GEMM extent >= 2^31");
  }
  d.M = (int)M;
  d.N = (int)N;
  d.K = (int)K;
  d.a_elems = (int64_t)prod_dims(A);
  d.b_elems = (int64_t)prod_dims(B);
  d.kaff.ok = 0;
  if (d.kA.n == 0) {
    d.kaff.ok = 0;  // K == 1: the single (partial) k-tile takes the table path
  } else if (d.kA.dim[d.kA.n - 1] % 16 == 0) {
    d.kaff.ok = (d.kA.dim[d.kA.n - 1] % 32 == 0) ? 2 : 1;  // k-tiles of 16 (or 32) stay affine
    d.kaff.ksA = d.kA.stride[d.kA.n - 1];
    d.kaff.ksB = d.kB.stride[d.kB.n - 1];
  } else if (d.kA.n == 2 && d.kA.dim[1] <= 16) {
    // two K digits, the inner one not a multiple of 16: offsets are periodic in k
    d.kaff.ok = 3;
    d.kaff.D0 = d.kA.dim[1];
    d.kaff.div0 = FastDiv((uint32_t)d.kA.dim[1]);
    d.kaff.s1A = d.kA.stride[0];
    d.kaff.s1B = d.kB.stride[0];
    d.kaff.s0A = d.kA.stride[1];
    d.kaff.s0B = d.kB.stride[1];
  }
  if (out_ld != 0 && (out_ld < N || out_ld >= (1ll << 31))) {
    if (tmp) cudaFreeAsync(tmp, st);
    return fail(TNB_EINVAL, "contract: out_ld must be 0 or >= the output column count");
  }
  d.out_ld = (int)(out_ld ? out_ld : N);
  if (out_order) {
    // physical order of the output axes (a's free axes, then b's, logically): element (m, n)
    // lands at rowC(m) + colC(n), digits in the same enumeration order as rowA / colB
    if (out_ld) {
      if (tmp) cudaFreeAsync(tmp, st);
      return fail(TNB_EINVAL, "contract: an output order needs a packed output");
    }
    std::vector<int64_t> odim;
    int na = 0;
    for (int k = 0; k < ra; ++k)
      if (!acon[k]) odim.push_back(A.ldim[k]), ++na;
    for (int k = 0; k < rb; ++k)
      if (!bcon[k]) odim.push_back(B.ldim[k]);
    const int ro = (int)odim.size();
    std::vector<int64_t> pstride(ro, 0);
    std::vector<int> seen(ro, 0);
    bool ident = true;
    int64_t acc_stride = 1;
    for (int q = ro - 1; q >= 0; --q) {
      const int x = out_order[q];
      if (x < 0 || x >= ro || seen[x]) {
        if (tmp) cudaFreeAsync(tmp, st);
        return fail(TNB_EINVAL, "contract: out_order is not a permutation of the output axes");
      }
      seen[x] = 1;
      ident = ident && x == q;
      pstride[x] = acc_stride;
      acc_stride *= odim[x];
    }
    if (!ident) {
      std::vector<Digit> rc, cc;
      for (int q = 0; q < ro; ++q) (q < na ? rc : cc).push_back({odim[q], pstride[q]});
      int64_t Mc, Nc;
      if (!build_group(merge_digits(rc), d.rowC, Mc) || !build_group(merge_digits(cc), d.colC, Nc) || Mc != M ||
          Nc != N) {
        if (tmp) cudaFreeAsync(tmp, st);
        return fail(TNB_EUNSUP, "contract: output order has too many non-mergeable axes");
      }
      d.outmap = 1;
    }
  }
  d.a_mfast = 1;
  if (!(d.rowA.n > 0 && d.rowA.stride[d.rowA.n - 1] == 1 && d.rowA.dim[d.rowA.n - 1] >= 4) && d.kA.n > 0 &&
      d.kA.stride[d.kA.n - 1] == 1)
    d.a_mfast = 0;
  d.b_nfast = 1;
  if (!(d.colB.n > 0 && d.colB.stride[d.colB.n - 1] == 1 && d.colB.dim[d.colB.n - 1] >= 4) && d.kB.n > 0 &&
      d.kB.stride[d.kB.n - 1] == 1)
    d.b_nfast = 0;
  static const bool dbg = getenv("TNB_DEBUG_GEMM") != nullptr;  // dev: the GEMM view of a contraction
  if (dbg) {
    fprintf(stderr, "[tnb gemm] M=%lld N=%lld K=%lld kaff=%d a_mfast=%d b_nfast=%d\n", (long long)M, (long long)N,
            (long long)K, d.kaff.ok, d.a_mfast, d.b_nfast);
    auto pr = [](const char* nm, const Group& g) {
      fprintf(stderr, "  %s:", nm);
      for (int q = 0; q < g.n; ++q) fprintf(stderr, " (%d,%lld)", g.dim[q], (long long)g.stride[q]);
      fprintf(stderr, "\n");
    };
    pr("rowA", d.rowA), pr("kA", d.kA), pr("kB", d.kB), pr("colB", d.colB);
  }
  if (!cplx) rc = dispatch<false, 0>(a, b, out, d, st);
  else if (cplx_mode == TNB_CPLX_3M) rc = dispatch<true, 1>(a, b, out, d, st);
  else rc = dispatch<true, 0>(a, b, out, d, st);
  if (tmp) cudaFreeAsync(tmp, st);
  return rc;
}

}  // namespace tnb

extern "C" int tnb_contract_dense(const void* a, int dtype_a, int rank_a, const int64_t* shape_a,
                                  const int32_t* perm_a, const void* b, int dtype_b, int rank_b,
                                  const int64_t* shape_b, const int32_t* perm_b, int nc, const int32_t* a_axes,
                                  const int32_t* b_axes, void* out, int cplx_mode, void* stream) {
  int rc = tnb::require_device();
  if (rc) return rc;
  if ((rank_a > 0 && (!shape_a || !perm_a)) || (rank_b > 0 && (!shape_b || !perm_b)) ||
      (nc > 0 && (!a_axes || !b_axes)) || !a || !b || !out)
    return tnb::fail(TNB_EINVAL, "contract: NULL argument");
  return tnb::contract_dense_device(a, dtype_a, rank_a, shape_a, perm_a, b, dtype_b, rank_b, shape_b, perm_b, nc,
                                    a_axes, b_axes, out, 0, cplx_mode, (cudaStream_t)stream);
}

extern "C" int tnb_contract_dense_out(const void* a, int dtype_a, int rank_a, const int64_t* shape_a,
                                      const int32_t* perm_a, const void* b, int dtype_b, int rank_b,
                                      const int64_t* shape_b, const int32_t* perm_b, int nc, const int32_t* a_axes,
                                      const int32_t* b_axes, void* out, const int32_t* out_order, int cplx_mode,
                                      void* stream) {
  int rc = tnb::require_device();
  if (rc) return rc;
  if ((rank_a > 0 && (!shape_a || !perm_a)) || (rank_b > 0 && (!shape_b || !perm_b)) ||
      (nc > 0 && (!a_axes || !b_axes)) || !a || !b || !out)
    return tnb::fail(TNB_EINVAL, "contract: NULL argument");
  return tnb::contract_dense_device(a, dtype_a, rank_a, shape_a, perm_a, b, dtype_b, rank_b, shape_b, perm_b, nc,
                                    a_axes, b_axes, out, 0, cplx_mode, (cudaStream_t)stream, out_order);
}

extern "C" int tnb_contract_dense_ld(const void* a, int dtype_a, int rank_a, const int64_t* shape_a,
                                     const int32_t* perm_a, const void* b, int dtype_b, int rank_b,
                                     const int64_t* shape_b, const int32_t* perm_b, int nc, const int32_t* a_axes,
                                     const int32_t* b_axes, void* out, int64_t out_ld, int cplx_mode, void* stream) {
  int rc = tnb::require_device();
  if (rc) return rc;
  if ((rank_a > 0 && (!shape_a || !perm_a)) || (rank_b > 0 && (!shape_b || !perm_b)) ||
      (nc > 0 && (!a_axes || !b_axes)) || !a || !b || !out)
    return tnb::fail(TNB_EINVAL, "contract: NULL argument");
  return tnb::contract_dense_device(a, dtype_a, rank_a, shape_a, perm_a, b, dtype_b, rank_b, shape_b, perm_b, nc,
                                    a_axes, b_axes, out, out_ld, cplx_mode, (cudaStream_t)stream);
}

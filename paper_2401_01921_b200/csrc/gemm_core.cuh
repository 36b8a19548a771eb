// FP64 DMMA tile-GEMM core shared by the dense contraction (gemm.cu) and the
// block-sparse grouped contraction (blocksparse.cu).
//
// A CTA owns a BM x BN output tile. Operands are gathered straight from the
// tensors' storage through "index groups" (lists of (dim, stride) digits): every
// element address is base + row_off[m] + k_off[k]. Row/col offsets are built
// once per (tile, operand pair); K offsets once per k-tile into a ring of
// STAGES+1 slots, one stage ahead of the cp.async that uses them.
//
// Math is mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4): the FP64 tensor-core path of
// sm_100a (tcgen05.mma has no f64 kind). Complex: MODE 0 = 4M (four real
// products per fragment pair), MODE 1 = 3M (Gauss).
#pragma once
#include "common.cuh"

namespace tnb {

constexpr int kMaxDig = 8;

// One index group: idx -> sum_d digit_d * stride_d, digits outer->inner.
struct Group {
  int n;
  int32_t dim[kMaxDig];
  FastDiv div[kMaxDig];
  int64_t stride[kMaxDig];
};

__device__ __forceinline__ int64_t group_offset(const Group& g, uint32_t idx) {
  int64_t off = 0;
#pragma unroll
  for (int q = kMaxDig - 1; q >= 0; --q) {
    if (q < g.n) {
      uint32_t quo = g.div[q].div(idx);
      uint32_t dig = idx - quo * (uint32_t)g.dim[q];
      idx = quo;
      off += (int64_t)dig * g.stride[q];
    }
  }
  return off;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc, bool valid) {
  int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(n));
}
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, bool valid) {
  int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ double dneg(double x) {
  return __longlong_as_double(__double_as_longlong(x) ^ (long long)0x8000000000000000ull);
}

template <bool CPLX>
struct Elem;
template <>
struct Elem<false> { using T = double; };
template <>
struct Elem<true> { using T = double2; };

template <bool CPLX, int MODE, int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES>
struct TileCore {
  using T = typename Elem<CPLX>::T;
  static constexpr int ES = CPLX ? 16 : 8;
  static constexpr int NT = WARPS_M * WARPS_N * 32;
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  static constexpr int MF = WTM / 8, NF = WTN / 8;
  // padded leading dims: 4 (mod 16) doubles / 2 (mod 8) complex -> conflict-free fragment loads
  static constexpr int LDA = BM + (CPLX ? 2 : 4);
  static constexpr int LDB = BN + (CPLX ? 2 : 4);
  static constexpr int KSLOTS = STAGES + 1;
  static constexpr int NACC = CPLX ? (MODE == 1 ? 3 : 2) : 1;
  static constexpr size_t kSmem =
      (size_t)STAGES * BK * (LDA + LDB) * ES + (size_t)(BM + BN) * 8 + (size_t)2 * KSLOTS * BK * 8;
  static_assert(BK % 4 == 0, "BK must be a multiple of 4");
  static_assert((BM * BK) % NT == 0 && (BN * BK) % NT == 0, "tile/threads mismatch");

  using Acc = double[NACC][MF][NF][2];

  // Warp -> (row group, column group) of the CTA tile. With a 4 x 4 warp grid the assignment
  // is a Latin square over the four SM sub-partitions (warp w issues on SMSP w % 4): every
  // SMSP holds one warp of each row group and one of each column group, so a tile whose
  // valid region covers only some row or column groups (block-sparse edge tiles, whose
  // all-padding fragments skip their DMMAs) still spreads its DMMAs over all four pipes.
  __device__ __forceinline__ static void warp_mn(int warp, int& wm, int& wn) {
    if constexpr (WARPS_M == 4 && WARPS_N == 4) {
      wn = warp >> 2;
      wm = (warp + wn) & 3;
    } else if constexpr (WARPS_M == 2 && WARPS_N == 4) {
      // SMSP s (warps s, s + 4) holds column groups s and s + 2: an edge tile with one or two
      // live column groups still spreads its DMMAs over two or four tensor pipes
      wm = warp >> 2;
      wn = (warp + 2 * wm) & 3;
    } else {
      wm = warp / WARPS_N;
      wn = warp % WARPS_N;
    }
  }

  __device__ static void zero(Acc& acc) {
#pragma unroll
    for (int q = 0; q < NACC; ++q)
#pragma unroll
      for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) acc[q][i][j][0] = acc[q][i][j][1] = 0.0;
  }

  // acc += A[m0:m0+BM, kbeg:kend] . B[kbeg:kend, n0:n0+BN]; rows >= M / cols >= N read as 0.
  // Must be called by all NT threads; leaves shared memory reusable (ends with a barrier).
  __device__ static void mainloop(unsigned char* smem, const T* __restrict__ A, const T* __restrict__ B,
                                  const Group& rowA, const Group& kA, const Group& kB, const Group& colB, int m0,
                                  int n0, int M, int N, int kbeg, int kend, bool a_mfast, bool b_nfast, Acc& acc) {
    T* As = reinterpret_cast<T*>(smem);
    T* Bs = As + STAGES * BK * LDA;
    int64_t* rowOffA = reinterpret_cast<int64_t*>(Bs + STAGES * BK * LDB);
    int64_t* colOffB = rowOffA + BM;
    int64_t* kOffA = colOffB + BN;         // [KSLOTS][BK]
    int64_t* kOffB = kOffA + KSLOTS * BK;  // [KSLOTS][BK]
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    int wm, wn;
    warp_mn(warp, wm, wn);
    const int KT = (kend - kbeg + BK - 1) / BK;

    for (int i = tid; i < BM; i += NT) rowOffA[i] = (m0 + i < M) ? group_offset(rowA, m0 + i) : -1;
    for (int i = tid; i < BN; i += NT) colOffB[i] = (n0 + i < N) ? group_offset(colB, n0 + i) : -1;
    auto fill_koff = [&](int kt) {
      const int slot = kt % KSLOTS;
      for (int i = tid; i < 2 * BK; i += NT) {
        const int kk = i % BK;
        const int k = kbeg + kt * BK + kk;
        const bool v = k < kend;
        if (i < BK) kOffA[slot * BK + kk] = v ? group_offset(kA, k) : -1;
        else kOffB[slot * BK + kk] = v ? group_offset(kB, k) : -1;
      }
    };
    for (int kt = 0; kt < STAGES && kt < KT; ++kt) fill_koff(kt);
    __syncthreads();
    // programmatic dependent launch: everything above reads only kernel parameters, so it
    // overlaps the previous kernel's tail; the operands may be that kernel's output
    pdl_wait();

    auto issue = [&](int kt) {
      const int stage = kt % STAGES;
      const int slot = kt % KSLOTS;
      T* as = As + stage * BK * LDA;
      T* bs = Bs + stage * BK * LDB;
      const int64_t* ka = kOffA + slot * BK;
      const int64_t* kb = kOffB + slot * BK;
#pragma unroll
      for (int i = 0; i < (BM * BK) / NT; ++i) {
        const int e = tid + i * NT;
        int m, kk;
        if (a_mfast) {
          m = e % BM;
          kk = e / BM;
        } else {  // 4 consecutive k x 8 rows per warp instruction
          kk = (e & 3) + 4 * (e / (4 * BM));
          m = (e >> 2) % BM;
        }
        const int64_t ro = rowOffA[m], ko = ka[kk];
        const bool v = (ro >= 0) && (ko >= 0);
        const T* src = v ? (A + ro + ko) : A;
        if constexpr (CPLX) cp_async16(as + kk * LDA + m, src, v);
        else cp_async8(as + kk * LDA + m, src, v);
      }
#pragma unroll
      for (int i = 0; i < (BN * BK) / NT; ++i) {
        const int e = tid + i * NT;
        int n, kk;
        if (b_nfast) {
          n = e % BN;
          kk = e / BN;
        } else {
          kk = (e & 3) + 4 * (e / (4 * BN));
          n = (e >> 2) % BN;
        }
        const int64_t co = colOffB[n], ko = kb[kk];
        const bool v = (co >= 0) && (ko >= 0);
        const T* src = v ? (B + co + ko) : B;
        if constexpr (CPLX) cp_async16(bs + kk * LDB + n, src, v);
        else cp_async8(bs + kk * LDB + n, src, v);
      }
    };

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < KT) issue(s);
      cp_async_commit();
    }
    const int arow = wm * WTM + (lane >> 2);
    const int bcol = wn * WTN + (lane >> 2);
    const int kq = lane & 3;

    for (int kt = 0; kt < KT; ++kt) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      if (kt + STAGES - 1 < KT) issue(kt + STAGES - 1);
      cp_async_commit();
      if (kt + STAGES < KT) fill_koff(kt + STAGES);

      const T* as = As + (kt % STAGES) * BK * LDA;
      const T* bs = Bs + (kt % STAGES) * BK * LDB;
#pragma unroll
      for (int k4 = 0; k4 < BK / 4; ++k4) {
        const int kr = k4 * 4 + kq;
        if constexpr (!CPLX) {
          double af[MF], bf[NF];
#pragma unroll
          for (int i = 0; i < MF; ++i) af[i] = as[kr * LDA + arow + i * 8];
#pragma unroll
          for (int j = 0; j < NF; ++j) bf[j] = bs[kr * LDB + bcol + j * 8];
#pragma unroll
          for (int i = 0; i < MF; ++i)
#pragma unroll
            for (int j = 0; j < NF; ++j) dmma(acc[0][i][j][0], acc[0][i][j][1], af[i], bf[j]);
        } else {
          double2 af[MF], bf[NF];
#pragma unroll
          for (int i = 0; i < MF; ++i) af[i] = as[kr * LDA + arow + i * 8];
#pragma unroll
          for (int j = 0; j < NF; ++j) bf[j] = bs[kr * LDB + bcol + j * 8];
          if constexpr (MODE == 0) {  // 4M: re += Ar Br - Ai Bi ; im += Ar Bi + Ai Br
#pragma unroll
            for (int i = 0; i < MF; ++i) {
              const double ain = dneg(af[i].y);
#pragma unroll
              for (int j = 0; j < NF; ++j) {
                dmma(acc[0][i][j][0], acc[0][i][j][1], af[i].x, bf[j].x);
                dmma(acc[0][i][j][0], acc[0][i][j][1], ain, bf[j].y);
                dmma(acc[1][i][j][0], acc[1][i][j][1], af[i].x, bf[j].y);
                dmma(acc[1][i][j][0], acc[1][i][j][1], af[i].y, bf[j].x);
              }
            }
          } else {  // 3M: T0 = Ar Br, T1 = Ai Bi, T2 = (Ar+Ai)(Br+Bi)
            double bsum[NF];
#pragma unroll
            for (int j = 0; j < NF; ++j) bsum[j] = bf[j].x + bf[j].y;
#pragma unroll
            for (int i = 0; i < MF; ++i) {
              const double asum = af[i].x + af[i].y;
#pragma unroll
              for (int j = 0; j < NF; ++j) {
                dmma(acc[0][i][j][0], acc[0][i][j][1], af[i].x, bf[j].x);
                dmma(acc[1][i][j][0], acc[1][i][j][1], af[i].y, bf[j].y);
                dmma(acc[2][i][j][0], acc[2][i][j][1], asum, bsum[j]);
              }
            }
          }
        }
      }
    }
    cp_async_wait<0>();
    __syncthreads();
  }

  // C[m, n] (row-major, leading dim ld) = acc for the tile at (m0, n0), clipped to M x N.
  __device__ static void store(T* __restrict__ C, int64_t ld, int m0, int n0, int M, int N, const Acc& acc) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int wm, wn;
    warp_mn(warp, wm, wn);
    const int kq = lane & 3;
#pragma unroll
    for (int i = 0; i < MF; ++i) {
      const int m = m0 + wm * WTM + i * 8 + (lane >> 2);
      if (m >= M) continue;
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const int n = n0 + wn * WTN + j * 8 + 2 * kq;
        T* dst = C + (int64_t)m * ld + n;
        if constexpr (!CPLX) {
          const double v0 = acc[0][i][j][0], v1 = acc[0][i][j][1];
          if (n + 1 < N && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
            *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
          } else {
            if (n < N) dst[0] = v0;
            if (n + 1 < N) dst[1] = v1;
          }
        } else {
          double re0, re1, im0, im1;
          if constexpr (MODE == 0) {
            re0 = acc[0][i][j][0];
            re1 = acc[0][i][j][1];
            im0 = acc[1][i][j][0];
            im1 = acc[1][i][j][1];
          } else {
            re0 = acc[0][i][j][0] - acc[1][i][j][0];
            re1 = acc[0][i][j][1] - acc[1][i][j][1];
            im0 = acc[2][i][j][0] - acc[0][i][j][0] - acc[1][i][j][0];
            im1 = acc[2][i][j][1] - acc[0][i][j][1] - acc[1][i][j][1];
          }
          if (n < N) dst[0] = make_double2(re0, im0);
          if (n + 1 < N) dst[1] = make_double2(re1, im1);
        }
      }
    }
  }
};


// ============================================================================
// Warp-specialised variant (the dense-contraction hot loop).
//
// Why: DMMA.8x8x4 issues at most one per 16 cycles per SMSP and ptxas pads every
// DMMA with a 16-cycle stall, so a math warp's timeline is DMMA-bound by itself;
// any gather / barrier work on the math warps leaves the pipe idle (66% pipe
// activity measured for the single-role kernel). Here a producer warpgroup (4
// warps, one per SMSP) owns all operand gathers (cp.async into a STAGES ring,
// completion signalled on per-stage "full" mbarriers with
// cp.async.mbarrier.arrive.noinc) and the math warps only do LDS + DMMA, handing
// stages back through "empty" mbarriers. No CTA-wide barrier in the main loop.
// setmaxnreg moves registers from the producers to the math warps.
namespace detail {
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
// A waiting warp may be suspended (up to this hint) instead of re-polling: spinning
// consumers would otherwise take issue slots from the producer warps on their SMSP.
#ifndef TNB_MBAR_WAIT
#define TNB_MBAR_WAIT 0
#endif
constexpr uint32_t kSuspendHintNs = 0x989680;
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
#if TNB_MBAR_WAIT == 0
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity), "r"(kSuspendHintNs));
#elif TNB_MBAR_WAIT == 1
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity));
#else
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity));
#endif
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)));
}
// Bulk (TMA engine) copy of `bytes` contiguous bytes global -> shared, completing as
// transaction bytes on `bar`; expect_tx raises the barrier's pending byte count first.
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)));
}
template <int N>
__device__ __forceinline__ void reg_alloc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void reg_dealloc() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N));
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n)); }
}  // namespace detail

// K offsets within one k-tile are affine (k_off(k0 + kk) = k_off(k0) + kk * ks) when
// the innermost contracted digit has extent divisible by BK (the host orders the K
// digits so that this holds whenever possible).
struct KAffine {
  int ok;              // 1/2: affine k-tiles (16 / 32 wide) for both operands; 3: periodic (below)
  int64_t ksA, ksB;    // strides of the innermost K digit
  // ok == 3: K = (outer digit) x (inner digit of D0 < 16 or not a multiple of 16):
  // offset(k) = (k / D0) * s1 + (k % D0) * s0 -- k-tiles need no offset table
  int D0;
  FastDiv div0;
  int64_t s1A, s1B, s0A, s0B;
};

template <bool CPLX, int MODE, int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, int REG_MATH,
          int REG_PROD>
struct TileCoreWS {
  using T = typename Elem<CPLX>::T;
  static constexpr int ES = CPLX ? 16 : 8;
  static constexpr int NMATH = WARPS_M * WARPS_N * 32;  // math threads
  static constexpr int NPROD = 128;                     // producer warpgroup
  static constexpr int NT = NMATH + NPROD;
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  static constexpr int MF = WTM / 8, NF = WTN / 8;
  static constexpr int LDA = BM + (CPLX ? 2 : 4);
  static constexpr int LDB = BN + (CPLX ? 2 : 4);
  static constexpr int NACC = CPLX ? (MODE == 1 ? 3 : 2) : 1;
  static constexpr size_t kOffTables = (size_t)(BM + BN) * 8 + (size_t)2 * 2 * BK * 8;
  static constexpr size_t kSmem = (size_t)STAGES * BK * (LDA + LDB) * ES + kOffTables + (size_t)2 * STAGES * 8;
  static_assert(NMATH % 128 == 0, "math warps must form whole warpgroups");
  static_assert((BM * BK) % NPROD == 0 && (BN * BK) % NPROD == 0, "tile/producer mismatch");
  using Acc = double[NACC][MF][NF][2];

  // Warp -> (row group, column group) of the CTA tile. With a 4 x 4 warp grid the assignment
  // is a Latin square over the four SM sub-partitions (warp w issues on SMSP w % 4): every
  // SMSP holds one warp of each row group and one of each column group, so a tile whose
  // valid region covers only some row or column groups (block-sparse edge tiles, whose
  // all-padding fragments skip their DMMAs) still spreads its DMMAs over all four pipes.
  __device__ __forceinline__ static void warp_mn(int warp, int& wm, int& wn) {
    if constexpr (WARPS_M == 4 && WARPS_N == 4) {
      wn = warp >> 2;
      wm = (warp + wn) & 3;
    } else if constexpr (WARPS_M == 2 && WARPS_N == 4) {
      // SMSP s (warps s, s + 4) holds column groups s and s + 2: an edge tile with one or two
      // live column groups still spreads its DMMAs over two or four tensor pipes
      wm = warp >> 2;
      wn = (warp + 2 * wm) & 3;
    } else {
      wm = warp / WARPS_N;
      wn = warp % WARPS_N;
    }
  }

  __device__ static void zero(Acc& acc) { TileCore<CPLX, MODE, BM, BN, BK, WARPS_M, WARPS_N, STAGES>::zero(acc); }

  // Returns true in math threads (acc valid); producers return false after the last stage.
  // AMF / BNF: operand A is M-fast (else K-fast), operand B is N-fast (else K-fast).
  template <bool AMF, bool BNF>
  __device__ static bool run(unsigned char* smem, const T* __restrict__ A, const T* __restrict__ B,
                             const Group& rowA, const Group& kA, const Group& kB, const Group& colB, int m0, int n0,
                             int M, int N, int kbeg, int kend, const KAffine& kaff, Acc& acc) {
    constexpr bool a_mfast = AMF, b_nfast = BNF;
    T* As = reinterpret_cast<T*>(smem);
    T* Bs = As + STAGES * BK * LDA;
    int64_t* rowOffA = reinterpret_cast<int64_t*>(Bs + STAGES * BK * LDB);
    int64_t* colOffB = rowOffA + BM;
    int64_t* kOffA = colOffB + BN;        // [2][BK]
    int64_t* kOffB = kOffA + 2 * BK;      // [2][BK]
    uint64_t* full = reinterpret_cast<uint64_t*>(kOffB + 2 * BK);
    uint64_t* empty = full + STAGES;
    const int tid = threadIdx.x;
    const int KT = (kend - kbeg + BK - 1) / BK;
    if (tid == 0) {
      for (int s = 0; s < STAGES; ++s) {
        detail::mbar_init(&full[s], NPROD);
        detail::mbar_init(&empty[s], NMATH / 32);
      }
    }
    __syncthreads();

    if (tid >= NMATH) {
      // ------------------------------------------------------------ producer
      if constexpr (REG_PROD > 0) detail::reg_dealloc<REG_PROD>();
      const int p = tid - NMATH;
      for (int i = p; i < BM; i += NPROD) rowOffA[i] = (m0 + i < M) ? group_offset(rowA, m0 + i) : -1;
      for (int i = p; i < BN; i += NPROD) colOffB[i] = (n0 + i < N) ? group_offset(colB, n0 + i) : -1;
      detail::named_sync(1, NPROD);
      constexpr int EA = (BM * BK) / NPROD, EB = (BN * BK) / NPROD;
      // element e of this thread -> (row, kk) of the tile (same mapping for every k-tile)
      auto mapA = [&](int i, int& m, int& kk) {
        const int e = p + i * NPROD;
        if (a_mfast) { m = e % BM; kk = e / BM; }
        else { kk = (e & 3) + 4 * (e / (4 * BM)); m = (e >> 2) % BM; }
      };
      auto mapB = [&](int i, int& n, int& kk) {
        const int e = p + i * NPROD;
        if (b_nfast) { n = e % BN; kk = e / BN; }
        else { kk = (e & 3) + 4 * (e / (4 * BN)); n = (e >> 2) % BN; }
      };
      // affine fast path: per-element offsets rowOff + kk*ks live in registers for the
      // whole tile; per k-tile one group_offset per operand and one 64-bit add per element
      const bool all_affine = (kaff.ok == 1 || kaff.ok == 2) && ((kend - kbeg) % BK == 0);
      if (all_affine) {
        // distinct rows / cols touched by this thread (compile-time structure of the
        // mapping): M-fast -> one row, K-fast -> 4 rows (one per i % 4)
        constexpr int RA = AMF ? 1 : 4, RB = BNF ? 1 : 4;
        int64_t rA[RA], rB[RB];
#pragma unroll
        for (int j = 0; j < RA; ++j) {
          int m, kk;
          mapA(j, m, kk);
          rA[j] = rowOffA[m];
        }
#pragma unroll
        for (int j = 0; j < RB; ++j) {
          int n, kk;
          mapB(j, n, kk);
          rB[j] = colOffB[n];
        }
        const uint32_t sAbase = smem_u32(As), sBbase = smem_u32(Bs);
        constexpr uint32_t stA = BK * LDA * ES, stB = BK * LDB * ES;
        for (int kt = 0; kt < KT; ++kt) {
          const int s = kt % STAGES;
          const int k0 = kbeg + kt * BK;
          const T* pa = A + group_offset(kA, k0);
          const T* pb = B + group_offset(kB, k0);
          if (kt >= STAGES) detail::mbar_wait(&empty[s], ((kt / STAGES) & 1) ^ 1);
#pragma unroll
          for (int i = 0; i < EA; ++i) {
            int m, kk;
            mapA(i, m, kk);
            const int64_t ro = rA[i % RA];
            const bool v = ro >= 0;
            const T* src = v ? pa + ro + (int64_t)kk * kaff.ksA : A;
            const uint32_t dst = sAbase + s * stA + (uint32_t)(kk * LDA + m) * ES;
            if constexpr (CPLX)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 16 : 0));
            else
              asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 8 : 0));
          }
#pragma unroll
          for (int i = 0; i < EB; ++i) {
            int n, kk;
            mapB(i, n, kk);
            const int64_t co = rB[i % RB];
            const bool v = co >= 0;
            const T* src = v ? pb + co + (int64_t)kk * kaff.ksB : B;
            const uint32_t dst = sBbase + s * stB + (uint32_t)(kk * LDB + n) * ES;
            if constexpr (CPLX)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 16 : 0));
            else
              asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 8 : 0));
          }
          detail::cp_async_mbar_arrive_noinc(&full[s]);
        }
        cp_async_wait<0>();
        return false;
      }
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        const int k0 = kbeg + kt * BK;
        const int64_t* ka = kOffA + (kt & 1) * BK;
        const int64_t* kb = kOffB + (kt & 1) * BK;
        // per-k offsets for this tile in a producer-private double buffer
        for (int i = p; i < 2 * BK; i += NPROD) {
          const int kk = i % BK, k = k0 + kk;
          const bool v = k < kend;
          if (i < BK) kOffA[(kt & 1) * BK + kk] = v ? group_offset(kA, k) : -1;
          else kOffB[(kt & 1) * BK + kk] = v ? group_offset(kB, k) : -1;
        }
        detail::named_sync(1, NPROD);
        if (kt >= STAGES) detail::mbar_wait(&empty[s], ((kt / STAGES) & 1) ^ 1);
        T* as = As + s * BK * LDA;
        T* bs = Bs + s * BK * LDB;
#pragma unroll
        for (int i = 0; i < EA; ++i) {
          int m, kk;
          mapA(i, m, kk);
          const int64_t ro = rowOffA[m];
          const int64_t ko = ka[kk];
          const bool v = (ro >= 0) && (ko >= 0);
          const T* src = v ? (A + ro + ko) : A;
          if constexpr (CPLX) cp_async16(as + kk * LDA + m, src, v);
          else cp_async8(as + kk * LDA + m, src, v);
        }
#pragma unroll
        for (int i = 0; i < EB; ++i) {
          int n, kk;
          mapB(i, n, kk);
          const int64_t co = colOffB[n];
          const int64_t ko = kb[kk];
          const bool v = (co >= 0) && (ko >= 0);
          const T* src = v ? (B + co + ko) : B;
          if constexpr (CPLX) cp_async16(bs + kk * LDB + n, src, v);
          else cp_async8(bs + kk * LDB + n, src, v);
        }
        detail::cp_async_mbar_arrive_noinc(&full[s]);
      }
      cp_async_wait<0>();
      return false;
    }

    // -------------------------------------------------------------- math warps
    if constexpr (REG_MATH > 0) detail::reg_alloc<REG_MATH>();
    const int lane = tid & 31, warp = tid >> 5;
    int wm, wn;
    warp_mn(warp, wm, wn);
    const int arow = wm * WTM + (lane >> 2);
    const int bcol = wn * WTN + (lane >> 2);
    const int kq = lane & 3;
    for (int kt = 0; kt < KT; ++kt) {
      const int s = kt % STAGES;
      detail::mbar_wait(&full[s], (kt / STAGES) & 1);
      const T* as = As + s * BK * LDA;
      const T* bs = Bs + s * BK * LDB;
#pragma unroll
      for (int k4 = 0; k4 < BK / 4; ++k4) {
        const int kr = k4 * 4 + kq;
        if constexpr (!CPLX) {
          double af[MF], bf[NF];
#pragma unroll
          for (int i = 0; i < MF; ++i) af[i] = as[kr * LDA + arow + i * 8];
#pragma unroll
          for (int j = 0; j < NF; ++j) bf[j] = bs[kr * LDB + bcol + j * 8];
#pragma unroll
          for (int i = 0; i < MF; ++i)
#pragma unroll
            for (int j = 0; j < NF; ++j) dmma(acc[0][i][j][0], acc[0][i][j][1], af[i], bf[j]);
        } else {
          double2 af[MF], bf[NF];
#pragma unroll
          for (int i = 0; i < MF; ++i) af[i] = as[kr * LDA + arow + i * 8];
#pragma unroll
          for (int j = 0; j < NF; ++j) bf[j] = bs[kr * LDB + bcol + j * 8];
          if constexpr (MODE == 0) {
#pragma unroll
            for (int i = 0; i < MF; ++i) {
              const double ain = dneg(af[i].y);
#pragma unroll
              for (int j = 0; j < NF; ++j) {
                dmma(acc[0][i][j][0], acc[0][i][j][1], af[i].x, bf[j].x);
                dmma(acc[0][i][j][0], acc[0][i][j][1], ain, bf[j].y);
                dmma(acc[1][i][j][0], acc[1][i][j][1], af[i].x, bf[j].y);
                dmma(acc[1][i][j][0], acc[1][i][j][1], af[i].y, bf[j].x);
              }
            }
          } else {
            double bsum[NF];
#pragma unroll
            for (int j = 0; j < NF; ++j) bsum[j] = bf[j].x + bf[j].y;
#pragma unroll
            for (int i = 0; i < MF; ++i) {
              const double asum = af[i].x + af[i].y;
#pragma unroll
              for (int j = 0; j < NF; ++j) {
                dmma(acc[0][i][j][0], acc[0][i][j][1], af[i].x, bf[j].x);
                dmma(acc[1][i][j][0], acc[1][i][j][1], af[i].y, bf[j].y);
                dmma(acc[2][i][j][0], acc[2][i][j][1], asum, bsum[j]);
              }
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) detail::mbar_arrive(&empty[s]);
    }
    return true;
  }

  __device__ static void store(T* __restrict__ C, int64_t ld, int m0, int n0, int M, int N, const Acc& acc) {
    TileCore<CPLX, MODE, BM, BN, BK, WARPS_M, WARPS_N, STAGES>::store(C, ld, m0, n0, M, N, acc);
  }
};

}  // namespace tnb

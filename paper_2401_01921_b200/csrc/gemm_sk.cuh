// Persistent, warp-specialised, stream-K FP64 DMMA GEMM core (the dense
// contraction hot loop, a11).
//
//  * one CTA per SM; CTA c owns the contiguous k-iteration range
//    [total*c/G, total*(c+1)/G) of the flattened (tile, k-tile) space, so every SM
//    gets the same amount of DMMA work whatever the tile count (no wave
//    quantisation, no split-K reduce pass);
//  * a producer warpgroup (4 warps) gathers operands for consecutive k-tiles --
//    across tile boundaries -- into a STAGES-deep ring (cp.async + "full"
//    mbarriers); 16 math warps (32x32 warp tiles of DMMA.8x8x4) consume and
//    release stages through "empty" mbarriers; no CTA-wide barrier in the loop;
//  * a tile split between CTAs is finished by the CTA that computes its last
//    k-tile ("owner"); earlier CTAs publish register partials to a workspace slot
//    and a flag; the owner adds them in CTA order (deterministic, no atomics on
//    data). All G CTAs are co-resident, so the owner's wait always completes.
#pragma once
#include "gemm_core.cuh"

namespace tnb {

struct GemmDesc {
  int M, N, K;
  int64_t a_elems, b_elems;  // operand extents (elements from the base pointers; checked builds)
  int tiles_m, tiles_n, splitk;
  int k_per_split;
  int a_mfast, b_nfast;
  int out_ld;
  // 1: every BM-row tile of A (BN-col tile of B) is one contiguous, 16-byte aligned run per
  // k: whole k-rows of the tile move by bulk copies instead of per-element cp.async
  int bulkA, bulkB;
  KAffine kaff;
  Group rowA, kA, kB, colB;
  // outmap: the output is written at rowC(m) + colC(n) (the caller's physical order of the
  // output axes, e.g. K-major for the step that consumes it) instead of m * out_ld + n
  int outmap;
  Group rowC, colC;
};

struct SKParams {
  int KT;          // k-tiles per output tile
  int G;           // persistent CTAs
  int64_t total;   // tiles * KT
  double* ws;      // [G][ACCN][NMATH] register partials
  int* flags;      // [G], zero before the launch
  int clear;       // owners reset the flags they consume (persistent workspace, no memset)
};

namespace detail {
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__host__ __device__ __forceinline__ int64_t sk_begin(int64_t total, int G, int c) { return total * c / G; }
__device__ __forceinline__ int sk_cta_of(int64_t total, int G, int64_t x) {
  int c = (int)((x * G) / total);
  while (c + 1 < G && sk_begin(total, G, c + 1) <= x) ++c;
  while (c > 0 && sk_begin(total, G, c) > x) --c;
  return c;
}
}  // namespace detail

template <bool CPLX, int MODE, int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, int NPROD_ = 128>
struct SKCore {
  using T = typename Elem<CPLX>::T;
  using Base = TileCore<CPLX, MODE, BM, BN, BK, WARPS_M, WARPS_N, STAGES>;
  static constexpr int ES = CPLX ? 16 : 8;
  static constexpr int NMATH = WARPS_M * WARPS_N * 32;
  static constexpr int NPROD = NPROD_;  // producer threads (whole warpgroups)
  static constexpr int NT = NMATH + NPROD;
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  static constexpr int MF = WTM / 8, NF = WTN / 8;
  static constexpr int LDA = BM + (CPLX ? 2 : 4);
  static constexpr int LDB = BN + (CPLX ? 2 : 4);
  static constexpr int NACC = CPLX ? (MODE == 1 ? 3 : 2) : 1;
  static constexpr int ACCN = NACC * MF * NF * 2;
  static constexpr int EA = (BM * BK) / NPROD, EB = (BN * BK) / NPROD;
  static constexpr int kMaxPeriod = 16;  // periodic-K offset tables: D0 <= 16 phases
  // warp-specialised register split (setmaxnreg) for the 640-thread dense kernel: launched at
  // kLaunchRegs per thread, producers drop to kProdRegs so the math warps can hold kMathRegs
  // (measured: chi=1024 f64 L.A.W.R GEMMs 1.356 -> 1.332 ms, c128 5.03 -> 4.96 ms)
  static constexpr bool kRegSplit = NMATH == 512 && NPROD == 128;
  static constexpr int kLaunchRegs = 96, kProdRegs = 64, kMathRegs = 104;
  static_assert(!kRegSplit || NMATH * (kMathRegs - kLaunchRegs) <= NPROD * (kLaunchRegs - kProdRegs),
                "register split must fit in the CTA's launch allocation");
  static constexpr size_t kSmem = (size_t)STAGES * BK * (LDA + LDB) * ES + (size_t)(BM + BN) * 8 +
                                  (size_t)2 * 2 * BK * 8 + (size_t)2 * STAGES * 8 + (size_t)2 * kMaxPeriod * BK * 8 +
                                  (size_t)(BM + BN) * 8;  // output-map offsets of the tile (outmap)
  static_assert(NMATH % 128 == 0, "math warps must form whole warpgroups");
  static_assert((BM * BK) % NPROD == 0 && (BN * BK) % NPROD == 0, "tile/producer mismatch");
  using Acc = typename Base::Acc;

  __device__ static void tile_coords(const GemmDesc& d, int64_t tile, int& m0, int& n0) {
    const int group = 8;
    const int per_group = group * d.tiles_n;
    const int t = (int)tile;
    const int g = t / per_group;
    const int first_m = g * group;
    const int gsz = min(d.tiles_m - first_m, group);
    const int in_g = t - g * per_group;
    m0 = (first_m + in_g % gsz) * BM;
    n0 = (in_g / gsz) * BN;
  }

  // Math warps: accumulate nk consecutive ring stages (gi = running stage counter).
  // mfa/nfa (< MF/NF on edge tiles): this warp's 8-row / 8-column fragments that hold
  // real output; the rest are padding and skip their DMMAs (warp-uniform).
  __device__ __forceinline__ static void consume(const T* As, const T* Bs, uint64_t* full, uint64_t* empty, uint32_t& gi, int nk,
                                 Acc& acc, int mfa = MF, int nfa = NF) {
    if (mfa >= MF && nfa >= NF) consume_impl<false>(As, Bs, full, empty, gi, nk, acc, MF, NF);
    else consume_impl<true>(As, Bs, full, empty, gi, nk, acc, mfa, nfa);
  }
  template <bool PRED>
  __device__ __forceinline__ static void consume_impl(const T* As, const T* Bs, uint64_t* full, uint64_t* empty, uint32_t& gi,
                                                      int nk, Acc& acc, int mfa, int nfa) {
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    int wm, wn;
    Base::warp_mn(warp, wm, wn);
    const int arow = wm * WTM + (lane >> 2);
    const int bcol = wn * WTN + (lane >> 2);
    const int kq = lane & 3;
    for (int kt = 0; kt < nk; ++kt, ++gi) {
      const int s = (int)(gi % STAGES);
      detail::mbar_wait(&full[s], (uint32_t)((gi / STAGES) & 1));
      if (PRED && (mfa <= 0 || nfa <= 0)) {  // all-padding warp tile: release the stage only
        __syncwarp();
        if (lane == 0) detail::mbar_arrive(&empty[s]);
        continue;
      }
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
            for (int j = 0; j < NF; ++j)
              if (!PRED || (i < mfa && j < nfa)) dmma(acc[0][i][j][0], acc[0][i][j][1], af[i], bf[j]);
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
                if (PRED && !(i < mfa && j < nfa)) continue;
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
                if (PRED && !(i < mfa && j < nfa)) continue;
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
  }

  // Epilogue through the output index map (outmap): element (m, n) at rowC(m) + colC(n); a
  // lane's column pair goes out as one 16-byte store when the two are adjacent and aligned.
  // The tile's BM row and BN column offsets are computed once (one per math thread) into
  // shared memory (tab: BM + BN entries) between two math-warp barriers.
  __device__ static void store_mapped(T* __restrict__ C, const GemmDesc& d, int m0, int n0, const Acc& acc,
                                      int64_t* tab) {
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    static_assert(BM + BN <= NMATH, "one output-map offset per math thread");
    if (tid < BM) tab[tid] = m0 + tid < d.M ? group_offset(d.rowC, (uint32_t)(m0 + tid)) : -1;
    else if (tid < BM + BN) tab[tid] = n0 + tid - BM < d.N ? group_offset(d.colC, (uint32_t)(n0 + tid - BM)) : -1;
    detail::named_sync(3, NMATH);
    int wm, wn;
    Base::warp_mn(warp, wm, wn);
    const int kq = lane & 3;
    int64_t co[NF][2];
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      const int n = wn * WTN + j * 8 + 2 * kq;
      co[j][0] = tab[BM + n];
      co[j][1] = tab[BM + n + 1];
    }
#pragma unroll
    for (int i = 0; i < MF; ++i) {
      const int64_t ro = tab[wm * WTM + i * 8 + (lane >> 2)];
      if (ro < 0) continue;
      T* row = C + ro;
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        T v0, v1;
        if constexpr (!CPLX) {
          v0 = acc[0][i][j][0];
          v1 = acc[0][i][j][1];
        } else if constexpr (MODE == 0) {
          v0 = make_double2(acc[0][i][j][0], acc[1][i][j][0]);
          v1 = make_double2(acc[0][i][j][1], acc[1][i][j][1]);
        } else {
          v0 = make_double2(acc[0][i][j][0] - acc[1][i][j][0], acc[2][i][j][0] - acc[0][i][j][0] - acc[1][i][j][0]);
          v1 = make_double2(acc[0][i][j][1] - acc[1][i][j][1], acc[2][i][j][1] - acc[0][i][j][1] - acc[1][i][j][1]);
        }
        if constexpr (!CPLX) {
          if (co[j][1] == co[j][0] + 1 && co[j][0] >= 0 && ((reinterpret_cast<uintptr_t>(row + co[j][0]) & 15) == 0)) {
            *reinterpret_cast<double2*>(row + co[j][0]) = make_double2(v0, v1);
            continue;
          }
        }
        if (co[j][0] >= 0) row[co[j][0]] = v0;
        if (co[j][1] >= 0) row[co[j][1]] = v1;
      }
    }
    detail::named_sync(3, NMATH);  // the table is rewritten by the next mapped epilogue
  }

  // Stream-K fix-up. A CTA that computed the head/middle of a tile finished by a later
  // CTA publishes its register partial to its workspace slot and raises its flag.
  __device__ __forceinline__ static void publish(double* ws, int* flags, int c, Acc& acc) {
    const int tid = threadIdx.x;
    double* flat = &acc[0][0][0][0];
    double* w = ws + (size_t)c * ACCN * NMATH;
#pragma unroll
    for (int r = 0; r < ACCN; ++r) __stcg(w + (size_t)r * NMATH + tid, flat[r]);
    // per warp: the warp barrier orders its lanes' stores before lane 0's gpu-scope release
    // (cumulative), so no CTA-wide barrier or per-thread fence: each warp moves on at once
    __syncwarp();
    if ((tid & 31) == 0) detail::red_release_add(flags + c, 1);
  }
  // The owner adds the partials of CTAs first..c-1 in CTA order (fixed summation
  // order). With clear, each consumed flag is reset (every CTA publishes at most
  // once per launch, so the flags are clean for the next launch without a memset).
  __device__ __forceinline__ static void absorb(const double* ws, int* flags, int first, int c, Acc& acc, bool clear) {
    const int tid = threadIdx.x;
    double* flat = &acc[0][0][0][0];
    for (int cc = first; cc < c; ++cc) {
      if (tid == 0) {
#if TNB_CHECKED
        long long spins = 0;
#endif
        while (detail::ld_acquire(flags + cc) < NMATH / 32) {  // every math warp of CTA cc published
#if TNB_CHECKED
          TNB_DCHECK(++spins < (1ll << 32), "stream-K partial never published");
#endif
        }
      }
      detail::named_sync(2, NMATH);
      const double* w = ws + (size_t)cc * ACCN * NMATH;
#pragma unroll
      for (int r = 0; r < ACCN; ++r) flat[r] += __ldcg(w + (size_t)r * NMATH + tid);
      if (clear && tid == 0) flags[cc] = 0;
    }
  }

  // Producer warp 0: the k-rows of a stage whose tile is contiguous per k go by bulk copy
  // (TMA engine; one copy per k-row: A rows by lanes 0..BK-1, B rows by lanes 16..16+BK-1),
  // completing as transaction bytes on full[s]. The k offset of row kk is per[kk] (periodic
  // K) or kk * ks (affine K).
  __device__ __forceinline__ static void bulk_rows(const GemmDesc& d, int s, const T* pa, const T* pb,
                                                   const int64_t* rowOffA, const int64_t* colOffB, const int64_t* pra,
                                                   const int64_t* prb, int64_t ksA, int64_t ksB, uint64_t* full,
                                                   uint32_t sAbase, uint32_t sBbase) {
    const int p = threadIdx.x - NMATH;
    if (p >= 32) return;
    constexpr uint32_t stA = BK * LDA * ES, stB = BK * LDB * ES;
    if (p == 0)
      detail::mbar_expect_tx(&full[s], (uint32_t)((d.bulkA ? BK * BM * ES : 0) + (d.bulkB ? BK * BN * ES : 0)));
    __syncwarp();
    if (d.bulkA && p < BK) {
      const T* src = pa + rowOffA[0] + (pra ? pra[p] : (int64_t)p * ksA);
      detail::bulk_load(sAbase + s * stA + (uint32_t)(p * LDA) * ES, src, BM * ES, &full[s]);
    }
    if (d.bulkB && p >= 16 && p < 16 + BK) {
      const int kk = p - 16;
      const T* src = pb + colOffB[0] + (prb ? prb[kk] : (int64_t)kk * ksB);
      detail::bulk_load(sBbase + s * stB + (uint32_t)(kk * LDB) * ES, src, BN * ES, &full[s]);
    }
  }
  template <bool AMF, bool BNF>
  __device__ static void run(unsigned char* smem, const T* __restrict__ A, const T* __restrict__ B,
                             T* __restrict__ C, const GemmDesc& d, const SKParams& sk) {
    T* As = reinterpret_cast<T*>(smem);
    T* Bs = As + STAGES * BK * LDA;
    int64_t* rowOffA = reinterpret_cast<int64_t*>(Bs + STAGES * BK * LDB);
    int64_t* colOffB = rowOffA + BM;
    int64_t* kOffA = colOffB + BN;    // [2][BK]
    int64_t* kOffB = kOffA + 2 * BK;  // [2][BK]
    uint64_t* full = reinterpret_cast<uint64_t*>(kOffB + 2 * BK);
    uint64_t* empty = full + STAGES;
    int64_t* perA = reinterpret_cast<int64_t*>(empty + STAGES);  // [D0][BK] periodic-K offsets
    int64_t* perB = perA + kMaxPeriod * BK;
    const int tid = threadIdx.x;
    const int c = blockIdx.x;
    const int64_t it0 = detail::sk_begin(sk.total, sk.G, c), it1 = detail::sk_begin(sk.total, sk.G, c + 1);
    const int KT = sk.KT;
    if (tid == 0) {
      for (int s = 0; s < STAGES; ++s) {
        detail::mbar_init(&full[s], NPROD);
        detail::mbar_init(&empty[s], NMATH / 32);
      }
    }
    __syncthreads();

    if (tid >= NMATH) {
      // ================================================================ producer
      // register split (launch: 96 per thread): the producer warpgroup gives 32 back, the
      // four math warpgroups take 8 more each (kRegSplit; the host checks the launch count)
      if constexpr (kRegSplit) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kProdRegs) : "memory");
      const int p = tid - NMATH;
      auto mapA = [&](int i, int& m, int& kk) {
        const int e = p + i * NPROD;
        if (AMF) { m = e % BM; kk = e / BM; }
        else { kk = (e & 3) + 4 * (e / (4 * BM)); m = (e >> 2) % BM; }
      };
      auto mapB = [&](int i, int& n, int& kk) {
        const int e = p + i * NPROD;
        if (BNF) { n = e % BN; kk = e / BN; }
        else { kk = (e & 3) + 4 * (e / (4 * BN)); n = (e >> 2) % BN; }
      };
      constexpr int RA = AMF ? 1 : 4, RB = BNF ? 1 : 4;
      const uint32_t sAbase = smem_u32(As), sBbase = smem_u32(Bs);
      constexpr uint32_t stA = BK * LDA * ES, stB = BK * LDB * ES;
      uint32_t gi = 0;  // stage counter (per CTA < 2^32)
      if (d.kaff.ok == 3) {
        // periodic K (two digits, inner width D0): offset(k0 + kk) = (k0 / D0) * s1 + per[k0 % D0][kk]
        const int D0 = d.kaff.D0;
        for (int x = p; x < D0 * BK; x += NPROD) {
          const int r = x / BK, kk = x - r * BK, t = r + kk, q = t / D0, rr = t - q * D0;
          perA[x] = (int64_t)q * d.kaff.s1A + (int64_t)rr * d.kaff.s0A;
          perB[x] = (int64_t)q * d.kaff.s1B + (int64_t)rr * d.kaff.s0B;
        }
        detail::named_sync(1, NPROD);
      }
      // segments in REVERSE range order: a CTA first publishes the partial of the tile it
      // shares with its successor and finishes (as owner) the tile it shares with its
      // predecessor last, so no CTA waits on one that is still early in its range
      for (int64_t e = it1; e > it0;) {
        const int64_t tile = (e - 1) / KT;
        const int64_t tstart = tile * KT;
        const int64_t sb = it0 > tstart ? it0 : tstart;
        const int kt0 = (int)(sb - tstart);
        const int kt1 = (int)(e - tstart);
        int m0, n0;
        tile_coords(d, tile, m0, n0);
        detail::named_sync(1, NPROD);  // previous segment's table reads are done
        for (int i = p; i < BM; i += NPROD) rowOffA[i] = (m0 + i < d.M) ? group_offset(d.rowA, m0 + i) : -1;
        for (int i = p; i < BN; i += NPROD) colOffB[i] = (n0 + i < d.N) ? group_offset(d.colB, n0 + i) : -1;
        detail::named_sync(1, NPROD);
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
        for (int kt = kt0; kt < kt1; ++kt, ++gi) {
          const int s = (int)(gi % STAGES);
          const int k0 = kt * BK;
          if (d.kaff.ok == 3 && k0 + BK <= d.K) {
            // periodic K: two digits, the inner one not a multiple of 16 wide
            const uint32_t q0 = d.kaff.div0.div((uint32_t)k0);
            const int r0 = k0 - (int)q0 * d.kaff.D0;
            const T* pa = A + (int64_t)q0 * d.kaff.s1A;
            const T* pb = B + (int64_t)q0 * d.kaff.s1B;
            const int64_t* pra = perA + r0 * BK;
            const int64_t* prb = perB + r0 * BK;
            if (gi >= STAGES) detail::mbar_wait(&empty[s], (uint32_t)(((gi / STAGES) & 1) ^ 1));
            if (d.bulkA | d.bulkB) bulk_rows(d, s, pa, pb, rowOffA, colOffB, pra, prb, 0, 0, full, sAbase, sBbase);
            if (!d.bulkA)
#pragma unroll
            for (int i = 0; i < EA; ++i) {
              int m, kk;
              mapA(i, m, kk);
              const int64_t ro = rA[i % RA];
              const bool v = ro >= 0;
              const T* src = v ? pa + ro + pra[kk] : A;
              TNB_DCHECK(!v || (src >= A && src - A < d.a_elems), "dense A gather (periodic K)");
              const uint32_t dst = sAbase + s * stA + (uint32_t)(kk * LDA + m) * ES;
              if constexpr (CPLX)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 16 : 0));
              else
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 8 : 0));
            }
if (!d.bulkB)
#pragma unroll
            for (int i = 0; i < EB; ++i) {
              int n, kk;
              mapB(i, n, kk);
              const int64_t co = rB[i % RB];
              const bool v = co >= 0;
              const T* src = v ? pb + co + prb[kk] : B;
              TNB_DCHECK(!v || (src >= B && src - B < d.b_elems), "dense B gather (periodic K)");
              const uint32_t dst = sBbase + s * stB + (uint32_t)(kk * LDB + n) * ES;
              if constexpr (CPLX)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 16 : 0));
              else
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 8 : 0));
            }
          } else if (d.kaff.ok >= 1 && d.kaff.ok <= 2 && d.kaff.ok >= (BK + 15) / 16 && k0 + BK <= d.K) {
            const T* pa = A + group_offset(d.kA, k0);
            const T* pb = B + group_offset(d.kB, k0);
            if (gi >= STAGES) detail::mbar_wait(&empty[s], (uint32_t)(((gi / STAGES) & 1) ^ 1));
            if (d.bulkA | d.bulkB)
              bulk_rows(d, s, pa, pb, rowOffA, colOffB, nullptr, nullptr, d.kaff.ksA, d.kaff.ksB, full, sAbase, sBbase);
            if (!d.bulkA)
#pragma unroll
            for (int i = 0; i < EA; ++i) {
              int m, kk;
              mapA(i, m, kk);
              const int64_t ro = rA[i % RA];
              const bool v = ro >= 0;
              const T* src = v ? pa + ro + (int64_t)kk * d.kaff.ksA : A;
              TNB_DCHECK(!v || (src >= A && src - A < d.a_elems), "dense A gather (affine K)");
              const uint32_t dst = sAbase + s * stA + (uint32_t)(kk * LDA + m) * ES;
              if constexpr (CPLX)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 16 : 0));
              else
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 8 : 0));
            }
if (!d.bulkB)
#pragma unroll
            for (int i = 0; i < EB; ++i) {
              int n, kk;
              mapB(i, n, kk);
              const int64_t co = rB[i % RB];
              const bool v = co >= 0;
              const T* src = v ? pb + co + (int64_t)kk * d.kaff.ksB : B;
              TNB_DCHECK(!v || (src >= B && src - B < d.b_elems), "dense B gather (affine K)");
              const uint32_t dst = sBbase + s * stB + (uint32_t)(kk * LDB + n) * ES;
              if constexpr (CPLX)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 16 : 0));
              else
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 8 : 0));
            }
          } else {
            // irregular K group or ragged last k-tile: per-k offsets through a table
            const int slot = (int)(gi & 1);
            for (int i = p; i < 2 * BK; i += NPROD) {
              const int kk = i % BK, k = k0 + kk;
              const bool v = k < d.K;
              if (i < BK) kOffA[slot * BK + kk] = v ? group_offset(d.kA, k) : -1;
              else kOffB[slot * BK + kk] = v ? group_offset(d.kB, k) : -1;
            }
            detail::named_sync(1, NPROD);
            if (gi >= STAGES) detail::mbar_wait(&empty[s], (uint32_t)(((gi / STAGES) & 1) ^ 1));
            const int64_t* ka = kOffA + slot * BK;
            const int64_t* kb = kOffB + slot * BK;
#pragma unroll
            for (int i = 0; i < EA; ++i) {
              int m, kk;
              mapA(i, m, kk);
              const int64_t ro = rA[i % RA], ko = ka[kk];
              const bool v = (ro >= 0) && (ko >= 0);
              const T* src = v ? A + ro + ko : A;
              TNB_DCHECK(!v || (src >= A && src - A < d.a_elems), "dense A gather (table)");
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
              const int64_t co = rB[i % RB], ko = kb[kk];
              const bool v = (co >= 0) && (ko >= 0);
              const T* src = v ? B + co + ko : B;
              TNB_DCHECK(!v || (src >= B && src - B < d.b_elems), "dense B gather (table)");
              const uint32_t dst = sBbase + s * stB + (uint32_t)(kk * LDB + n) * ES;
              if constexpr (CPLX)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 16 : 0));
              else
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 8 : 0));
            }
          }
          detail::cp_async_mbar_arrive_noinc(&full[s]);
        }
        e = sb;
      }
      cp_async_wait<0>();
      return;
    }

    // ================================================================== math warps
    if constexpr (kRegSplit) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kMathRegs) : "memory");
    uint32_t gi = 0;
    Acc acc;
    // segments in REVERSE range order: a CTA first publishes the partial of the tile it
    // shares with its successor and finishes (as owner) the tile it shares with its
    // predecessor last, so no CTA waits on one that is still early in its range
    for (int64_t e = it1; e > it0;) {
      const int64_t tile = (e - 1) / KT;
      const int64_t tstart = tile * KT;
      const int64_t sb = it0 > tstart ? it0 : tstart;
      const int kt0 = (int)(sb - tstart);
      const int kt1 = (int)(e - tstart);
      Base::zero(acc);
      consume(As, Bs, full, empty, gi, kt1 - kt0, acc);
      // ---- epilogue of this segment
      int m0, n0;
      tile_coords(d, tile, m0, n0);
      if (kt1 < KT) {
        publish(sk.ws, sk.flags, c, acc);
      } else {
        if (kt0 > 0) absorb(sk.ws, sk.flags, detail::sk_cta_of(sk.total, sk.G, tile * (int64_t)KT), c, acc, sk.clear != 0);
        if (d.outmap) store_mapped(C, d, m0, n0, acc, perB + kMaxPeriod * BK);
        else Base::store(C, d.out_ld, m0, n0, d.M, d.N, acc);
      }
      e = sb;
    }
  }
};

}  // namespace tnb

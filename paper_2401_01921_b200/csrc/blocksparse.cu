// a12: U(1)/Z_n block-sparse pairwise contraction -- the B200 replacement for
// _contract_pair_blocks (pkg/src/tnkit/contract.py:137-167).
//
// Reference semantics:
//   b_by_key[qn_b[b_pos]] -> [j ascending]                       (contract.py:148-151)
//   for i in a-block order: for j in b_by_key[qn_a[a_pos]]:       (contract.py:152-156)
//       out[out_qn] += tensordot(A_i, B_j, (a_pos, b_pos))       (contract.py:157-164)
//   out_qn = qn_a[a_free] + qn_b[b_free]; every zero-flux output block exists
//   and starts at zero (contract.py:145-146).
//
// B200 design:
//   1. One H2D copy of all block metadata (qn tuples, per-block address groups,
//      output tile list) from a pinned staging buffer, once per block STRUCTURE
//      (plans are cached on the device).
//   2. pairing kernel (ON DEVICE, one CTA, qn tables staged in shared memory):
//      thread per output block o finds its contributing pairs (i asc, j asc) --
//      exactly the reference's accumulation order restricted to o -- and writes
//      a CSR (out_ptr, pair list); then the per-tile k-iteration counts
//      (sum over the tile's pairs of ceil(K_i / BK)) are scanned into tile_kbeg.
//   3. grouped stream-K GEMM (one persistent CTA per SM, warp-specialised like
//      the dense path, gemm_sk.cuh): the k-iterations of ALL output tiles -- each
//      tile's pairs concatenated in reference order -- form one flat iteration
//      space split evenly over the CTAs, so the few large sectors no longer set
//      the critical path. A producer warpgroup gathers A/B k-tiles pair by pair
//      (index groups per block, cp.async into an mbarrier ring); 16 math warps
//      only do LDS + DMMA. A tile split across CTAs is finished by the CTA that
//      holds its last k-iteration, adding the earlier CTAs' partials in CTA
//      order (deterministic, no data atomics; flags self-reset for the next
//      launch). Tiles of blocks without pairs are stored as zeros.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <array>
#include <climits>
#include <map>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "gemm_sk.cuh"

#ifndef TNB_TWIN_WM
#define TNB_TWIN_WM 4
#endif
#ifndef TNB_TWIN_STAGES
#define TNB_TWIN_STAGES 6
#endif
#ifndef TNB_BS_NPROD0
#define TNB_BS_NPROD0 256
#endif
#ifndef TNB_BS_NPROD1
#define TNB_BS_NPROD1 128  // twin plan: one producer warpgroup (64 x C4: 1.031 -> 1.016 ms)
#endif

namespace tnb {
namespace {

struct alignas(16) BlockDesc {
  Group free_g;  // A: rows (a_free), B: cols (b_free)
  Group k_g;     // contracted axes, in shared-label order (not merged; consistent across A/B)
  int32_t F;     // product of free dims
  int32_t K;     // product of contracted dims
};

struct TileRef {
  int32_t o, m0, n0, panel;  // panel = (o, m0 / TNB_BS_PANEL_ROWS) in output-block order
};

struct BsMeta {
  int na, nb, nout, ntiles;
  int ra, rb, ro, nc, nfa, nfb;
  int32_t a_axes[TNB_MAX_RANK], b_axes[TNB_MAX_RANK];
  int32_t a_free[TNB_MAX_RANK], b_free[TNB_MAX_RANK];
  // device pointers into the metadata blob
  const int32_t* a_qn;
  const int32_t* b_qn;
  const int32_t* out_qn;
  const int32_t* out_M;
  const int32_t* out_N;
  const BlockDesc* da;
  const BlockDesc* db;
  const TileRef* tiles;
  const void* const* ptrs;  // device table [na + nb + nout] (large plans); else PtrTable
  int32_t* out_ptr;   // [nout+1] written by the pairing kernel
  int32_t* pairs;     // [max pairs][2] (i, j) grouped by output block
  int32_t* err;       // [1]
  const uint8_t* mask;  // per-panel "compute here" flags (multi-GPU partition) or nullptr
  int32_t* tile_kbeg;   // [ntiles+1] prefix sums of per-tile k-iterations, in SCHEDULE order
  int32_t* tile_cnt;    // [ntiles] scratch: k-iterations per tile in list order
  TileRef* stiles;      // [ntiles] the tiles in schedule order (written by the pairing kernel)
  int64_t max_pairs;
  int bk;               // k-tile depth of the GEMM (per-tile iteration counts)
  int qn_smem;          // qn tables fit in the pairing kernel's shared memory
  int sched_smem;       // bytes of schedule tables the GEMM stages in shared memory (0 = read from global)
  int desc_smem;        // the GEMM also stages the block descriptors (da, db) in shared memory
  // the schedule tables (tile_kbeg, stiles, out_ptr, pairs, out_M, out_N) and then da, db lie
  // back to back in the blob in exactly the shared-memory layout: one flat uint4 copy stages them
  const uint4* img;
  // batched execute: nbatch contractions of this structure in one launch (tile space
  // nbatch x ntiles; pointer table [nbatch][na + nb + nout] in device memory)
  int nbatch;
  // whole-tile schedule (single contractions): the pairing kernel assigns whole tiles to the
  // sched_G CTAs by LPT when the makespan stays within lpt_slack k-iterations of the even
  // split, lays the schedule out CTA by CTA and writes each CTA's range start to cta_beg
  // ([sched_G + 1]; cta_beg[0] = -1: stream-K split instead).
  int32_t* cta_beg;
  int sched_G;
  int lpt_slack;
};

// Schedule tables the grouped GEMM reads on every segment / pair switch (dependent
// loads): staged once per CTA in shared memory, right after the GEMM's own buffers.
__host__ __device__ inline size_t al16(size_t x) { return (x + 15) / 16 * 16; }
__host__ __device__ inline size_t sched_bytes(int ntiles, int nout, int64_t npairs) {
  return al16((size_t)(ntiles + 1) * 4) + (size_t)ntiles * 16 + al16((size_t)(nout + 1) * 4) +
         al16((size_t)npairs * 8) + 2 * al16((size_t)nout * 4);
}

// ---- pairing: one CTA; thread per output block -----------------------------
__device__ __forceinline__ bool a_matches(const BsMeta& m, const int32_t* aqn, const int32_t* oqn, int i, int o) {
  const int32_t* aq = aqn + (int64_t)i * m.ra;
  const int32_t* oq = oqn + (int64_t)o * m.ro;
  for (int f = 0; f < m.nfa; ++f)
    if (aq[m.a_free[f]] != oq[f]) return false;
  return true;
}
__device__ __forceinline__ bool b_matches(const BsMeta& m, const int32_t* aqn, const int32_t* bqn,
                                          const int32_t* oqn, int i, int j, int o) {
  const int32_t* aq = aqn + (int64_t)i * m.ra;
  const int32_t* bq = bqn + (int64_t)j * m.rb;
  const int32_t* oq = oqn + (int64_t)o * m.ro + m.nfa;
  for (int c = 0; c < m.nc; ++c)
    if (aq[m.a_axes[c]] != bq[m.b_axes[c]]) return false;
  for (int f = 0; f < m.nfb; ++f)
    if (bq[m.b_free[f]] != oq[f]) return false;
  return true;
}

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// In place: a[0..n) := inclusive prefix sums (one CTA, blockDim a multiple of 32).
__device__ void cta_inclusive_scan(int32_t* a, int n) {
  __shared__ int32_t carry;
  __shared__ int32_t wsum[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int base = 0; base < n; base += blockDim.x) {
    const int o = base + threadIdx.x;
    int v = (o < n) ? a[o] : 0;
    for (int s = 1; s < 32; s <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, v, s);
      if (lane >= s) v += t;
    }
    if (lane == 31) wsum[warp] = v;
    __syncthreads();
    if (warp == 0) {
      int w = (lane < (int)(blockDim.x >> 5)) ? wsum[lane] : 0;
      for (int s = 1; s < 32; s <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, w, s);
        if (lane >= s) w += t;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    const int incl = v + (warp > 0 ? wsum[warp - 1] : 0) + carry;
    __syncthreads();
    if (o < n) a[o] = incl;
    if (threadIdx.x == blockDim.x - 1) carry = incl;
    __syncthreads();
  }
}

// Shared-memory layout of the pairing kernel (qn tables, CSR, per-tile counts): every
// table is re-read many times by dependent loops, so all of it lives on chip when it fits.
constexpr int kLptMaxG = 1024;  // whole-tile LPT schedules for grids up to this size
// A whole-tile schedule is used when its makespan exceeds the even stream-K split by at most
// this many k-iterations: every stream-K segment boundary costs a partial publish or absorb
// and a segment start (~1-2 us each, per-CTA traces), i.e. several k-iterations of 64 x 64 DMMA.
constexpr int kLptSlackDefault = 12;
__host__ __device__ inline size_t lpt_smem_offset(const BsMeta& m) {
  return al16(((size_t)m.na * m.ra + (size_t)m.nb * m.rb + (size_t)m.nout * m.ro) * 4) +
         al16((size_t)(m.nout + 1) * 4) + al16((size_t)m.na * 4) + al16((size_t)m.ntiles * 4) +
         al16((size_t)m.ntiles * 8);
}
__host__ __device__ inline size_t pair_smem_bytes(const BsMeta& m) {
  const size_t lpt = (m.cta_beg && m.sched_G > 0 && m.sched_G <= kLptMaxG)
                         ? al16((size_t)m.ntiles * 8) + (size_t)m.sched_G * 12 : 0;
  return lpt_smem_offset(m) + lpt;
}

__global__ void __launch_bounds__(1024) bs_pair_kernel(const BsMeta m) {
  extern __shared__ __align__(16) unsigned char psm[];
  long long* stamp = reinterpret_cast<long long*>(m.err + 4);  // dev: phase timestamps
  int nst = 0;
#define TNB_STAMP() \
  if (threadIdx.x == 0 && nst < 16) stamp[nst++] = gtimer();
  TNB_STAMP()
  const int32_t* aqn = m.a_qn;
  const int32_t* bqn = m.b_qn;
  const int32_t* oqn = m.out_qn;
  int32_t* optr = m.out_ptr;    // [nout+1]: counts, then the CSR row pointer
  int32_t* tcnt = m.tile_cnt;   // [ntiles] k-iterations per tile (list order)
  int32_t* kblk = nullptr;      // [na] K of each A block (smem only)
  const int na_ = m.na * m.ra, nb_ = m.nb * m.rb, no_ = m.nout * m.ro;
  if (m.qn_smem) {
    int32_t* q = reinterpret_cast<int32_t*>(psm);
    for (int x = threadIdx.x; x < na_; x += blockDim.x) q[x] = m.a_qn[x];
    for (int x = threadIdx.x; x < nb_; x += blockDim.x) q[na_ + x] = m.b_qn[x];
    for (int x = threadIdx.x; x < no_; x += blockDim.x) q[na_ + nb_ + x] = m.out_qn[x];
    aqn = q;
    bqn = q + na_;
    oqn = q + na_ + nb_;
    unsigned char* r = psm + al16((size_t)(na_ + nb_ + no_) * 4);
    optr = reinterpret_cast<int32_t*>(r);
    r += al16((size_t)(m.nout + 1) * 4);
    kblk = reinterpret_cast<int32_t*>(r);
    r += al16((size_t)m.na * 4);
    tcnt = reinterpret_cast<int32_t*>(r);
    for (int x = threadIdx.x; x < m.na; x += blockDim.x) kblk[x] = m.da[x].K;
    __syncthreads();
  }
  TNB_STAMP()
  // warp per output block: the A-block test is warp-uniform, lanes sweep the B blocks
  // (a thread-per-block loop nest diverges and serialises across the warp)
  const int lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  for (int o = threadIdx.x >> 5; o < m.nout; o += nwarp) {
    int c = 0;
    for (int i = 0; i < m.na; ++i) {
      if (!a_matches(m, aqn, oqn, i, o)) continue;
      for (int j0 = 0; j0 < m.nb; j0 += 32) {
        const bool hit = j0 + lane < m.nb && b_matches(m, aqn, bqn, oqn, i, j0 + lane, o);
        c += __popc(__ballot_sync(0xffffffffu, hit));
      }
    }
    if (lane == 0) optr[o + 1] = c;
  }
  if (threadIdx.x == 0) optr[0] = 0;
  __syncthreads();
  TNB_STAMP()
  cta_inclusive_scan(optr + 1, m.nout);
  TNB_STAMP()
  // write pairs of each output block in reference order (i asc, j asc)
  if (optr[m.nout] > m.max_pairs) {
    if (threadIdx.x == 0) m.err[0] = 1;
    return;
  }
  for (int o = threadIdx.x >> 5; o < m.nout; o += nwarp) {
    int p = optr[o];
    int kt = 0;
    for (int i = 0; i < m.na; ++i) {
      if (!a_matches(m, aqn, oqn, i, o)) continue;
      const int kti = ((kblk ? kblk[i] : m.da[i].K) + m.bk - 1) / m.bk;
      for (int j0 = 0; j0 < m.nb; j0 += 32) {
        const bool hit = j0 + lane < m.nb && b_matches(m, aqn, bqn, oqn, i, j0 + lane, o);
        const unsigned bal = __ballot_sync(0xffffffffu, hit);
        if (hit) {
          const int q = p + __popc(bal & ((1u << lane) - 1u));  // j ascending within i
          m.pairs[2 * q] = i;
          m.pairs[2 * q + 1] = j0 + lane;
        }
        p += __popc(bal);
        kt += __popc(bal) * kti;
      }
    }
    if (lane == 0) {
      m.out_ptr[o + 1] = optr[o + 1];  // the CSR row pointer the GEMM reads
      if (o == 0) m.out_ptr[0] = 0;
      // every tile of block o has the same k-iterations; tile_kbeg (ntiles+1 >= nout
      // entries) serves as scratch for them until the final prefix sums overwrite it
      m.tile_kbeg[o] = kt;
    }
  }
  __syncthreads();
  TNB_STAMP()
  // k-iterations per output tile (0 for tiles of other ranks' panels)
  for (int t = threadIdx.x; t < m.ntiles; t += blockDim.x) {
    const TileRef tr = m.tiles[t];
    tcnt[t] = (!m.mask || m.mask[tr.panel]) ? m.tile_kbeg[tr.o] : 0;
  }
  __syncthreads();
  // schedule order: tiles ranked by k-iterations (descending, stable), laid out
  // big, small, big, small, ... so that every stream-K range holds at most a few
  // short segments (each segment / pair switch has a fixed gather set-up latency)
  TNB_STAMP()
  const bool reorder = m.qn_smem && m.ntiles <= 4096;
  if (reorder && m.cta_beg && m.sched_G > 0 && m.sched_G <= kLptMaxG) {
    // whole-tile LPT: rank tiles by k-iterations (descending, stable), then one warp hands
    // each tile in rank order to the least-loaded CTA (lowest index on ties). Scratch lives
    // in shared memory after the pairing tables (pair_smem_bytes reserves it).
    const int G = m.sched_G;
    unsigned char* r0 = psm + lpt_smem_offset(m);
    int32_t* lrank = reinterpret_cast<int32_t*>(r0);
    int32_t* lasg = lrank + m.ntiles;
    long long* lload = reinterpret_cast<long long*>(r0 + al16((size_t)m.ntiles * 8));
    int32_t* lnext = reinterpret_cast<int32_t*>(lload + G);
    __shared__ int lpt_ok;
    for (int t = threadIdx.x; t < m.ntiles; t += blockDim.x) {
      const int ct = tcnt[t];
      int r = 0;
      for (int u = 0; u < m.ntiles; ++u) {
        const int cu = tcnt[u];
        r += (cu > ct || (cu == ct && u < t)) ? 1 : 0;
      }
      lrank[r] = t;
    }
    for (int c = threadIdx.x; c < G; c += blockDim.x) {
      lload[c] = 0;
      lnext[c] = 0;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      long long total = 0, mk = 0;
      for (int r = 0; r < m.ntiles; ++r) {
        const int t = lrank[r];
        long long bv = LLONG_MAX;
        int bc = G;
        for (int c = lane; c < G; c += 32)
          if (lload[c] < bv) { bv = lload[c]; bc = c; }  // strided scan: the lane's first minimum
#pragma unroll
        for (int s = 16; s; s >>= 1) {
          const long long ov = __shfl_xor_sync(0xffffffffu, bv, s);
          const int oc = __shfl_xor_sync(0xffffffffu, bc, s);
          if (ov < bv || (ov == bv && oc < bc)) { bv = ov; bc = oc; }
        }
        __syncwarp();
        if (lane == 0) {
          lload[bc] += tcnt[t];
          lasg[t] = bc;
        }
        total += tcnt[t];
        mk = max(mk, bv + tcnt[t]);
        __syncwarp();
      }
      if (lane == 0) lpt_ok = mk <= (total + G - 1) / G + m.lpt_slack;
    }
    __syncthreads();
    if (lpt_ok) {
      // layout CTA by CTA (a CTA's tiles in rank order); cta_beg = prefix sums of the loads
      for (int t = threadIdx.x; t < m.ntiles; t += blockDim.x) atomicAdd(&lnext[lasg[t]], 1);
      __syncthreads();
      if (threadIdx.x == 0) {
        int pos = 0;
        long long kb = 0;
        for (int c = 0; c < G; ++c) {
          const int n = lnext[c];
          lnext[c] = pos;
          pos += n;
          m.cta_beg[c] = (int32_t)kb;
          kb += lload[c];
        }
        m.cta_beg[G] = (int32_t)kb;
        for (int r = 0; r < m.ntiles; ++r) {
          const int t = lrank[r];
          const int p = lnext[lasg[t]]++;
          m.stiles[p] = m.tiles[t];
          m.tile_cnt[p] = tcnt[t];
        }
      }
      __syncthreads();
      for (int t = threadIdx.x; t < m.ntiles; t += blockDim.x) tcnt[t] = m.tile_cnt[t];
      __syncthreads();
      cta_inclusive_scan(tcnt, m.ntiles);
      for (int t = threadIdx.x; t <= m.ntiles; t += blockDim.x) m.tile_kbeg[t] = t ? tcnt[t - 1] : 0;
      return;
    }
    if (threadIdx.x == 0) m.cta_beg[0] = -1;
    __syncthreads();
  } else if (m.cta_beg && threadIdx.x == 0) {
    m.cta_beg[0] = -1;
  }
  for (int t = threadIdx.x; t < m.ntiles; t += blockDim.x) {
    int pos = t;
    const int ct = tcnt[t];
    if (reorder) {
      int r = 0;
      for (int u = 0; u < m.ntiles; ++u) {
        const int cu = tcnt[u];
        r += (cu > ct || (cu == ct && u < t)) ? 1 : 0;
      }
      const int half = (m.ntiles + 1) / 2;
      pos = r < half ? 2 * r : 2 * (m.ntiles - 1 - r) + 1;
    }
    m.stiles[pos] = m.tiles[t];
    m.tile_cnt[pos] = ct;  // (global copy, schedule order)
  }
  __syncthreads();
  for (int t = threadIdx.x; t < m.ntiles; t += blockDim.x) tcnt[t] = m.tile_cnt[t];
  __syncthreads();
  TNB_STAMP()
  cta_inclusive_scan(tcnt, m.ntiles);
  TNB_STAMP()
  for (int t = threadIdx.x; t <= m.ntiles; t += blockDim.x) m.tile_kbeg[t] = t ? tcnt[t - 1] : 0;
  TNB_STAMP()
#undef TNB_STAMP
}

// ---- grouped stream-K GEMM --------------------------------------------------
template <bool CPLX, int MODE, int SHAPE = 0>
struct BsCfg {
  // 64x64 tiles suit the sector sizes; at this tile size the gather rate, not the DMMA
  // rate, is the limit, so two producer warpgroups feed the 16 math warps (measured: 4 math
  // warps of 32x32 tiles at 1 or 2 CTAs per SM 15% slower; 8 math warps of 32x16 tiles + one
  // producer warpgroup at 2 CTAs per SM 10% slower)
  // (r02, 64 x C4 batch: NPROD 64 / 128 and BK 32 with 4-5 stages measured no better)
  // SHAPE 1 (float64 batches): 64 x 128 tiles, 6 stages -- per stage twice the DMMA work for
  // the same ring hand-off, which pays once every CTA walks thousands of k-iterations (64 x C4:
  // 1.116 -> 1.021 ms) but not for one contraction (C4: 33.3 -> 35.4 us)
  static constexpr int BM = 64, BN = SHAPE ? 128 : 64, BK = CPLX ? 8 : 16, WM = SHAPE ? TNB_TWIN_WM : 4, WN = 4,
                       STAGES = SHAPE ? TNB_TWIN_STAGES : 8, NPROD = SHAPE ? TNB_BS_NPROD1 : TNB_BS_NPROD0;
  using Core = SKCore<CPLX, MODE, BM, BN, BK, WM, WN, STAGES, NPROD>;
};

// Per-call data pointers (A blocks, B blocks, output blocks) travel as a kernel
// parameter when they fit, so a cached plan needs no per-call H2D copy.
// Two sizes: the parameter block is copied at every launch, so small structures
// (<= 128 blocks in all) do not pay for 8 KB of unused slots.
constexpr int kInlinePtrs = 1024, kInlinePtrsSmall = 128;
template <int NP>
struct PtrTable {
  const void* p[NP];
};

struct BsSK {
  double* ws;  // [G][ACCN][NMATH] register partials
  int* flags;  // [G], zero between launches (consumers reset them)
  // dev instrumentation (TNB_BS_TRACE=file): per CTA [kTraceW] int64 of %globaltimer stamps
  long long* trace;
  // dev experiments (TNB_BS_EXP): bit 0 = producers issue no copies, bit 1 = math warps
  // issue no DMMA (the skeleton's cost without memory traffic / tensor work), bits 2 / 3 =
  // whole k-tiles skip their A / B copies
  int exp;
};
constexpr int kTraceW = 64;


template <bool CPLX, int MODE, bool AMF, bool BNF, int NP, int SHAPE>
__global__ void __launch_bounds__(BsCfg<CPLX, MODE, SHAPE>::Core::NT, 1)
    bs_sk_kernel(const __grid_constant__ BsMeta m, const __grid_constant__ PtrTable<NP> pt, const BsSK sk) {
  using Cfg = BsCfg<CPLX, MODE, SHAPE>;
  using Core = typename Cfg::Core;
  using Base = typename Core::Base;
  using T = typename Core::T;
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES;
  constexpr int NMATH = Core::NMATH, NPROD = Core::NPROD, ES = Core::ES;
  constexpr int LDA = Core::LDA, LDB = Core::LDB, EA = Core::EA, EB = Core::EB;
  extern __shared__ __align__(16) unsigned char smem[];
  T* As = reinterpret_cast<T*>(smem);
  T* Bs = As + STAGES * BK * LDA;
  int64_t* rowOffA = reinterpret_cast<int64_t*>(Bs + STAGES * BK * LDB);
  int64_t* colOffB = rowOffA + BM;
  int64_t* kOffA = colOffB + BN;    // [2][BK]
  int64_t* kOffB = kOffA + 2 * BK;  // [2][BK]
  uint64_t* full = reinterpret_cast<uint64_t*>(kOffB + 2 * BK);
  uint64_t* empty = full + STAGES;

  const long long t_entry = sk.trace ? gtimer() : 0;
  const void* const* ptrs = m.ptrs ? m.ptrs : pt.p;
  const int tid = threadIdx.x;
  const int c = blockIdx.x;
  // whole-tile schedule bounds: loaded first, in flight while the tables are staged
  int32_t wb0 = -1, wb1 = -1, wbz = -1;
  if (m.nbatch == 1 && m.cta_beg && m.sched_G == (int)gridDim.x) {
    wbz = __ldg(m.cta_beg);
    wb0 = __ldg(m.cta_beg + c);
    wb1 = __ldg(m.cta_beg + c + 1);
  }
  const int* kbeg = m.tile_kbeg;
  const TileRef* tiles = m.stiles;
  const BlockDesc* DA = m.da;
  const BlockDesc* DB = m.db;
  const int32_t* optr = m.out_ptr;
  const int32_t* pairs = m.pairs;
  const int32_t* oM = m.out_M;
  const int32_t* oN = m.out_N;
  if (m.sched_smem) {
    // one round of independent loads instead of a chain of dependent ones per segment
    unsigned char* q = smem + al16(Core::kSmem);
    int32_t* s_kbeg = reinterpret_cast<int32_t*>(q);
    q += al16((size_t)(m.ntiles + 1) * 4);
    TileRef* s_tiles = reinterpret_cast<TileRef*>(q);
    q += (size_t)m.ntiles * 16;
    int32_t* s_optr = reinterpret_cast<int32_t*>(q);
    q += al16((size_t)(m.nout + 1) * 4);
    int32_t* s_pairs = reinterpret_cast<int32_t*>(q);
    q += al16((size_t)m.max_pairs * 8);
    int32_t* s_oM = reinterpret_cast<int32_t*>(q);
    q += al16((size_t)m.nout * 4);
    int32_t* s_oN = reinterpret_cast<int32_t*>(q);
    {
      // one flat copy of the blob's image of this region: all loads of a thread are
      // independent (a cold-L2 round trip once, not once per table)
      uint4* dst = reinterpret_cast<uint4*>(smem + al16(Core::kSmem));
      const int n16 = m.sched_smem / 16, nt = blockDim.x;
      for (int x = tid; x < n16; x += 4 * nt) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (x + u * nt < n16) v[u] = __ldg(m.img + x + u * nt);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (x + u * nt < n16) dst[x + u * nt] = v[u];
      }
    }
    if (m.desc_smem) {
      // block descriptors: read on every pair switch by the producers
      q += al16((size_t)m.nout * 4);
      DA = reinterpret_cast<const BlockDesc*>(q);
      DB = DA + m.na;
    }
    kbeg = s_kbeg;
    tiles = s_tiles;
    optr = s_optr;
    pairs = s_pairs;
    oM = s_oM;
    oN = s_oN;
  }
  __syncthreads();
  const int64_t per = kbeg[m.ntiles];  // k-iterations of one contraction
  const int64_t total = per * m.nbatch;
  const int NPI = m.na + m.nb + m.nout;  // pointers per batch item
  // stream-K participants: >= 4 k-iterations each, so no participant has an empty range
  // (an owner waits on EVERY participant between a tile's first CTA and itself)
  // whole-tile schedule (no tile split across CTAs: no partial publish / absorb) when the
  // pairing kernel laid one out for exactly this grid; else the even stream-K split
  const bool whole = wbz == 0;
  const int G = whole ? (int)gridDim.x : (int)min((int64_t)gridDim.x, max(total / 4, (int64_t)1));
  const int64_t it0 = whole ? wb0 : (c < G ? detail::sk_begin(total, G, c) : 0);
  const int64_t it1 = whole ? wb1 : (c < G ? detail::sk_begin(total, G, c + 1) : 0);
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      detail::mbar_init(&full[s], NPROD);
      detail::mbar_init(&empty[s], NMATH / 32);
    }
  }
  __syncthreads();
  // batch item of a flattened k-iteration, and the item's first k-iteration
  auto item_of = [&](int64_t x, int64_t& base) {
    const int b = m.nbatch == 1 ? 0 : (int)(x / per);
    base = (int64_t)b * per;
    return b;
  };
  // largest tile t with kbeg[t] <= x (skips empty tiles, whose kbeg equals the next one's)
  auto tile_of = [&](int64_t x) {
    int lo = 0, hi = m.ntiles - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (kbeg[mid] <= x) lo = mid;
      else hi = mid - 1;
    }
    return lo;
  };

  if (tid >= NMATH) {
    // ================================================================ producer
    const int p = tid - NMATH;
    auto mapA = [&](int i, int& mm, int& kk) {
      const int e = p + i * NPROD;
      if (AMF) { mm = e % BM; kk = e / BM; }
      else { kk = (e & 3) + 4 * (e / (4 * BM)); mm = (e >> 2) % BM; }
    };
    auto mapB = [&](int i, int& nn, int& kk) {
      const int e = p + i * NPROD;
      if (BNF) { nn = e % BN; kk = e / BN; }
      else { kk = (e & 3) + 4 * (e / (4 * BN)); nn = (e >> 2) % BN; }
    };
    constexpr int RA = AMF ? 1 : 4, RB = BNF ? 1 : 4;
    const uint32_t sAbase = smem_u32(As), sBbase = smem_u32(Bs);
    constexpr uint32_t stA = BK * LDA * ES, stB = BK * LDB * ES;
    uint32_t gi = 0;  // stage counter (per CTA < 2^32)
    for (int64_t e = it1; e > it0;) {
      int64_t bbase;
      const int bi = item_of(e - 1, bbase);
      const void* const* bptrs = ptrs + (size_t)bi * NPI;
      const int t = tile_of(e - 1 - bbase);
      const int64_t tstart = bbase + kbeg[t];
      const int64_t sb = it0 > tstart ? it0 : tstart;
      const TileRef tr = tiles[t];
      const int M = oM[tr.o], N = oN[tr.o];
      // walk the tile's pairs (reference order) over local k-iterations [sb, e) - tstart
      int64_t kt = sb - tstart;
      const int64_t kend = e - tstart;
      int64_t pbase = 0;
      for (int q = optr[tr.o]; q < optr[tr.o + 1] && kt < kend; ++q) {
        const int i = pairs[2 * q], j = pairs[2 * q + 1];
        const BlockDesc& da = DA[i];
        const BlockDesc& db = DB[j];
        const int nkt = (da.K + BK - 1) / BK;
        if (kt >= pbase + nkt) {
          pbase += nkt;
          continue;
        }
        const T* A = static_cast<const T*>(bptrs[i]);
        const T* B = static_cast<const T*>(bptrs[m.na + j]);
        detail::named_sync(1, NPROD);  // previous pair's table reads are done
        for (int x = p; x < BM + BN; x += NPROD) {
          if (x < BM) rowOffA[x] = (tr.m0 + x < M) ? group_offset(da.free_g, tr.m0 + x) : -1;
          else colOffB[x - BM] = (tr.n0 + x - BM < N) ? group_offset(db.free_g, tr.n0 + x - BM) : -1;
        }
        detail::named_sync(1, NPROD);
        // affine k-tiles (K group of one digit, or an innermost digit that BK divides):
        // offset(k0 + kk) = offset(k0) + kk * stride_inner -- no per-k table, no barrier
        const int nA = da.k_g.n, nB = db.k_g.n;
        const bool aff = (nA <= 1 || da.k_g.dim[nA - 1] % BK == 0) && (nB <= 1 || db.k_g.dim[nB - 1] % BK == 0);
        const int64_t ksA = nA ? da.k_g.stride[nA - 1] : 0, ksB = nB ? db.k_g.stride[nB - 1] : 0;
        const int Kp = da.K;
        int64_t rA[RA], rB[RB];
#pragma unroll
        for (int jj = 0; jj < RA; ++jj) {
          int mm, kk;
          mapA(jj, mm, kk);
          rA[jj] = rowOffA[mm];
        }
#pragma unroll
        for (int jj = 0; jj < RB; ++jj) {
          int nn, kk;
          mapB(jj, nn, kk);
          rB[jj] = colOffB[nn];
        }
        // this thread's gathers for the whole pair: 32-bit element offsets from the block base
        // (-1 = padding row/col) and shared-memory byte offsets within a stage; per k-tile only
        // the k offset moves
        int32_t oA[EA], oB[EB];
        uint32_t dA[EA], dB[EB];
#pragma unroll
        for (int x = 0; x < EA; ++x) {
          int mm, kk;
          mapA(x, mm, kk);
          const int64_t ro = rA[x % RA];
          oA[x] = ro >= 0 ? (int32_t)(ro + (int64_t)kk * ksA) : -1;
          dA[x] = (uint32_t)(kk * LDA + mm) * ES;
        }
#pragma unroll
        for (int x = 0; x < EB; ++x) {
          int nn, kk;
          mapB(x, nn, kk);
          const int64_t co = rB[x % RB];
          oB[x] = co >= 0 ? (int32_t)(co + (int64_t)kk * ksB) : -1;
          dB[x] = (uint32_t)(kk * LDB + nn) * ES;
        }
        const int64_t lend = (kend - pbase) < nkt ? (kend - pbase) : nkt;
        for (int64_t lk = kt - pbase; lk < lend; ++lk, ++gi) {
          const int s = (int)(gi % STAGES);
          const int k0 = (int)lk * BK;
          if (aff) {
            const int32_t koA = nA == 0 ? 0 : (nA == 1 ? k0 * (int32_t)ksA : (int32_t)group_offset(da.k_g, k0));
            const int32_t koB = nB == 0 ? 0 : (nB == 1 ? k0 * (int32_t)ksB : (int32_t)group_offset(db.k_g, k0));
            const int krem = Kp - k0;
            if (gi >= STAGES) detail::mbar_wait(&empty[s], ((gi / STAGES) & 1) ^ 1);
            const uint32_t sa = sAbase + s * stA, sbb = sBbase + s * stB;
            if (sk.exp & 1) {
            } else if (krem >= BK) {  // whole k-tile: validity = padding row/col only
#pragma unroll
              for (int x = 0; x < EA; ++x) {
                if (sk.exp & 4) break;
                const bool v = oA[x] >= 0;
                const T* src = A + (v ? oA[x] + koA : 0);
                TNB_DCHECK(!v || (oA[x] + koA >= 0 && (int64_t)oA[x] + koA < (int64_t)da.F * da.K), "bs A gather");
                if constexpr (CPLX)
                  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa + dA[x]), "l"(src), "r"(v ? 16 : 0));
                else
                  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa + dA[x]), "l"(src), "r"(v ? 8 : 0));
              }
#pragma unroll
              for (int x = 0; x < EB; ++x) {
                if (sk.exp & 8) break;
                const bool v = oB[x] >= 0;
                const T* src = B + (v ? oB[x] + koB : 0);
                TNB_DCHECK(!v || (oB[x] + koB >= 0 && (int64_t)oB[x] + koB < (int64_t)db.F * db.K), "bs B gather");
                if constexpr (CPLX)
                  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sbb + dB[x]), "l"(src), "r"(v ? 16 : 0));
                else
                  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sbb + dB[x]), "l"(src), "r"(v ? 8 : 0));
              }
            } else {  // ragged last k-tile of the pair
#pragma unroll
              for (int x = 0; x < EA; ++x) {
                int mm, kk;
                mapA(x, mm, kk);
                const bool v = oA[x] >= 0 && kk < krem;
                const T* src = A + (v ? oA[x] + koA : 0);
                TNB_DCHECK(!v || (oA[x] + koA >= 0 && (int64_t)oA[x] + koA < (int64_t)da.F * da.K), "bs A gather");
                if constexpr (CPLX)
                  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa + dA[x]), "l"(src), "r"(v ? 16 : 0));
                else
                  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa + dA[x]), "l"(src), "r"(v ? 8 : 0));
              }
#pragma unroll
              for (int x = 0; x < EB; ++x) {
                int nn, kk;
                mapB(x, nn, kk);
                const bool v = oB[x] >= 0 && kk < krem;
                const T* src = B + (v ? oB[x] + koB : 0);
                TNB_DCHECK(!v || (oB[x] + koB >= 0 && (int64_t)oB[x] + koB < (int64_t)db.F * db.K), "bs B gather");
                if constexpr (CPLX)
                  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sbb + dB[x]), "l"(src), "r"(v ? 16 : 0));
                else
                  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sbb + dB[x]), "l"(src), "r"(v ? 8 : 0));
              }
            }
            detail::cp_async_mbar_arrive_noinc(&full[s]);
            continue;
          }
          const int slot = (int)(gi & 1);
          for (int x = p; x < 2 * BK; x += NPROD) {
            const int kk = x % BK, k = k0 + kk;
            const bool v = k < da.K;
            if (x < BK) kOffA[slot * BK + kk] = v ? group_offset(da.k_g, k) : -1;
            else kOffB[slot * BK + kk] = v ? group_offset(db.k_g, k) : -1;
          }
          detail::named_sync(1, NPROD);
          if (gi >= STAGES) detail::mbar_wait(&empty[s], (uint32_t)(((gi / STAGES) & 1) ^ 1));
          const int64_t* ka = kOffA + slot * BK;
          const int64_t* kb = kOffB + slot * BK;
#pragma unroll
          for (int x = 0; x < EA; ++x) {
            int mm, kk;
            mapA(x, mm, kk);
            const int64_t ro = rA[x % RA], ko = ka[kk];
            const bool v = (ro >= 0) && (ko >= 0);
            const T* src = v ? A + ro + ko : A;
            TNB_DCHECK(!v || (ro + ko >= 0 && ro + ko < (int64_t)da.F * da.K), "bs A gather (table)");
            const uint32_t dst = sAbase + s * stA + (uint32_t)(kk * LDA + mm) * ES;
            if constexpr (CPLX)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 16 : 0));
            else
              asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 8 : 0));
          }
#pragma unroll
          for (int x = 0; x < EB; ++x) {
            int nn, kk;
            mapB(x, nn, kk);
            const int64_t co = rB[x % RB], ko = kb[kk];
            const bool v = (co >= 0) && (ko >= 0);
            const T* src = v ? B + co + ko : B;
            TNB_DCHECK(!v || (co + ko >= 0 && co + ko < (int64_t)db.F * db.K), "bs B gather (table)");
            const uint32_t dst = sBbase + s * stB + (uint32_t)(kk * LDB + nn) * ES;
            if constexpr (CPLX)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 16 : 0));
            else
              asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 8 : 0));
          }
          detail::cp_async_mbar_arrive_noinc(&full[s]);
        }
        kt = pbase + lend;
        pbase += nkt;
      }
      e = sb;
    }
    cp_async_wait<0>();
    return;
  }

  // ================================================================== math warps
  typename Core::Acc acc;
  // tiles whose output block has no pair (or whose rank owns them but K is empty) are zeros
  Base::zero(acc);
  for (int bt = c; bt < m.ntiles * m.nbatch; bt += gridDim.x) {
    const int bi = bt / m.ntiles, t = bt - bi * m.ntiles;
    if (kbeg[t + 1] != kbeg[t]) continue;
    const TileRef tr = tiles[t];
    if (m.mask && !m.mask[tr.panel]) continue;
    const int M = oM[tr.o], N = oN[tr.o];
    Base::store(static_cast<T*>(const_cast<void*>(ptrs[(size_t)bi * NPI + m.na + m.nb + tr.o])), N, tr.m0, tr.n0, M, N,
                acc);
  }
  uint32_t gi = 0;
  long long* tr_ = (sk.trace && tid == 0) ? sk.trace + (size_t)c * kTraceW : nullptr;
  int nseg = 0;
  if (tr_) {
    tr_[0] = gtimer();
    tr_[kTraceW - 1] = t_entry;
  }
  for (int64_t e = it1; e > it0;) {
    int64_t bbase;
    const int bi = item_of(e - 1, bbase);
    const int t = tile_of(e - 1 - bbase);
    const int64_t tstart = bbase + kbeg[t], tend = bbase + kbeg[t + 1];
    const int64_t sb = it0 > tstart ? it0 : tstart;
    Base::zero(acc);
    {
      // fragments of this warp's 16x16 tile that lie inside the output block
      const TileRef tr = tiles[t];
      const int warp = tid >> 5;
      int wm, wn;
      Base::warp_mn(warp, wm, wn);
      const int r0 = tr.m0 + wm * Core::WTM, c0 = tr.n0 + wn * Core::WTN;
      const int mfa = (oM[tr.o] - r0 + 7) >> 3, nfa = (oN[tr.o] - c0 + 7) >> 3;
      Core::consume(As, Bs, full, empty, gi, (int)(e - sb), acc, (sk.exp & 2) ? 0 : mfa, (sk.exp & 2) ? 0 : nfa);
    }
    if (tr_ && nseg < 14) tr_[4 + 4 * nseg] = gtimer();
    if (e < tend) {
      Core::publish(sk.ws, sk.flags, c, acc);
    } else {
      if (sb > tstart) Core::absorb(sk.ws, sk.flags, detail::sk_cta_of(total, G, tstart), c, acc, true);
      const TileRef tr = tiles[t];
      const int M = oM[tr.o], N = oN[tr.o];
      Base::store(static_cast<T*>(const_cast<void*>(ptrs[(size_t)bi * NPI + m.na + m.nb + tr.o])), N, tr.m0, tr.n0,
                  M, N, acc);
    }
    if (tr_ && nseg < 14) {
      tr_[5 + 4 * nseg] = gtimer();
      tr_[6 + 4 * nseg] = t;
      tr_[7 + 4 * nseg] = e - sb;
    }
    ++nseg;
    e = sb;
  }
  if (tr_) {
    tr_[1] = gtimer();
    tr_[2] = nseg;
    tr_[3] = it1 - it0;
  }
}

// ---- host ---------------------------------------------------------------------
struct Digit {
  int64_t dim, stride;
};

bool fill_group(std::vector<Digit> digs, bool merge, Group& g) {
  memset(&g, 0, sizeof(g));
  std::vector<Digit> out;
  for (auto& x : digs) {
    if (x.dim == 1) continue;
    if (merge && !out.empty() && out.back().stride == x.dim * x.stride) {
      out.back().dim *= x.dim;
      out.back().stride = x.stride;
    } else {
      out.push_back(x);
    }
  }
  if ((int)out.size() > kMaxDig) return false;
  g.n = (int)out.size();
  for (int q = 0; q < g.n; ++q) {
    if (out[q].dim >= (1ll << 31)) return false;
    g.dim[q] = (int32_t)out[q].dim;
    g.div[q] = FastDiv((uint32_t)out[q].dim);
    g.stride[q] = out[q].stride;
  }
  return true;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// A block-sparse contraction plan: everything that depends only on the block
// STRUCTURE (qn tuples, block shapes, perms, contracted axes). Built once per
// structure -- metadata uploaded, pairing table computed by the pairing kernel --
// and cached on the device; every later call with the same structure launches
// just the grouped GEMM with its data pointers as a kernel parameter.
// A structure's build inputs, kept so a batched execute can derive the wide-tile twin plan.
struct PlanInputs {
  int dtype, na, nb, nout, rank_a, rank_b, nc;
  std::vector<int32_t> a_qn, a_perm, b_qn, b_perm, a_axes, b_axes, out_qn;
  std::vector<int64_t> a_shape, b_shape, out_shape;
};

struct Plan {
  unsigned char* dblob = nullptr;
  BsMeta meta;
  int shape = 0;       // BsCfg tile shape (1: 64 x 128 tiles, float64 batches)
  int64_t twin = 0;    // plan id of the shape-1 twin (0: not built)
  std::shared_ptr<PlanInputs> in;  // shape-0, unmasked plans
  int64_t npairs = 0;
  size_t o_optr = 0, o_pairs = 0;
  int dtype = 0;
  bool amf = true, bnf = true;  // operand gather orientation (coalescing only)
  bool captured = false;         // executed under stream capture: a graph points into dblob
};

// One cache per device (plans, workspace, staging ring and events are device objects);
// all caches are guarded by one mutex, g_bs_mu.
struct PlanCache {
  std::unordered_map<std::string, int64_t> index;  // structure key -> slot in plans
  std::vector<Plan> plans;
  uint32_t gen = 1;  // bumped when the cache is flushed: stale plan ids are rejected
  std::vector<unsigned char*> retained;  // dblobs of flushed plans that captured graphs still read
  // pinned staging for large pointer tables: a ring of slots, each reusable once the copy
  // out of it has run (its event), so the host does not wait on the previous call's copy
  static constexpr int kRing = 8;
  void* stage[kRing] = {};
  size_t stage_cap[kRing] = {};
  cudaEvent_t stage_ev[kRing] = {};
  int stage_next = 0;
  // stream-K partials + flags, shared by all plans of this device. Launches are
  // serialised through ws_ev when they come from different streams.
  void* ws = nullptr;
  size_t ws_bytes = 0;
  cudaEvent_t ws_ev = nullptr;
  cudaStream_t ws_stream = nullptr;
};
std::mutex g_bs_mu;
constexpr int kMaxDevices = 64;
PlanCache* g_caches[kMaxDevices] = {};

// The current device's cache (caller holds g_bs_mu).
PlanCache& cur_cache() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
    cudaGetLastError();
    dev = 0;
  }
  if (!g_caches[dev]) g_caches[dev] = new PlanCache();  // process lifetime (device memory)
  return *g_caches[dev];
}

constexpr int kMaxBsCtas = 2048;  // flags region: one int per persistent CTA
constexpr size_t kBsPartialOff = 16384;

template <bool CPLX, int MODE, bool AMF, bool BNF, int NP, int SHAPE>
int launch_bs_one(const BsMeta& meta, const void* const* hp, int nptr, BsSK sk, bool capturing, cudaStream_t st) {
  using Core = typename BsCfg<CPLX, MODE, SHAPE>::Core;
  auto kern = bs_sk_kernel<CPLX, MODE, AMF, BNF, NP, SHAPE>;
  PtrTable<NP> pt;
  for (int x = 0; x < nptr && x < NP; ++x) pt.p[x] = hp[x];
  const size_t smem = al16(Core::kSmem) + (size_t)meta.sched_smem;
  static size_t configured = 0;
  static size_t occ_smem = 0;
  static int occ = 0;
  if (configured < smem) {
    TNB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  if (occ_smem != smem) {  // persistent grid = every CTA slot: all co-resident (stream-K hand-offs)
    TNB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Core::NT, smem));
    occ_smem = smem;
  }
  if (occ < 1) return fail(TNB_ECUDA, "bs_contract: grouped GEMM kernel does not fit on an SM");
  const int G = std::min(sm_count() * occ, kMaxBsCtas);
  // workspace: flags (self-resetting) at offset 0, register partials after kBsPartialOff
  const size_t need = kBsPartialOff + (size_t)G * Core::ACCN * Core::NMATH * 8;
  void* graph_ws = nullptr;
  if (capturing) {
    // the graph owns its workspace (stream-ordered allocation node + flag memset node):
    // a replay never shares flags/partials with eager launches or other graphs, and a
    // later eager call that grows the shared workspace cannot free memory a graph reads
    int rc = capture_device_ws(st, need, &graph_ws);
    if (rc) return rc;
    TNB_CUDA_CHECK(cudaMemsetAsync(graph_ws, 0, kBsPartialOff, st));
    sk.flags = static_cast<int*>(graph_ws);
    sk.ws = reinterpret_cast<double*>(static_cast<char*>(graph_ws) + kBsPartialOff);
  } else {
    release_deferred_host();  // memory of destroyed graphs
    PlanCache& C = cur_cache();
    if (C.ws_bytes < need) {
      if (C.ws) {
        TNB_CUDA_CHECK(cudaDeviceSynchronize());
        cudaFree(C.ws);
        C.ws = nullptr;
        C.ws_bytes = 0;
      }
      TNB_CUDA_CHECK(cudaMalloc(&C.ws, need));
      TNB_CUDA_CHECK(cudaMemset(C.ws, 0, need));
      C.ws_bytes = need;
    }
    sk.flags = static_cast<int*>(C.ws);
    sk.ws = reinterpret_cast<double*>(static_cast<char*>(C.ws) + kBsPartialOff);
  }
  sk.trace = nullptr;
  static const int exp_mode = getenv("TNB_BS_EXP") ? atoi(getenv("TNB_BS_EXP")) : 0;
  sk.exp = exp_mode;
  static const char* trace_path = getenv("TNB_BS_TRACE");
  if (trace_path && !capturing) {
    TNB_CUDA_CHECK(cudaMallocAsync((void**)&sk.trace, (size_t)G * kTraceW * 8, st));
    TNB_CUDA_CHECK(cudaMemsetAsync(sk.trace, 0, (size_t)G * kTraceW * 8, st));
  }
  {
    KTimer kt(TNB_KF_BS_GEMM, st, 0.0);
    TNB_CUDA_CHECK(launch_cooperative(kern, (unsigned)G, (unsigned)Core::NT, smem, st, meta, pt, sk));
  }
  count_launch();
  {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "bs_contract: grouped GEMM launch");
  }
  if (sk.trace) {
    std::vector<long long> h((size_t)G * kTraceW);
    TNB_CUDA_CHECK(cudaMemcpyAsync(h.data(), sk.trace, h.size() * 8, cudaMemcpyDeviceToHost, st));
    TNB_CUDA_CHECK(cudaStreamSynchronize(st));
    cudaFreeAsync(sk.trace, st);
    if (FILE* f = fopen(trace_path, "ab")) {
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
  }
  return TNB_OK;
}

// Caller holds g_cache.mu.
template <bool CPLX, int MODE, int SH>
int launch_bs(const Plan& plan, const BsMeta& meta, const void* const* hp, int nptr, cudaStream_t st) {
  if (meta.ntiles == 0) return TNB_OK;
  const bool capturing = tnb::capturing(st);
  PlanCache& C = cur_cache();
  if (!capturing && C.ws_ev && C.ws_stream != st) TNB_CUDA_CHECK(cudaStreamWaitEvent(st, C.ws_ev, 0));
  BsSK sk;
  int rc;
  const bool small = meta.ptrs || nptr <= kInlinePtrsSmall;
  constexpr int S = kInlinePtrsSmall, L = kInlinePtrs;
  if (plan.amf && plan.bnf)
    rc = small ? launch_bs_one<CPLX, MODE, true, true, S, SH>(meta, hp, nptr, sk, capturing, st)
               : launch_bs_one<CPLX, MODE, true, true, L, SH>(meta, hp, nptr, sk, capturing, st);
  else if (plan.amf)
    rc = small ? launch_bs_one<CPLX, MODE, true, false, S, SH>(meta, hp, nptr, sk, capturing, st)
               : launch_bs_one<CPLX, MODE, true, false, L, SH>(meta, hp, nptr, sk, capturing, st);
  else if (plan.bnf)
    rc = small ? launch_bs_one<CPLX, MODE, false, true, S, SH>(meta, hp, nptr, sk, capturing, st)
               : launch_bs_one<CPLX, MODE, false, true, L, SH>(meta, hp, nptr, sk, capturing, st);
  else
    rc = small ? launch_bs_one<CPLX, MODE, false, false, S, SH>(meta, hp, nptr, sk, capturing, st)
               : launch_bs_one<CPLX, MODE, false, false, L, SH>(meta, hp, nptr, sk, capturing, st);
  if (rc) return rc;
  if (!capturing) {
    if (!C.ws_ev) TNB_CUDA_CHECK(cudaEventCreateWithFlags(&C.ws_ev, cudaEventDisableTiming));
    TNB_CUDA_CHECK(cudaEventRecord(C.ws_ev, st));
    C.ws_stream = st;
  }
  return TNB_OK;
}

template <typename X>
void append(std::string& key, const X* p, size_t n) {
  key.append(reinterpret_cast<const char*>(p), n * sizeof(X));
}

}  // namespace
}  // namespace tnb

namespace tnb {
namespace {

// Caller holds g_cache.mu. Builds (pairing kernel on `st`) or finds the plan of a structure.
int bs_plan_locked(int dtype, int na, int nb, int nout, int rank_a, int rank_b, const int32_t* a_qn,
                   const int64_t* a_shape, const int32_t* a_perm, const int32_t* b_qn, const int64_t* b_shape,
                   const int32_t* b_perm, int nc, const int32_t* a_axes, const int32_t* b_axes,
                   const int32_t* out_qn, const int64_t* out_shape, int64_t npanels, const uint8_t* panel_mask,
                   cudaStream_t st, int64_t* plan_id, int64_t* npairs, int shape = 0) {
  int rc = require_device();
  if (rc) return rc;
  if (dtype != TNB_F64 && dtype != TNB_C128)
    return fail(TNB_EUNSUP, "bs_contract: only float64 and complex128 are supported on the GPU path");
  if (na < 0 || nb < 0 || nout < 1 || rank_a < 1 || rank_b < 1 || rank_a > TNB_MAX_RANK || rank_b > TNB_MAX_RANK ||
      nc < 0 || nc > rank_a || nc > rank_b)
    return fail(TNB_EINVAL, "bs_contract: bad sizes");
  const int ro = rank_a + rank_b - 2 * nc;
  if (ro < 1) return fail(TNB_EINVAL, "bs_contract: scalar output is handled by the host layer");
  // ---- plan lookup (structure only)
  std::string key;
  {
    int32_t hdr[8] = {dtype, na, nb, nout, rank_a, rank_b, nc, shape};
    append(key, hdr, 8);
    append(key, a_qn, (size_t)na * rank_a);
    append(key, a_shape, (size_t)na * rank_a);
    append(key, a_perm, (size_t)rank_a);
    append(key, b_qn, (size_t)nb * rank_b);
    append(key, b_shape, (size_t)nb * rank_b);
    append(key, b_perm, (size_t)rank_b);
    append(key, a_axes, (size_t)nc);
    append(key, b_axes, (size_t)nc);
    append(key, out_qn, (size_t)nout * ro);
    append(key, out_shape, (size_t)nout * ro);
    if (panel_mask && npanels > 0) {
      key.push_back('M');
      append(key, panel_mask, (size_t)npanels);
    }
  }
  PlanCache& g_cache = cur_cache();
  auto hit = g_cache.index.find(key);
  if (hit == g_cache.index.end()) {
    if (g_cache.plans.size() >= 256) {
      TNB_CUDA_CHECK(cudaDeviceSynchronize());
      // plans a captured graph launched stay allocated: the graph's kernel nodes hold
      // pointers into their dblob for as long as the graph lives
      for (auto& pl : g_cache.plans) {
        if (pl.captured) g_cache.retained.push_back(pl.dblob);
        else cudaFree(pl.dblob);
      }
      g_cache.plans.clear();
      g_cache.index.clear();
      ++g_cache.gen;
    }
    Plan plan;
    plan.dtype = dtype;
    plan.shape = shape;
    if (shape == 0 && !(panel_mask && npanels > 0)) {
      auto in = std::make_shared<PlanInputs>();
      *in = {dtype, na, nb, nout, rank_a, rank_b, nc, {}, {}, {}, {}, {}, {}, {}, {}, {}, {}};
      in->a_qn.assign(a_qn, a_qn + (size_t)na * rank_a);
      in->a_shape.assign(a_shape, a_shape + (size_t)na * rank_a);
      in->a_perm.assign(a_perm, a_perm + rank_a);
      in->b_qn.assign(b_qn, b_qn + (size_t)nb * rank_b);
      in->b_shape.assign(b_shape, b_shape + (size_t)nb * rank_b);
      in->b_perm.assign(b_perm, b_perm + rank_b);
      in->a_axes.assign(a_axes, a_axes + nc);
      in->b_axes.assign(b_axes, b_axes + nc);
      in->out_qn.assign(out_qn, out_qn + (size_t)nout * ro);
      in->out_shape.assign(out_shape, out_shape + (size_t)nout * ro);
      plan.in = in;
    }
    BsMeta& meta = plan.meta;
    memset(&meta, 0, sizeof(meta));
    meta.nbatch = 1;
    meta.na = na;
    meta.nb = nb;
    meta.nout = nout;
    meta.ra = rank_a;
    meta.rb = rank_b;
    meta.ro = ro;
    meta.nc = nc;
    std::vector<int> acon(rank_a, 0), bcon(rank_b, 0);
    for (int c = 0; c < nc; ++c) {
      if (a_axes[c] < 0 || a_axes[c] >= rank_a || b_axes[c] < 0 || b_axes[c] >= rank_b || acon[a_axes[c]] ||
          bcon[b_axes[c]])
        return fail(TNB_EINVAL, "bs_contract: bad contracted axes");
      acon[a_axes[c]] = bcon[b_axes[c]] = 1;
      meta.a_axes[c] = a_axes[c];
      meta.b_axes[c] = b_axes[c];
    }
    for (int k = 0; k < rank_a; ++k)
      if (!acon[k]) meta.a_free[meta.nfa++] = k;
    for (int k = 0; k < rank_b; ++k)
      if (!bcon[k]) meta.b_free[meta.nfb++] = k;
    // per-block address groups (host integer work, O(blocks * rank), once per plan)
    auto block_desc = [&](int rank, const int64_t* shp, const int32_t* perm, const int* con, const int32_t* axes,
                          BlockDesc& bd) -> bool {
      std::vector<int64_t> ss(rank, 1);
      for (int a = rank - 2; a >= 0; --a) ss[a] = ss[a + 1] * shp[a + 1];
      std::vector<Digit> fr, kk;
      int64_t F = 1, K = 1;
      for (int k = 0; k < rank; ++k) {
        int p = perm[k];
        if (!con[k]) {
          fr.push_back({shp[p], ss[p]});
          F *= shp[p];
        }
      }
      for (int c = 0; c < nc; ++c) {
        int p = perm[axes[c]];
        kk.push_back({shp[p], ss[p]});
        K *= shp[p];
      }
      if (F * K >= (1ll << 31)) return false;  // 32-bit element offsets inside a block
      bd.F = (int32_t)F;
      bd.K = (int32_t)K;
      return fill_group(fr, true, bd.free_g) && fill_group(kk, false, bd.k_g);
    };
    std::vector<BlockDesc> da(na), db(nb);
    for (int i = 0; i < na; ++i)
      if (!block_desc(rank_a, a_shape + (int64_t)i * rank_a, a_perm, acon.data(), a_axes, da[i]))
        return fail(TNB_EUNSUP, "bs_contract: block index group too large");
    for (int j = 0; j < nb; ++j)
      if (!block_desc(rank_b, b_shape + (int64_t)j * rank_b, b_perm, bcon.data(), b_axes, db[j]))
        return fail(TNB_EUNSUP, "bs_contract: block index group too large");
    // gather orientation (the dense rule of gemm.cu per block), majority by block work
    {
      double wa[2] = {0, 0}, wb[2] = {0, 0};
      for (int i = 0; i < na; ++i) {
        const Group& f = da[i].free_g;
        const Group& k = da[i].k_g;
        const bool fast = (f.n > 0 && f.stride[f.n - 1] == 1 && f.dim[f.n - 1] >= 4) ||
                          !(k.n > 0 && k.stride[k.n - 1] == 1);
        wa[fast ? 1 : 0] += (double)da[i].F * da[i].K;
      }
      for (int j = 0; j < nb; ++j) {
        const Group& f = db[j].free_g;
        const Group& k = db[j].k_g;
        const bool fast = (f.n > 0 && f.stride[f.n - 1] == 1 && f.dim[f.n - 1] >= 4) ||
                          !(k.n > 0 && k.stride[k.n - 1] == 1);
        wb[fast ? 1 : 0] += (double)db[j].F * db[j].K;
      }
      plan.amf = wa[1] >= wa[0];
      plan.bnf = wb[1] >= wb[0];
    }
    const int BM = BsCfg<false, 0>::BM, BN = shape ? BsCfg<false, 0, 1>::BN : BsCfg<false, 0>::BN;
    static_assert(BsCfg<false, 0, 1>::BM == BsCfg<false, 0>::BM, "panels are BM-row based in every shape");
    meta.bk = (dtype == TNB_C128) ? BsCfg<true, 0>::BK : BsCfg<false, 0>::BK;
    std::vector<int32_t> oM(nout), oN(nout);
    std::vector<TileRef> tiles;
    int32_t panel = 0;
    static_assert(TNB_BS_PANEL_ROWS % 64 == 0, "panels must hold whole 64-row tiles");
    for (int o = 0; o < nout; ++o) {
      int64_t Mo = 1, No = 1;
      for (int f = 0; f < meta.nfa; ++f) Mo *= out_shape[(int64_t)o * ro + f];
      for (int f = meta.nfa; f < ro; ++f) No *= out_shape[(int64_t)o * ro + f];
      if (Mo >= (1ll << 31) || No >= (1ll << 31)) return fail(TNB_EUNSUP, "bs_contract: output block too large");
      oM[o] = (int32_t)Mo;
      oN[o] = (int32_t)No;
      for (int64_t m0 = 0; m0 < Mo; m0 += BM) {
        const int32_t pnl = panel + (int32_t)(m0 / TNB_BS_PANEL_ROWS);
        for (int64_t n0 = 0; n0 < No; n0 += BN) tiles.push_back({o, (int32_t)m0, (int32_t)n0, pnl});
      }
      panel += (int32_t)((Mo + TNB_BS_PANEL_ROWS - 1) / TNB_BS_PANEL_ROWS);
    }
    if (panel_mask && npanels != panel) return fail(TNB_EINVAL, "bs_contract: panel mask has the wrong length");
    if (tiles.size() >= (1u << 31)) return fail(TNB_EUNSUP, "bs_contract: too many tiles");
    meta.ntiles = (int)tiles.size();
    // exact pair count from a key histogram (O(na + nb)) sizes the device pair table;
    // which pairs, their order and their output blocks are computed on the device
    int64_t exact_pairs = 0;
    {
      std::map<std::vector<int32_t>, int64_t> hist;
      std::vector<int32_t> kv(nc);
      for (int j = 0; j < nb; ++j) {
        for (int c = 0; c < nc; ++c) kv[c] = b_qn[(int64_t)j * rank_b + b_axes[c]];
        hist[kv]++;
      }
      for (int i = 0; i < na; ++i) {
        for (int c = 0; c < nc; ++c) kv[c] = a_qn[(int64_t)i * rank_a + a_axes[c]];
        auto it = hist.find(kv);
        if (it != hist.end()) exact_pairs += it->second;
      }
    }
    meta.max_pairs = std::max<int64_t>(exact_pairs, 1);
    {
      static_assert(sizeof(BlockDesc) % 16 == 0, "block descriptors are staged as uint4");
      const size_t sb = sched_bytes((int)tiles.size(), nout, meta.max_pairs);
      const size_t db_bytes = sizeof(BlockDesc) * (size_t)(na + nb);
      meta.sched_smem = sb <= 32 * 1024 ? (int)sb : 0;
      meta.desc_smem = (meta.sched_smem && db_bytes <= 48 * 1024) ? 1 : 0;
      if (meta.desc_smem) meta.sched_smem += (int)db_bytes;
    }
    size_t off = 0;
    auto take = [&](size_t bytes) {
      size_t o = align_up(off, 16);
      off = o + bytes;
      return o;
    };
    // the GEMM's shared-memory image first (see BsMeta::img; same order and padding as
    // sched_bytes), then the pairing kernel's inputs and scratch
    const size_t o_kbeg = take(al16((size_t)(tiles.size() + 1) * 4)), o_stiles = take(sizeof(TileRef) * tiles.size()),
                 o_optr = take(al16((size_t)(nout + 1) * 4)), o_pairs = take(al16((size_t)meta.max_pairs * 8)),
                 o_oM = take(al16((size_t)nout * 4)), o_oN = take(al16((size_t)nout * 4)),
                 o_da = take(sizeof(BlockDesc) * na), o_db = take(sizeof(BlockDesc) * nb);
    const size_t o_aqn = take((size_t)na * rank_a * 4), o_bqn = take((size_t)nb * rank_b * 4),
                 o_oqn = take((size_t)nout * ro * 4), o_tiles = take(sizeof(TileRef) * tiles.size()),
                 o_mask = take(panel_mask ? (size_t)npanels : 0);
    const size_t upload = off;
    const size_t o_err = take(16 + 16 * 8), o_tcnt = take((size_t)tiles.size() * 4);
    // whole-tile LPT schedule for single contractions on a one-CTA-per-SM persistent grid
    static const int lpt_slack = getenv("TNB_BS_LPT_SLACK") ? atoi(getenv("TNB_BS_LPT_SLACK")) : kLptSlackDefault;
    meta.sched_G = lpt_slack >= 0 ? std::min(sm_count(), kLptMaxG) : 0;
    meta.lpt_slack = lpt_slack;
    const size_t o_ctab = take((size_t)(meta.sched_G + 2) * 4);
    const size_t total = off;
    if (o_oM - o_kbeg != sched_bytes((int)tiles.size(), nout, meta.max_pairs) - 2 * al16((size_t)nout * 4) ||
        o_da != o_kbeg + sched_bytes((int)tiles.size(), nout, meta.max_pairs))
      return fail(TNB_EUNSUP, "bs_contract: schedule image layout mismatch");
    std::vector<unsigned char> h(upload);
    memcpy(h.data() + o_aqn, a_qn, (size_t)na * rank_a * 4);
    memcpy(h.data() + o_bqn, b_qn, (size_t)nb * rank_b * 4);
    memcpy(h.data() + o_oqn, out_qn, (size_t)nout * ro * 4);
    memcpy(h.data() + o_oM, oM.data(), (size_t)nout * 4);
    memcpy(h.data() + o_oN, oN.data(), (size_t)nout * 4);
    memcpy(h.data() + o_da, da.data(), sizeof(BlockDesc) * na);
    memcpy(h.data() + o_db, db.data(), sizeof(BlockDesc) * nb);
    memcpy(h.data() + o_tiles, tiles.data(), sizeof(TileRef) * tiles.size());
    if (panel_mask) memcpy(h.data() + o_mask, panel_mask, (size_t)npanels);
    TNB_CUDA_CHECK(cudaMalloc((void**)&plan.dblob, total));
    unsigned char* dblob = plan.dblob;
    TNB_CUDA_CHECK(cudaMemcpyAsync(dblob, h.data(), upload, cudaMemcpyHostToDevice, st));  // staged, then returns
    TNB_CUDA_CHECK(cudaMemsetAsync(dblob + o_err, 0, 16 + 16 * 8, st));
    meta.a_qn = reinterpret_cast<const int32_t*>(dblob + o_aqn);
    meta.b_qn = reinterpret_cast<const int32_t*>(dblob + o_bqn);
    meta.out_qn = reinterpret_cast<const int32_t*>(dblob + o_oqn);
    meta.out_M = reinterpret_cast<const int32_t*>(dblob + o_oM);
    meta.out_N = reinterpret_cast<const int32_t*>(dblob + o_oN);
    meta.da = reinterpret_cast<const BlockDesc*>(dblob + o_da);
    meta.db = reinterpret_cast<const BlockDesc*>(dblob + o_db);
    meta.tiles = reinterpret_cast<const TileRef*>(dblob + o_tiles);
    meta.out_ptr = reinterpret_cast<int32_t*>(dblob + o_optr);
    meta.err = reinterpret_cast<int32_t*>(dblob + o_err);
    meta.pairs = reinterpret_cast<int32_t*>(dblob + o_pairs);
    meta.mask = panel_mask ? reinterpret_cast<const uint8_t*>(dblob + o_mask) : nullptr;
    meta.tile_kbeg = reinterpret_cast<int32_t*>(dblob + o_kbeg);
    meta.tile_cnt = reinterpret_cast<int32_t*>(dblob + o_tcnt);
    meta.stiles = reinterpret_cast<TileRef*>(dblob + o_stiles);
    meta.img = reinterpret_cast<const uint4*>(dblob + o_kbeg);
    meta.cta_beg = reinterpret_cast<int32_t*>(dblob + o_ctab);
    meta.ptrs = nullptr;
    meta.qn_smem = 1;
    size_t pair_smem = pair_smem_bytes(meta);
    if (pair_smem > 200 * 1024) {  // very large structures: tables stay in global memory
      meta.qn_smem = 0;
      pair_smem = 0;
    }
    if (pair_smem > 48 * 1024)
      TNB_CUDA_CHECK(cudaFuncSetAttribute(bs_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pair_smem));
    {
      KTimer kt(TNB_KF_BS_PAIR, st, 0.0);
      bs_pair_kernel<<<1, 1024, pair_smem, st>>>(meta);
    }
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      cudaFree(dblob);
      return cuda_fail(e, "bs_contract: pairing kernel launch");
    }
    if (getenv("TNB_BS_TRACE")) {
      long long st16[16];
      TNB_CUDA_CHECK(cudaMemcpyAsync(st16, dblob + o_err + 16, sizeof(st16), cudaMemcpyDeviceToHost, st));
      TNB_CUDA_CHECK(cudaStreamSynchronize(st));
      fprintf(stderr, "[tnb pair phases us]");
      for (int q = 1; q < 16 && st16[q] > 0; ++q) fprintf(stderr, " %.1f", (st16[q] - st16[0]) / 1e3);
      fprintf(stderr, "\n");
    }
    plan.npairs = exact_pairs;
    plan.o_optr = o_optr;
    plan.o_pairs = o_pairs;
    g_cache.plans.push_back(plan);
    hit = g_cache.index.emplace(key, (int64_t)g_cache.plans.size() - 1).first;
  }
  *plan_id = ((int64_t)g_cache.gen << 32) | hit->second;
  if (npairs) *npairs = g_cache.plans[hit->second].npairs;
  return TNB_OK;
}

Plan* plan_of(int64_t id) {
  PlanCache& g_cache = cur_cache();
  const uint32_t gen = (uint32_t)((uint64_t)id >> 32);
  const int64_t slot = id & 0xffffffffll;
  if (gen != g_cache.gen || slot < 0 || slot >= (int64_t)g_cache.plans.size()) return nullptr;
  return &g_cache.plans[slot];
}

// Caller holds g_cache.mu. One grouped GEMM launch with this call's data pointers.
int bs_execute_locked(Plan& plan, const void* const* a_ptrs, const void* const* b_ptrs, void* const* out_ptrs,
                      cudaStream_t st, int64_t nbatch = 1) {
  BsMeta meta = plan.meta;
  const int na = meta.na, nb = meta.nb, nout = meta.nout;
  int rc = TNB_OK;
  if (nbatch < 1) return fail(TNB_EINVAL, "bs_execute: nbatch must be >= 1");
  if ((int64_t)meta.ntiles * nbatch >= (1ll << 31) ||
      (int64_t)(meta.ntiles + 1) * nbatch * 1024 >= (1ll << 40))
    return fail(TNB_EUNSUP, "bs_execute: batch too large");
  meta.nbatch = (int)nbatch;
  // ---- per-call data pointers ([nbatch][na + nb + nout])
  const int nptr1 = na + nb + nout;
  const int64_t nptr = (int64_t)nptr1 * nbatch;
  std::vector<const void*> hv;
  if (nptr <= kInlinePtrs) {
    hv.resize(nptr);
    for (int64_t q = 0; q < nbatch; ++q) {
      const void** h = hv.data() + q * nptr1;
      for (int i = 0; i < na; ++i) h[i] = a_ptrs[q * na + i];
      for (int j = 0; j < nb; ++j) h[na + j] = b_ptrs[q * nb + j];
      for (int o = 0; o < nout; ++o) h[na + nb + o] = out_ptrs[q * nout + o];
    }
    meta.ptrs = nullptr;
  } else {
    const size_t bytes = (size_t)nptr * sizeof(void*);
    const bool capturing = tnb::capturing(st);
    PlanCache& g_cache = cur_cache();
    void* host = nullptr;
    int slot = -1;
    if (capturing) {
      // a captured copy re-reads its source at every replay: its own pinned buffer, owned
      // (and eventually freed) by the graph
      rc = capture_pinned(st, bytes, &host);
      if (rc) return rc;
    } else {
      release_deferred_host();
      slot = g_cache.stage_next;
      g_cache.stage_next = (slot + 1) % PlanCache::kRing;
      if (g_cache.stage_ev[slot]) TNB_CUDA_CHECK(cudaEventSynchronize(g_cache.stage_ev[slot]));
      if (g_cache.stage_cap[slot] < bytes) {
        if (g_cache.stage[slot]) cudaFreeHost(g_cache.stage[slot]);
        g_cache.stage_cap[slot] = std::max(bytes, (size_t)1 << 16);
        TNB_CUDA_CHECK(cudaMallocHost(&g_cache.stage[slot], g_cache.stage_cap[slot]));
      }
      if (!g_cache.stage_ev[slot])
        TNB_CUDA_CHECK(cudaEventCreateWithFlags(&g_cache.stage_ev[slot], cudaEventDisableTiming));
      host = g_cache.stage[slot];
    }
    const void** hp = static_cast<const void**>(host);
    for (int64_t q = 0; q < nbatch; ++q) {
      const void** h = hp + q * nptr1;
      for (int i = 0; i < na; ++i) h[i] = a_ptrs[q * na + i];
      for (int j = 0; j < nb; ++j) h[na + j] = b_ptrs[q * nb + j];
      for (int o = 0; o < nout; ++o) h[na + nb + o] = out_ptrs[q * nout + o];
    }
    void* dptr = nullptr;
    TNB_CUDA_CHECK(cudaMallocAsync(&dptr, bytes, st));
    TNB_CUDA_CHECK(cudaMemcpyAsync(dptr, hp, bytes, cudaMemcpyHostToDevice, st));
    if (slot >= 0) TNB_CUDA_CHECK(cudaEventRecord(g_cache.stage_ev[slot], st));
    meta.ptrs = static_cast<const void* const*>(dptr);
  }
  if (tnb::capturing(st)) plan.captured = true;
  const void* const* hp = meta.ptrs ? nullptr : hv.data();
  const int nin = meta.ptrs ? 0 : (int)nptr;
  if (plan.dtype == TNB_F64) rc = plan.shape ? launch_bs<false, 0, 1>(plan, meta, hp, nin, st)
                                             : launch_bs<false, 0, 0>(plan, meta, hp, nin, st);
  else rc = launch_bs<true, 0, 0>(plan, meta, hp, nin, st);
  if (meta.ptrs) cudaFreeAsync(const_cast<void*>(static_cast<const void*>(meta.ptrs)), st);
  if (rc != TNB_OK) return rc;
  return TNB_OK;
}

// Caller holds g_cache.mu. (i, j, out_idx) triples in reference order (synchronises).
int bs_pairs_locked(Plan& plan, int64_t max_pairs, int32_t* pairs_out, int64_t* npairs, cudaStream_t st) {
  const int nout = plan.meta.nout;
  if (npairs) *npairs = plan.npairs;
  {
    if (max_pairs < plan.npairs) return fail(TNB_EINVAL, "bs_contract: pairs_out too small");
    // bookkeeping readback: CSR grouped by output block -> reference order (i asc, j asc)
    std::vector<int32_t> optr(nout + 1);
    int32_t err = 0;
    TNB_CUDA_CHECK(cudaMemcpyAsync(optr.data(), plan.dblob + plan.o_optr, (size_t)(nout + 1) * 4,
                                   cudaMemcpyDeviceToHost, st));
    TNB_CUDA_CHECK(cudaMemcpyAsync(&err, plan.meta.err, 4, cudaMemcpyDeviceToHost, st));
    TNB_CUDA_CHECK(cudaStreamSynchronize(st));
    if (err) return fail(TNB_EINVAL, "bs_contract: device pairing overflow");
    int64_t np = optr[nout];
    std::vector<int32_t> pl((size_t)np * 2);
    if (np) TNB_CUDA_CHECK(cudaMemcpy(pl.data(), plan.dblob + plan.o_pairs, (size_t)np * 8, cudaMemcpyDeviceToHost));
    std::vector<std::array<int32_t, 3>> trip;
    trip.reserve(np);
    for (int o = 0; o < nout; ++o)
      for (int p = optr[o]; p < optr[o + 1]; ++p) trip.push_back({pl[2 * p], pl[2 * p + 1], o});
    std::sort(trip.begin(), trip.end());
    for (int64_t q = 0; q < np; ++q) {
      pairs_out[3 * q] = trip[q][0];
      pairs_out[3 * q + 1] = trip[q][1];
      pairs_out[3 * q + 2] = trip[q][2];
    }
    if (npairs) *npairs = np;
  }
  return TNB_OK;
}


}  // namespace
}  // namespace tnb

extern "C" int tnb_bs_plan(int dtype, int na, int nb, int nout, int rank_a, int rank_b, const int32_t* a_qn,
                           const int64_t* a_shape, const int32_t* a_perm, const int32_t* b_qn,
                           const int64_t* b_shape, const int32_t* b_perm, int nc, const int32_t* a_axes,
                           const int32_t* b_axes, const int32_t* out_qn, const int64_t* out_shape, int64_t npanels,
                           const uint8_t* panel_mask, int64_t* plan_id, int64_t* npairs, void* stream) {
  using namespace tnb;
  int rc = require_device();
  if (rc) return rc;
  if (!plan_id) return fail(TNB_EINVAL, "bs_plan: plan_id is NULL");
  std::lock_guard<std::mutex> lock(g_bs_mu);
  return bs_plan_locked(dtype, na, nb, nout, rank_a, rank_b, a_qn, a_shape, a_perm, b_qn, b_shape, b_perm, nc, a_axes,
                        b_axes, out_qn, out_shape, npanels, panel_mask, (cudaStream_t)stream, plan_id, npairs);
}

extern "C" int tnb_bs_execute(int64_t plan_id, const void* const* a_ptrs, const void* const* b_ptrs,
                              void* const* out_ptrs, void* stream) {
  using namespace tnb;
  int rc = require_device();
  if (rc) return rc;
  std::lock_guard<std::mutex> lock(g_bs_mu);
  Plan* plan = plan_of(plan_id);
  if (!plan) return fail(TNB_EINVAL, "bs_execute: stale or unknown plan id (plan cache was flushed)");
  if ((plan->meta.na && !a_ptrs) || (plan->meta.nb && !b_ptrs) || !out_ptrs)
    return fail(TNB_EINVAL, "bs_execute: NULL pointer table");
  return bs_execute_locked(*plan, a_ptrs, b_ptrs, out_ptrs, (cudaStream_t)stream);
}

extern "C" int tnb_bs_execute_batched(int64_t plan_id, int64_t nbatch, const void* const* a_ptrs,
                                      const void* const* b_ptrs, void* const* out_ptrs, void* stream) {
  using namespace tnb;
  int rc = require_device();
  if (rc) return rc;
  std::lock_guard<std::mutex> lock(g_bs_mu);
  Plan* plan = plan_of(plan_id);
  if (!plan) return fail(TNB_EINVAL, "bs_execute_batched: stale or unknown plan id (plan cache was flushed)");
  if ((plan->meta.na && !a_ptrs) || (plan->meta.nb && !b_ptrs) || !out_ptrs)
    return fail(TNB_EINVAL, "bs_execute_batched: NULL pointer table");
  if (plan->meta.mask && nbatch != 1)
    return fail(TNB_EUNSUP, "bs_execute_batched: panel-masked plans run one contraction per launch");
  // float64 batches of >= kWideBatch contractions run on the structure's 64 x 128-tile twin
  // (built once from the stored inputs; same pairs and per-tile pair order)
  constexpr int64_t kWideBatch = 4;
  static const bool no_wide = getenv("TNB_BS_NO_WIDE") != nullptr;  // dev A/B switch
  if (!no_wide && nbatch >= kWideBatch && plan->dtype == TNB_F64 && plan->shape == 0 && plan->in) {
    Plan* twin = plan->twin ? plan_of(plan->twin) : nullptr;
    // (not built under stream capture: its pairing kernel would only run when the graph does,
    // leaving the twin's schedule unwritten for eager calls; the parent plan serves instead)
    if (!twin && !tnb::capturing((cudaStream_t)stream)) {
      std::shared_ptr<PlanInputs> in = plan->in;  // (plan may move: the cache vector grows)
      int64_t tid = 0;
      rc = bs_plan_locked(in->dtype, in->na, in->nb, in->nout, in->rank_a, in->rank_b, in->a_qn.data(),
                          in->a_shape.data(), in->a_perm.data(), in->b_qn.data(), in->b_shape.data(),
                          in->b_perm.data(), in->nc, in->a_axes.data(), in->b_axes.data(), in->out_qn.data(),
                          in->out_shape.data(), 0, nullptr, (cudaStream_t)stream, &tid, nullptr, 1);
      if (rc) return rc;
      plan = plan_of(plan_id);
      if (!plan) return fail(TNB_EINVAL, "bs_execute_batched: stale or unknown plan id (plan cache was flushed)");
      plan->twin = tid;
      twin = plan_of(tid);
    }
    if (twin) return bs_execute_locked(*twin, a_ptrs, b_ptrs, out_ptrs, (cudaStream_t)stream, nbatch);
  }
  return bs_execute_locked(*plan, a_ptrs, b_ptrs, out_ptrs, (cudaStream_t)stream, nbatch);
}

extern "C" int tnb_bs_plan_pairs(int64_t plan_id, int64_t max_pairs, int32_t* pairs_out, int64_t* npairs,
                                 void* stream) {
  using namespace tnb;
  int rc = require_device();
  if (rc) return rc;
  if (!pairs_out) return fail(TNB_EINVAL, "bs_plan_pairs: pairs_out is NULL");
  std::lock_guard<std::mutex> lock(g_bs_mu);
  Plan* plan = plan_of(plan_id);
  if (!plan) return fail(TNB_EINVAL, "bs_plan_pairs: stale or unknown plan id");
  return bs_pairs_locked(*plan, max_pairs, pairs_out, npairs, (cudaStream_t)stream);
}

extern "C" int tnb_bs_contract_masked(int dtype, int na, int nb, int nout, int rank_a, int rank_b,
                                      const int32_t* a_qn, const int64_t* a_shape, const int32_t* a_perm,
                                      const int32_t* b_qn, const int64_t* b_shape, const int32_t* b_perm, int nc,
                                      const int32_t* a_axes, const int32_t* b_axes, const int32_t* out_qn,
                                      const int64_t* out_shape, const void* const* a_ptrs,
                                      const void* const* b_ptrs, void* const* out_ptrs, int64_t npanels,
                                      const uint8_t* panel_mask, int64_t max_pairs, int32_t* pairs_out,
                                      int64_t* npairs, void* stream) {
  using namespace tnb;
  int rc = require_device();
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  std::lock_guard<std::mutex> lock(g_bs_mu);
  int64_t id = 0;
  rc = bs_plan_locked(dtype, na, nb, nout, rank_a, rank_b, a_qn, a_shape, a_perm, b_qn, b_shape, b_perm, nc, a_axes,
                      b_axes, out_qn, out_shape, npanels, panel_mask, st, &id, npairs);
  if (rc) return rc;
  Plan* plan = plan_of(id);
  rc = bs_execute_locked(*plan, a_ptrs, b_ptrs, out_ptrs, st);
  if (rc || !pairs_out) return rc;
  return bs_pairs_locked(*plan, max_pairs, pairs_out, npairs, st);
}

extern "C" int tnb_bs_contract(int dtype, int na, int nb, int nout, int rank_a, int rank_b, const int32_t* a_qn,
                               const int64_t* a_shape, const int32_t* a_perm, const int32_t* b_qn,
                               const int64_t* b_shape, const int32_t* b_perm, int nc, const int32_t* a_axes,
                               const int32_t* b_axes, const int32_t* out_qn, const int64_t* out_shape,
                               const void* const* a_ptrs, const void* const* b_ptrs, void* const* out_ptrs,
                               int64_t max_pairs, int32_t* pairs_out, int64_t* npairs, void* stream) {
  return tnb_bs_contract_masked(dtype, na, nb, nout, rank_a, rank_b, a_qn, a_shape, a_perm, b_qn, b_shape, b_perm, nc,
                                a_axes, b_axes, out_qn, out_shape, a_ptrs, b_ptrs, out_ptrs, 0, nullptr, max_pairs,
                                pairs_out, npairs, stream);
}

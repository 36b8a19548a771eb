// a7: materialise a lazy permute -- the B200 replacement for
//     np.ascontiguousarray(self.view())   (pkg/src/tnkit/storage.py:122, :126, :143)
//
// Design:
//   * host: drop unit axes, merge logical axes that stay adjacent in storage,
//     then choose a tile = (input-fast axis group G_in) x (output-fast group
//     G_out): G_in is a storage suffix long enough that each warp READS >=256 B
//     contiguous runs, G_out an output suffix long enough that each warp
//     WRITES >=256 B contiguous runs. All other axes are "batch" axes.
//   * device: persistent CTAs loop over tiles. Each tile is read in storage
//     order (coalesced 8/16-byte lanes) into a padded shared-memory tile, then
//     written in output order (coalesced). Per-tile index math is O(rank);
//     per-element math is one multiply-high division and 1-3 shared-memory
//     table lookups (tables built once per CTA).
//   * bit-exact: pure data movement of elem_size-byte words.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace tnb {
namespace {

constexpr int kMaxR = TNB_MAX_RANK;
constexpr int kThreads = 256;  // generic tiled kernel: 4+ CTAs (tiles) in flight per SM

template <int ES>
struct Word;
template <>
struct Word<1> { using T = uint8_t; };
template <>
struct Word<2> { using T = uint16_t; };
template <>
struct Word<4> { using T = uint32_t; };
template <>
struct Word<8> { using T = unsigned long long; };
template <>
struct Word<16> { using T = uint4; };

struct PermDesc {
  int r;                     // merged rank
  int nb;                    // number of batch axes (nt > 1), output order outer->inner
  int nuin, nuout;           // |U| in input order / output order (same set)
  int gin, gout;             // innermost counts forming G_in (of uin) / G_out (of uout)
  int N_t, N_in, N_out, rowp;  // tile elements, input run, output run, padded row length
  int n_hi_in, n_hi_out;     // N_t / N_in, N_t / N_out
  int a_in, a_out;           // partial (split) axes or -1
  int64_t ntiles;
  int64_t dim[kMaxR];
  int64_t istride[kMaxR];    // storage stride of storage axis a
  int64_t ostride[kMaxR];    // output stride of storage axis a
  int32_t ext[kMaxR];        // tile extent along storage axis a (1 if not in U)
  int32_t bax[kMaxR];        // batch axes
  uint32_t bnt[kMaxR];       // tiles along batch axis
  FastDiv bdiv[kMaxR];
  int32_t uin[kMaxR];        // U axes in storage order (outer->inner)
  int32_t uout[kMaxR];       // U axes in output order (outer->inner)
  int32_t pts[kMaxR];        // padded smem tile stride of storage axis a
  int32_t tsi[kMaxR];        // unpadded input-order tile stride (boundary path)
  int32_t tso[kMaxR];        // output-order tile stride (boundary path)
  FastDiv div_in, div_out;   // by N_in, N_out
  FastDiv cin_div, cout_div; // by ceil(N_in / 32), ceil(N_out / 32): 32-element items per run
  FastDiv tsi_div[kMaxR], tso_div[kMaxR], ext_div[kMaxR];
};

// Shared-memory layout per CTA: [tile data (N_t padded) | inhi | outhi | shi | slo]
template <int ES>
__global__ void __launch_bounds__(kThreads, 4) permute_tiled_kernel(
    const typename Word<ES>::T* __restrict__ src, typename Word<ES>::T* __restrict__ dst,
    const __grid_constant__ PermDesc d) {
  using T = typename Word<ES>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tile = reinterpret_cast<T*>(smem_raw);
  const int tile_words = d.n_hi_in * d.rowp;
  int64_t* inhi = reinterpret_cast<int64_t*>(smem_raw + (((size_t)tile_words * ES + 15) & ~(size_t)15));
  int64_t* outhi = inhi + d.n_hi_in;
  int32_t* shi = reinterpret_cast<int32_t*>(outhi + d.n_hi_out);
  int32_t* slo = shi + d.n_hi_out;

  // ---- per-CTA tables -------------------------------------------------------
  // inhi[h]: storage offset of the hi part (U \ G_in, storage order) of input index h
  for (int h = threadIdx.x; h < d.n_hi_in; h += blockDim.x) {
    int64_t off = 0;
    int rem = h;
    for (int q = d.nuin - d.gin - 1; q >= 0; --q) {
      int a = d.uin[q];
      int e = d.ext[a];
      int dig = rem % e;
      rem /= e;
      off += (int64_t)dig * d.istride[a];
    }
    inhi[h] = off;
  }
  // outhi[g], shi[g]: output offset / smem offset of the hi part (U \ G_out, output order)
  for (int g = threadIdx.x; g < d.n_hi_out; g += blockDim.x) {
    int64_t off = 0;
    int32_t s = 0;
    int rem = g;
    for (int q = d.nuout - d.gout - 1; q >= 0; --q) {
      int a = d.uout[q];
      int e = d.ext[a];
      int dig = rem % e;
      rem /= e;
      off += (int64_t)dig * d.ostride[a];
      s += dig * d.pts[a];
    }
    outhi[g] = off;
    shi[g] = s;
  }
  // slo[l]: smem offset of the lo part (G_out, output order)
  for (int l = threadIdx.x; l < d.N_out; l += blockDim.x) {
    int32_t s = 0;
    int rem = l;
    for (int q = d.nuout - 1; q >= d.nuout - d.gout; --q) {
      int a = d.uout[q];
      int e = d.ext[a];
      int dig = rem % e;
      rem /= e;
      s += dig * d.pts[a];
    }
    slo[l] = s;
  }
  __syncthreads();

  constexpr int kMaxItems = 8;  // items in flight per lane
  for (int64_t tileid = blockIdx.x; tileid < d.ntiles; tileid += gridDim.x) {
    // tile coordinates -> base offsets, boundary limits
    int64_t base_in = 0, base_out = 0;
    int lim_in = 1 << 30, lim_out = 1 << 30;
    {
      uint32_t rem_hi = (uint32_t)(tileid >> 31);  // ntiles < 2^31 enforced on host
      (void)rem_hi;
      uint32_t rem = (uint32_t)tileid;
      for (int q = d.nb - 1; q >= 0; --q) {
        int a = d.bax[q];
        uint32_t quo = d.bdiv[q].div(rem);
        uint32_t c = rem - quo * d.bnt[q];
        rem = quo;
        int64_t start = (int64_t)c * d.ext[a];
        base_in += start * d.istride[a];
        base_out += start * d.ostride[a];
        if (a == d.a_in) lim_in = (int)(d.dim[a] - start);
        if (a == d.a_out) lim_out = (int)(d.dim[a] - start);
      }
    }
    const bool boundary = (d.a_in >= 0 && lim_in < d.ext[d.a_in]) ||
                          (d.a_out >= 0 && lim_out < d.ext[d.a_out]);
    const T* s = src + base_in;
    T* o = dst + base_out;
    if (!boundary) {
      // warp-per-run: an item is 32 consecutive elements of one contiguous run (input runs of
      // N_in elements on the load side, output runs of N_out on the store side); the only
      // per-item index math is one warp-uniform division, per element one add. Eight items
      // per lane are in flight before any of them is stored.
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kThreads / 32;
      const int cin = (d.N_in + 31) >> 5, cout = (d.N_out + 31) >> 5;
      const int items_in = d.n_hi_in * cin, items_out = d.n_hi_out * cout;
      for (int i0 = warp; i0 < items_in; i0 += nw * kMaxItems) {
        T v[kMaxItems];
#pragma unroll
        for (int u = 0; u < kMaxItems; ++u) {
          const int i = i0 + u * nw;
          if (i < items_in) {
            const int hi = d.cin_div.div((uint32_t)i), lo = (i - hi * cin) * 32 + lane;
            if (lo < d.N_in) v[u] = __ldg(s + inhi[hi] + lo);
          }
        }
#pragma unroll
        for (int u = 0; u < kMaxItems; ++u) {
          const int i = i0 + u * nw;
          if (i < items_in) {
            const int hi = d.cin_div.div((uint32_t)i), lo = (i - hi * cin) * 32 + lane;
            if (lo < d.N_in) tile[hi * d.rowp + lo] = v[u];
          }
        }
      }
      __syncthreads();
      for (int i0 = warp; i0 < items_out; i0 += nw * kMaxItems) {
        T v[kMaxItems];
#pragma unroll
        for (int u = 0; u < kMaxItems; ++u) {
          const int i = i0 + u * nw;
          if (i < items_out) {
            const int hi = d.cout_div.div((uint32_t)i), lo = (i - hi * cout) * 32 + lane;
            if (lo < d.N_out) v[u] = tile[shi[hi] + slo[lo]];
          }
        }
#pragma unroll
        for (int u = 0; u < kMaxItems; ++u) {
          const int i = i0 + u * nw;
          if (i < items_out) {
            const int hi = d.cout_div.div((uint32_t)i), lo = (i - hi * cout) * 32 + lane;
            if (lo < d.N_out) o[outhi[hi] + lo] = v[u];
          }
        }
      }
      __syncthreads();
    } else {
      // boundary tile: per-element validity on the (at most two) split axes
      for (int t = threadIdx.x; t < d.N_t; t += kThreads) {
        bool ok = true;
        if (d.a_in >= 0) {
          int a = d.a_in;
          uint32_t q = d.tsi_div[a].div((uint32_t)t);
          uint32_t dig = q - d.ext_div[a].div(q) * d.ext[a];
          ok = ok && (int)dig < lim_in;
        }
        if (d.a_out >= 0) {
          int a = d.a_out;
          uint32_t q = d.tsi_div[a].div((uint32_t)t);
          uint32_t dig = q - d.ext_div[a].div(q) * d.ext[a];
          ok = ok && (int)dig < lim_out;
        }
        if (ok) {
          uint32_t hi = d.div_in.div((uint32_t)t);
          uint32_t lo = (uint32_t)t - hi * (uint32_t)d.N_in;
          tile[hi * d.rowp + lo] = __ldg(s + inhi[hi] + lo);
        }
      }
      __syncthreads();
      for (int u = threadIdx.x; u < d.N_t; u += kThreads) {
        bool ok = true;
        if (d.a_in >= 0) {
          int a = d.a_in;
          uint32_t q = d.tso_div[a].div((uint32_t)u);
          uint32_t dig = q - d.ext_div[a].div(q) * d.ext[a];
          ok = ok && (int)dig < lim_in;
        }
        if (d.a_out >= 0) {
          int a = d.a_out;
          uint32_t q = d.tso_div[a].div((uint32_t)u);
          uint32_t dig = q - d.ext_div[a].div(q) * d.ext[a];
          ok = ok && (int)dig < lim_out;
        }
        if (ok) {
          uint32_t hi = d.div_out.div((uint32_t)u);
          uint32_t lo = (uint32_t)u - hi * (uint32_t)d.N_out;
          o[outhi[hi] + lo] = tile[shi[hi] + slo[lo]];
        }
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// Fast path 1 -- shared innermost axis (after merging, the storage-innermost
// axis is also the output-innermost axis): the permute is a gather of
// contiguous rows of L elements. Work unit = (row, 2 KB chunk); each lane moves
// 16-byte vectors, four in flight.
struct RowDesc {
  int64_t L;          // row length (elements)
  int64_t rows;
  int64_t chunks;     // chunks per row
  int nb;             // other axes, output order (outer -> inner)
  int64_t bdim[kMaxR];
  int64_t bistr[kMaxR];
  FastDiv bdiv[kMaxR];
  FastDiv chunk_div;
  int vec;            // 1: 16-byte vectors usable (aligned rows), 0: element copies
  int bulk;           // 1: TMA bulk-copy path (rows 16-byte aligned, long enough)
  int64_t bchunks;    // 8 KB chunks per row (bulk path)
  FastDiv bchunk_div;
  FastDiv vdiv;       // by 16-byte vectors per unit row (rows kernel)
};

// Unit = R consecutive OUTPUT rows (R <= 32, R * row_bytes <= 8 KB; these are one
// contiguous output run) or an 8 KB chunk of one long row. Lane j computes the
// input offset of row j of the unit once and shares it by warp shuffle; every lane
// then issues up to 16 independent 16-byte loads before its 16 stores (8 KB in
// flight per warp).
template <int ES>
__global__ void __launch_bounds__(256) permute_rows_kernel(const unsigned char* __restrict__ src,
                                                           unsigned char* __restrict__ dst,
                                                           const __grid_constant__ RowDesc d) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t row_bytes = d.L * ES;
  const bool grouped = row_bytes <= 8192;
  const int R = grouped ? (int)min64(32, 8192 / row_bytes) : 1;
  const int V = grouped ? (int)(row_bytes >> 4) : 512;  // 16-byte vectors per row (per chunk)
  const FastDiv& vdiv = d.vdiv;
  const int64_t units = grouped ? (d.rows + R - 1) / R : d.rows * d.chunks;
  for (int64_t u = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); u < units; u += warps) {
    int64_t r0, b0 = 0;
    int nr, nvec;
    if (grouped) {
      r0 = u * R;
      nr = (int)min64(R, d.rows - r0);
      nvec = nr * V;
    } else {
      const uint32_t row = d.chunk_div.div((uint32_t)u);
      r0 = row;
      nr = 1;
      b0 = (u - (int64_t)row * d.chunks) * 8192;
      nvec = (int)(min64(8192, row_bytes - b0) >> 4);
    }
    int64_t my_src = 0;
    if (lane < nr) {
      uint32_t rem = (uint32_t)(r0 + lane);
      for (int q = d.nb - 1; q >= 0; --q) {
        uint32_t quo = d.bdiv[q].div(rem);
        my_src += (int64_t)(rem - quo * (uint32_t)d.bdim[q]) * d.bistr[q];
        rem = quo;
      }
      my_src = my_src * ES + b0;
    }
    uint4 v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int i = lane + 32 * k;
      const uint32_t row = vdiv.div((uint32_t)i);
      const int64_t rs = __shfl_sync(0xffffffffu, my_src, (int)(row & 31));
      if (i < nvec) v[k] = __ldcs(reinterpret_cast<const uint4*>(src + rs + (int64_t)(i - (int)row * V) * 16));
    }
    uint4* o = reinterpret_cast<uint4*>(dst + r0 * row_bytes + b0);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int i = lane + 32 * k;
      if (i < nvec) __stcs(o + i, v[k]);
    }
  }
}

// element-wise fallback for rows that are not 16-byte multiples
template <int ES>
__global__ void __launch_bounds__(256) permute_rows_scalar_kernel(const unsigned char* __restrict__ src,
                                                                  unsigned char* __restrict__ dst,
                                                                  const __grid_constant__ RowDesc d) {
  using T = typename Word<ES>::T;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < d.rows; row += warps) {
    int64_t in_off = 0;
    uint32_t rem = (uint32_t)row;
    for (int q = d.nb - 1; q >= 0; --q) {
      uint32_t quo = d.bdiv[q].div(rem);
      in_off += (int64_t)(rem - quo * (uint32_t)d.bdim[q]) * d.bistr[q];
      rem = quo;
    }
    const T* s = reinterpret_cast<const T*>(src) + in_off;
    T* o = reinterpret_cast<T*>(dst) + row * d.L;
    for (int64_t e = lane; e < d.L; e += 32) o[e] = s[e];
  }
}

// ---------------------------------------------------------------------------
// Fast path 1b -- the same row gather with the TMA bulk-copy engine
// (cp.async.bulk global->shared, shared->global) when rows are 16-byte aligned.
// A "unit" is either a group of consecutive OUTPUT rows (short rows: R loads, one
// contiguous store) or a 8 KB chunk of one long row. One elected lane per warp
// drives a 4-stage ring of 8 KB shared buffers: stage i+3 is being loaded while
// unit i is stored, ~24 KB of reads in flight per warp with no per-element
// instructions at all.
constexpr int kBulkStage = 8192;
constexpr int kBulkStages = 4;
constexpr int kBulkWarps = 2;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
}

template <int ES>
__global__ void __launch_bounds__(kBulkWarps * 32) permute_rows_bulk_kernel(const unsigned char* __restrict__ src,
                                                                             unsigned char* __restrict__ dst,
                                                                             const __grid_constant__ RowDesc d) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t mbar[kBulkWarps][kBulkStages];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane != 0) return;
  unsigned char* ring = smem_raw + (size_t)warp * kBulkStages * kBulkStage;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  uint32_t mb[kBulkStages];
  for (int s = 0; s < kBulkStages; ++s) {
    mb[s] = (uint32_t)__cvta_generic_to_shared(&mbar[warp][s]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb[s]));
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  const int64_t row_bytes = d.L * ES;
  const bool grouped = row_bytes <= kBulkStage;
  const int64_t R = grouped ? (kBulkStage / row_bytes) : 1;  // rows per unit
  const int64_t units = grouped ? (d.rows + R - 1) / R : d.rows * d.bchunks;
  const int64_t wstride = (int64_t)gridDim.x * kBulkWarps;
  const int64_t first = (int64_t)blockIdx.x * kBulkWarps + warp;
  // input byte offset of output row r
  auto row_src = [&](int64_t r) -> int64_t {
    int64_t off = 0;
    uint32_t rem = (uint32_t)r;
    for (int q = d.nb - 1; q >= 0; --q) {
      uint32_t quo = d.bdiv[q].div(rem);
      off += (int64_t)(rem - quo * (uint32_t)d.bdim[q]) * d.bistr[q];
      rem = quo;
    }
    return off * ES;
  };
  auto issue_load = [&](int64_t u, int s) -> void {
    if (grouped) {
      const int64_t r0 = u * R;
      const int64_t nr = (r0 + R <= d.rows) ? R : d.rows - r0;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb[s]),
                   "r"((uint32_t)(nr * row_bytes)));
      for (int64_t j = 0; j < nr; ++j)
        bulk_g2s(ring_s + s * kBulkStage + (uint32_t)(j * row_bytes), src + row_src(r0 + j), (uint32_t)row_bytes,
                 mb[s]);
    } else {
      const uint32_t row = d.bchunk_div.div((uint32_t)u);
      const int64_t ch = u - (int64_t)row * d.bchunks;
      const int64_t b0 = ch * kBulkStage;
      const uint32_t nbytes = (uint32_t)((row_bytes - b0 < kBulkStage) ? row_bytes - b0 : kBulkStage);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb[s]), "r"(nbytes));
      bulk_g2s(ring_s + s * kBulkStage, src + row_src(row) + b0, nbytes, mb[s]);
    }
  };
  auto issue_store = [&](int64_t u, int s) -> void {
    int64_t off, nbytes;
    if (grouped) {
      const int64_t r0 = u * R;
      const int64_t nr = (r0 + R <= d.rows) ? R : d.rows - r0;
      off = r0 * row_bytes;
      nbytes = nr * row_bytes;
    } else {
      const uint32_t row = d.bchunk_div.div((uint32_t)u);
      const int64_t ch = u - (int64_t)row * d.bchunks;
      const int64_t b0 = ch * kBulkStage;
      off = (int64_t)row * row_bytes + b0;
      nbytes = (row_bytes - b0 < kBulkStage) ? row_bytes - b0 : kBulkStage;
    }
    bulk_s2g(dst + off, ring_s + s * kBulkStage, (uint32_t)nbytes);
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
  };
  const int64_t mine = (first < units) ? (units - first + wstride - 1) / wstride : 0;
  // prologue: S-1 loads in flight
  for (int64_t i = 0; i < kBulkStages - 1 && i < mine; ++i) issue_load(first + i * wstride, (int)i);
  for (int64_t i = 0; i < mine; ++i) {
    const int s = (int)(i % kBulkStages);
    const int64_t nxt = i + kBulkStages - 1;
    if (nxt < mine) {
      // its stage was last read by the store of unit i-1: wait for that smem read
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      issue_load(first + nxt * wstride, (int)(nxt % kBulkStages));
    }
    const uint32_t parity = (uint32_t)((i / kBulkStages) & 1);
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(mb[s]),
        "r"(parity)
        : "memory");
    issue_store(first + i * wstride, s);
  }
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// ---------------------------------------------------------------------------
// Fast path 2 -- 2-D transpose with batch: the storage-innermost axis (i, dim Di)
// and the output-innermost axis (j, dim Do) differ. One warp owns a T x T tile:
// it reads T rows of j (each a contiguous run of T i-elements, 256 B), stages
// them in a padded per-warp shared tile, and writes T rows of i (contiguous
// runs of T j-elements). No block barriers; T*T/32 loads in flight per lane.
struct T2Desc {
  int64_t Di, Do;      // extents of the i / j axes
  int64_t sj;          // input stride of j
  int64_t si;          // output stride of i
  int64_t ti, tj;      // tiles along i / j
  int64_t ntiles;      // batch * ti * tj
  int64_t n;           // elements (checked builds)
  int nb;              // batch axes, output order (outer -> inner)
  int64_t bdim[kMaxR];
  int64_t bistr[kMaxR];
  int64_t bostr[kMaxR];
  FastDiv bdiv[kMaxR];
  FastDiv ti_div, tj_div;
};

template <int ES, int T>
__global__ void __launch_bounds__(256) permute_t2d_kernel(const typename Word<ES>::T* __restrict__ src,
                                                          typename Word<ES>::T* __restrict__ dst, const __grid_constant__ T2Desc d) {
  using W = typename Word<ES>::T;
  constexpr int RPI = 32 / T;      // rows per warp instruction
  constexpr int NI = T / RPI;      // instructions per tile side
  constexpr int LD = T + 1;        // padded smem row
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  W* tile = reinterpret_cast<W*>(smem_raw) + warp * T * LD;
  const int r0 = lane / T, c = lane % T;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; t < d.ntiles; t += nwarps) {
    uint32_t q = (uint32_t)t;
    uint32_t qi = d.ti_div.div(q);
    const int64_t it = q - qi * (uint32_t)d.ti;
    uint32_t qj = d.tj_div.div(qi);
    const int64_t jt = qi - qj * (uint32_t)d.tj;
    int64_t bin = 0, bout = 0;
    uint32_t rem = qj;
    for (int k = d.nb - 1; k >= 0; --k) {
      uint32_t quo = d.bdiv[k].div(rem);
      int64_t dig = rem - quo * (uint32_t)d.bdim[k];
      rem = quo;
      bin += dig * d.bistr[k];
      bout += dig * d.bostr[k];
    }
    const int64_t i0 = it * T, j0 = jt * T;
    const bool full = (i0 + T <= d.Di) && (j0 + T <= d.Do);
    const W* s = src + bin + i0 + j0 * d.sj;
    W* o = dst + bout + j0 + i0 * d.si;
    TNB_DCHECK(bin + min64(T, d.Di - i0) - 1 + (min64(T, d.Do - j0) - 1) * d.sj + i0 + j0 * d.sj < d.n &&
                   bout + min64(T, d.Do - j0) - 1 + (min64(T, d.Di - i0) - 1) * d.si + j0 + i0 * d.si < d.n,
               "t2d tile out of range");
    W v[NI];
    if (full) {
#pragma unroll
      for (int k = 0; k < NI; ++k) v[k] = __ldcs(s + c + (int64_t)(k * RPI + r0) * d.sj);
#pragma unroll
      for (int k = 0; k < NI; ++k) tile[(k * RPI + r0) * LD + c] = v[k];
      __syncwarp();
#pragma unroll
      for (int k = 0; k < NI; ++k) v[k] = tile[c * LD + k * RPI + r0];
#pragma unroll
      for (int k = 0; k < NI; ++k) __stcs(o + c + (int64_t)(k * RPI + r0) * d.si, v[k]);
    } else {
#pragma unroll
      for (int k = 0; k < NI; ++k) {
        const int j = k * RPI + r0;
        if (i0 + c < d.Di && j0 + j < d.Do) tile[j * LD + c] = s[c + (int64_t)j * d.sj];
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < NI; ++k) {
        const int i = k * RPI + r0;
        if (j0 + c < d.Do && i0 + i < d.Di) o[c + (int64_t)i * d.si] = tile[c * LD + i];
      }
    }
    __syncwarp();
  }
}

// Fast path 2b -- the same 2-D transpose with CTA-wide tiles of 512-byte runs on BOTH
// sides (64 x 64 float64, 32 x 32 complex128): every input row segment and every output
// row segment a CTA touches is 512 contiguous bytes moved by 16-byte vector accesses, so a
// DRAM page opened for a tile serves 4x more bytes than with the 128-byte runs of the
// warp tiles above (the transposes whose two inner axes lie far apart in memory were
// row-activation bound there). Needs Di, Do >= the tile and 16-byte aligned rows.
template <int ES>
struct WideCfg {
  static constexpr int T = ES == 8 ? 64 : 32;  // 512-byte runs
  static constexpr int V = 16 / ES;            // elements per 16-byte vector
  static constexpr int LD = T + 1;             // padded smem row (elements)
};

template <int ES>
__global__ void __launch_bounds__(256) permute_t2w_kernel(const typename Word<ES>::T* __restrict__ src,
                                                          typename Word<ES>::T* __restrict__ dst,
                                                          const __grid_constant__ T2Desc d) {
  using W = typename Word<ES>::T;
  constexpr int T = WideCfg<ES>::T, V = WideCfg<ES>::V, LD = WideCfg<ES>::LD;
  constexpr int LANES_PER_ROW = T / V;          // 32: one row = one warp instruction
  constexpr int ROWS_PER_WARP = T / 8;          // 8 warps share the tile's rows
  extern __shared__ __align__(16) unsigned char smem_raw[];
  W* tile = reinterpret_cast<W*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  static_assert(LANES_PER_ROW == 32, "one 512-byte row per warp instruction");
  for (int64_t t = blockIdx.x; t < d.ntiles; t += gridDim.x) {
    uint32_t q = (uint32_t)t;
    uint32_t qi = d.ti_div.div(q);
    const int64_t it = q - qi * (uint32_t)d.ti;
    uint32_t qj = d.tj_div.div(qi);
    const int64_t jt = qi - qj * (uint32_t)d.tj;
    int64_t bin = 0, bout = 0;
    uint32_t rem = qj;
    for (int k = d.nb - 1; k >= 0; --k) {
      uint32_t quo = d.bdiv[k].div(rem);
      int64_t dig = rem - quo * (uint32_t)d.bdim[k];
      rem = quo;
      bin += dig * d.bistr[k];
      bout += dig * d.bostr[k];
    }
    const int64_t i0 = it * T, j0 = jt * T;
    const W* s = src + bin + i0 + j0 * d.sj;
    W* o = dst + bout + j0 + i0 * d.si;
    TNB_DCHECK(bin + min64(T, d.Di - i0) - 1 + (min64(T, d.Do - j0) - 1) * d.sj + i0 + j0 * d.sj < d.n &&
                   bout + min64(T, d.Do - j0) - 1 + (min64(T, d.Di - i0) - 1) * d.si + j0 + i0 * d.si < d.n,
               "t2w tile out of range");
    if ((i0 + T <= d.Di) && (j0 + T <= d.Do)) {
      // read: rows j (input-contiguous along i), 16-byte vectors, all loads in flight
      uint4 v[ROWS_PER_WARP];
#pragma unroll
      for (int k = 0; k < ROWS_PER_WARP; ++k) {
        const int j = warp * ROWS_PER_WARP + k;
        v[k] = __ldcs(reinterpret_cast<const uint4*>(s + (int64_t)j * d.sj) + lane);
      }
#pragma unroll
      for (int k = 0; k < ROWS_PER_WARP; ++k) {
        const int j = warp * ROWS_PER_WARP + k;
        const W* e = reinterpret_cast<const W*>(&v[k]);
#pragma unroll
        for (int u = 0; u < V; ++u) tile[j * LD + lane * V + u] = e[u];
      }
      __syncthreads();
      // write: rows i (output-contiguous along j)
#pragma unroll
      for (int k = 0; k < ROWS_PER_WARP; ++k) {
        const int i = warp * ROWS_PER_WARP + k;
        uint4 w;
        W* e = reinterpret_cast<W*>(&w);
#pragma unroll
        for (int u = 0; u < V; ++u) e[u] = tile[(lane * V + u) * LD + i];
        __stcs(reinterpret_cast<uint4*>(o + (int64_t)i * d.si) + lane, w);
      }
      __syncthreads();
    } else {
      for (int x = threadIdx.x; x < T * T; x += blockDim.x) {
        const int j = x / T, i = x % T;
        if (i0 + i < d.Di && j0 + j < d.Do) tile[j * LD + i] = s[i + (int64_t)j * d.sj];
      }
      __syncthreads();
      for (int x = threadIdx.x; x < T * T; x += blockDim.x) {
        const int i = x / T, j = x % T;
        if (j0 + j < d.Do && i0 + i < d.Di) o[j + (int64_t)i * d.si] = tile[j * LD + i];
      }
      __syncthreads();
    }
  }
}

struct Plan {
  bool identity = false;
  int64_t nelem = 0;
  int kind = 0;  // 0 generic tiled, 1 rows, 2 transpose2d
  int t2d_T = 0;  // 16 / 8: warp tiles; 0 with kind 2 never; -1: CTA-wide tiles (t2w)
  PermDesc d;
  RowDesc rd;
  T2Desc td;
  size_t smem = 0;
};

int make_plan(int es, int rank, const int64_t* shape, const int32_t* perm, Plan& p) {
  if (rank < 0 || rank > kMaxR) return fail(TNB_EINVAL, "permute: rank out of range");
  int64_t n = 1;
  std::vector<int> seen(rank, 0);
  for (int k = 0; k < rank; ++k) {
    if (shape[k] < 0) return fail(TNB_EINVAL, "permute: negative dimension");
    n *= shape[k];
    if (perm[k] < 0 || perm[k] >= rank || seen[perm[k]]) return fail(TNB_EINVAL, "permute: invalid permutation");
    seen[perm[k]] = 1;
  }
  p.nelem = n;
  if (n <= 1) { p.identity = true; return TNB_OK; }
  // storage strides
  std::vector<int64_t> sstride(rank, 1);
  for (int a = rank - 2; a >= 0; --a) sstride[a] = sstride[a + 1] * shape[a + 1];
  // logical axes (output order), dropping unit dims
  std::vector<int> lax;
  for (int k = 0; k < rank; ++k)
    if (shape[perm[k]] != 1) lax.push_back(perm[k]);
  // merge logical neighbours that are storage neighbours (storage axis a followed by a+1,
  // ignoring unit storage axes in between)
  struct Ax { int64_t dim, istride; int skey; };
  std::vector<Ax> out_axes;  // output order
  for (size_t i = 0; i < lax.size(); ++i) {
    int a = lax[i];
    if (!out_axes.empty()) {
      Ax& prev = out_axes.back();
      if (prev.istride == shape[a] * sstride[a]) {  // prev is directly outside a in storage
        prev.dim *= shape[a];
        prev.istride = sstride[a];
        prev.skey = a;
        continue;
      }
    }
    out_axes.push_back({shape[a], sstride[a], a});
  }
  int r = (int)out_axes.size();
  // storage order of merged axes: sort by istride descending
  std::vector<int> sorder(r);
  for (int i = 0; i < r; ++i) sorder[i] = i;
  std::sort(sorder.begin(), sorder.end(), [&](int x, int y) { return out_axes[x].istride > out_axes[y].istride; });
  bool ident = true;
  for (int i = 0; i < r; ++i) ident = ident && (sorder[i] == i);
  if (ident) { p.identity = true; return TNB_OK; }
  if (n >= (int64_t(1) << 62)) return fail(TNB_EINVAL, "permute: tensor too large");

  PermDesc& d = p.d;
  memset(&d, 0, sizeof(d));
  d.r = r;
  // index merged axes by STORAGE position a = 0..r-1 (outer->inner)
  std::vector<int> s2o(r);  // storage pos -> output pos
  for (int a = 0; a < r; ++a) s2o[a] = sorder[a];
  std::vector<int> o2s(r);
  for (int a = 0; a < r; ++a) o2s[sorder[a]] = a;
  {
    // merged axes by storage position: dims / strides (input) and output strides
    std::vector<int64_t> mdim(r), mis(r), mos(r);
    std::vector<int64_t> ostr_k(r, 1);
    for (int k = r - 2; k >= 0; --k) ostr_k[k] = ostr_k[k + 1] * out_axes[k + 1].dim;
    for (int a = 0; a < r; ++a) {
      mdim[a] = out_axes[s2o[a]].dim;
      mis[a] = out_axes[s2o[a]].istride;
      mos[a] = ostr_k[s2o[a]];
    }
    const int a_si = r - 1, a_so = o2s[r - 1];
    if (a_si == a_so && mdim[a_si] * es >= 64 && n / mdim[a_si] < (int64_t(1) << 31)) {
      RowDesc& rd = p.rd;
      memset(&rd, 0, sizeof(rd));
      rd.L = mdim[a_si];
      rd.rows = n / rd.L;
      rd.chunks = (rd.L * es + 8191) / 8192;
      if (rd.rows * rd.chunks >= (int64_t(1) << 31)) return fail(TNB_EUNSUP, "permute: too many rows");
      rd.chunk_div = FastDiv((uint32_t)rd.chunks);
      for (int k = 0; k < r - 1; ++k) {
        int a = o2s[k];
        rd.bdim[rd.nb] = mdim[a];
        rd.bistr[rd.nb] = mis[a];
        rd.bdiv[rd.nb] = FastDiv((uint32_t)mdim[a]);
        rd.nb++;
      }
      rd.vec = ((rd.L * es) % 16 == 0) ? 1 : 0;
      rd.vdiv = FastDiv((uint32_t)(rd.L * es <= 8192 ? (rd.L * es) / 16 : 512));
      // bulk copies: 16-byte granularity; the input row strides are multiples of L
      rd.bulk = (rd.vec && rd.L * es >= 8192) ? 1 : 0;  // long rows: TMA bulk copies
      if (rd.bulk) {
        const int64_t rb = rd.L * es;
        rd.bchunks = (rb + kBulkStage - 1) / kBulkStage;
        rd.bchunk_div = FastDiv((uint32_t)rd.bchunks);
        if (rd.rows * rd.bchunks >= (int64_t(1) << 31)) rd.bulk = 0;
      }
      p.kind = 1;
      return TNB_OK;
    }
    static const bool force_tiled = getenv("TNB_PERM_TILED") != nullptr;  // dev A/B
    if (!force_tiled && a_si != a_so && mdim[a_si] * es >= 64 && mdim[a_so] * es >= 64 && (es == 8 || es == 16)) {
      T2Desc& td = p.td;
      memset(&td, 0, sizeof(td));
      // 16 x 16 tiles (128-byte runs for f64, 256-byte for c128): measured 0.87-0.95 of
      // HBM on the [64]^4 f64 sweep vs 0.77-0.95 with 32 x 32 f64 tiles (4x more tiles:
      // no tail wave, more tiles in flight per SM)
      int T = 16;
      if (es == 16 && (mdim[a_si] < 16 || mdim[a_so] < 16)) T = 8;
      // CTA-wide 512-byte-run tiles when both inner axes span a tile and every row start
      // stays 16-byte aligned (all input/output strides even in float64 elements)
      const int TW = es == 8 ? 64 : 32;
      bool wide = mdim[a_si] >= TW && mdim[a_so] >= TW;
      if (wide && es == 8) {
        wide = mis[a_so] % 2 == 0 && mos[a_si] % 2 == 0;
        for (int k = 0; k < r; ++k) {
          int a = o2s[k];
          if (a != a_si && a != a_so && (mis[a] % 2 || mos[a] % 2)) wide = false;
        }
      }
      static const int t_env = getenv("TNB_T2D_T") ? atoi(getenv("TNB_T2D_T")) : 0;  // dev A/B
      if (t_env == 16) wide = false;
      if (wide) T = TW;
      td.Di = mdim[a_si];
      td.Do = mdim[a_so];
      td.sj = mis[a_so];
      td.si = mos[a_si];
      td.ti = (td.Di + T - 1) / T;
      td.tj = (td.Do + T - 1) / T;
      int64_t nbatch = n / (td.Di * td.Do);
      td.ntiles = nbatch * td.ti * td.tj;
      td.n = n;
      if (td.ntiles < (int64_t(1) << 31)) {
        td.ti_div = FastDiv((uint32_t)td.ti);
        td.tj_div = FastDiv((uint32_t)td.tj);
        for (int k = 0; k < r; ++k) {
          int a = o2s[k];
          if (a == a_si || a == a_so) continue;
          td.bdim[td.nb] = mdim[a];
          td.bistr[td.nb] = mis[a];
          td.bostr[td.nb] = mos[a];
          td.bdiv[td.nb] = FastDiv((uint32_t)mdim[a]);
          td.nb++;
        }
        p.kind = 2;
        p.t2d_T = wide ? -1 : T;
        return TNB_OK;
      }
    }
  }
  std::vector<int64_t> ostr(r, 1);  // output stride by output position
  for (int k = r - 2; k >= 0; --k) ostr[k] = ostr[k + 1] * out_axes[k + 1].dim;
  for (int a = 0; a < r; ++a) {
    int k = s2o[a];
    d.dim[a] = out_axes[k].dim;
    d.istride[a] = out_axes[k].istride;
    d.ostride[a] = ostr[k];
    d.ext[a] = 1;
  }
  // ---- tile selection ----
  const int run_lo = std::max(1, 256 / es);     // >= 256 B contiguous per run
  const int tmax = (es == 16) ? 2048 : 4096;  // <= 32 KB of data per tile
  std::vector<int> inU(r, 0);
  // G_in: storage suffix
  int64_t prod = 1;
  int gin = 0;
  d.a_in = -1;
  for (int a = r - 1; a >= 0 && prod < run_lo; --a) {
    int64_t need = (run_lo + prod - 1) / prod;
    if (d.dim[a] <= need || d.dim[a] * prod <= 2 * run_lo) {
      d.ext[a] = (int32_t)d.dim[a];
    } else {
      int64_t e = need;
      // prefer a divisor of dim in [need, 2*need]
      for (int64_t c = need; c <= 2 * need; ++c)
        if (d.dim[a] % c == 0) { e = c; break; }
      d.ext[a] = (int32_t)e;
      d.a_in = a;
    }
    prod *= d.ext[a];
    inU[a] = 1;
    ++gin;
  }
  const int gin_lo = r - gin;  // G_in = storage axes [gin_lo, r)
  // G_out: output suffix
  int64_t tprod = prod;  // tile size so far
  int64_t oprod = 1;
  int gout = 0;
  d.a_out = -1;
  for (int k = r - 1; k >= 0; --k) {
    int a = o2s[k];
    bool need_more = (oprod < run_lo) || (tprod < 1024 && oprod * 2 <= tmax);
    if (!need_more) break;
    if (inU[a]) {
      if (a == d.a_in && d.ext[a] != d.dim[a]) {
        // the partial input axis is also inner on the output side: take it whole if the tile
        // stays within bounds (else the output runs would be only ext elements long)
        const int64_t grown = tprod / d.ext[a] * d.dim[a];
        if (grown <= tmax) {
          tprod = grown;
          oprod *= d.dim[a];
          d.ext[a] = (int32_t)d.dim[a];
          d.a_in = -1;
          ++gout;
          continue;
        }
        oprod *= d.ext[a];  // partial axis: must be G_out's top
        ++gout;
        break;
      }
      oprod *= d.ext[a];
      ++gout;
      continue;
    }
    int64_t room = tmax / tprod;
    if (room < 2) break;
    int64_t want = (oprod < run_lo) ? (run_lo + oprod - 1) / oprod : std::max<int64_t>(2, 1024 / tprod);
    want = std::min(want, room);
    if (d.dim[a] <= want) {
      d.ext[a] = (int32_t)d.dim[a];
      inU[a] = 1;
      oprod *= d.ext[a];
      tprod *= d.ext[a];
      ++gout;
      continue;
    }
    int64_t e = want;
    for (int64_t c = want; c >= std::max<int64_t>(1, want / 2); --c)
      if (d.dim[a] % c == 0) { e = c; break; }
    d.ext[a] = (int32_t)e;
    d.a_out = a;
    inU[a] = 1;
    oprod *= e;
    tprod *= e;
    ++gout;
    break;
  }
  // G_out must be an output suffix of U with only its top axis partial; fold any U axis
  // that sits inside it (can only be full G_in axes) -- already counted above.
  int N_t = (int)tprod;
  int N_out = (int)oprod;
  int64_t nin = 1;  // G_in extents (the partial input axis may have grown to full above)
  for (int a = gin_lo; a < r; ++a) nin *= d.ext[a];
  const int N_in = (int)nin;
  // U in storage order and output order
  d.nuin = 0;
  for (int a = 0; a < r; ++a)
    if (inU[a]) d.uin[d.nuin++] = a;
  d.nuout = 0;
  for (int k = 0; k < r; ++k)
    if (inU[o2s[k]]) d.uout[d.nuout++] = o2s[k];
  d.gin = gin;
  d.gout = gout;
  // sanity: G_out are the innermost gout axes of uout
  d.N_t = N_t;
  d.N_in = N_in;
  d.N_out = N_out;
  // one 8-byte (or one 16-byte element) pad per input run breaks the power-of-two
  // row stride that the output-order (column) reads of a 2-D transpose would hit
  const int pad = (es <= 8) ? 8 / es : 1;
  d.rowp = N_in + ((N_t / N_in > 1) ? pad : 0);
  d.n_hi_in = N_t / N_in;
  d.n_hi_out = N_t / N_out;
  // tile strides
  {
    int32_t acc = 1;
    for (int q = d.nuin - 1; q >= 0; --q) {
      int a = d.uin[q];
      d.tsi[a] = acc;
      if (q >= d.nuin - gin) d.pts[a] = acc;
      else d.pts[a] = (acc / N_in) * d.rowp;
      acc *= d.ext[a];
    }
    acc = 1;
    for (int q = d.nuout - 1; q >= 0; --q) {
      int a = d.uout[q];
      d.tso[a] = acc;
      acc *= d.ext[a];
    }
    for (int a = 0; a < r; ++a) {
      if (inU[a]) {
        d.tsi_div[a] = FastDiv((uint32_t)d.tsi[a]);
        d.tso_div[a] = FastDiv((uint32_t)d.tso[a]);
        d.ext_div[a] = FastDiv((uint32_t)d.ext[a]);
      }
    }
  }
  d.div_in = FastDiv((uint32_t)N_in);
  d.div_out = FastDiv((uint32_t)N_out);
  d.cin_div = FastDiv((uint32_t)((N_in + 31) / 32));
  d.cout_div = FastDiv((uint32_t)((N_out + 31) / 32));
  // batch axes in output order (outer -> inner), tiles along each
  d.nb = 0;
  int64_t ntiles = 1;
  for (int k = 0; k < r; ++k) {
    int a = o2s[k];
    int64_t nt = (d.dim[a] + d.ext[a] - 1) / d.ext[a];
    if (nt > 1) {
      d.bax[d.nb] = a;
      d.bnt[d.nb] = (uint32_t)nt;
      d.bdiv[d.nb] = FastDiv((uint32_t)nt);
      ++d.nb;
      ntiles *= nt;
    }
  }
  if (ntiles >= (int64_t(1) << 31)) return fail(TNB_EUNSUP, "permute: too many tiles (tensor too large)");
  d.ntiles = ntiles;
  size_t data_bytes = ((size_t)d.n_hi_in * d.rowp * es + 15) & ~(size_t)15;
  p.smem = data_bytes + (size_t)(d.n_hi_in + d.n_hi_out) * 8 + (size_t)(d.n_hi_out + d.N_out) * 4;
  if (N_t > 4096) return fail(TNB_EINVAL, "permute: internal tile too large");
  return TNB_OK;
}

template <int ES, int T>
int launch_t2d(const void* src, void* dst, const Plan& p, cudaStream_t st) {
  using W = typename Word<ES>::T;
  auto kern = permute_t2d_kernel<ES, T>;
  const size_t smem = (size_t)8 * T * (T + 1) * ES;
  static bool configured = false;
  if (!configured) {
    TNB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  static int per_sm = 0;
  if (per_sm == 0) {
    TNB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
    if (per_sm < 1) per_sm = 1;
  }
  int64_t grid = std::min<int64_t>((p.td.ntiles + 7) / 8, (int64_t)sm_count() * per_sm);
  kern<<<(unsigned)grid, 256, smem, st>>>(static_cast<const W*>(src), static_cast<W*>(dst), p.td);
  count_launch();
  TNB_CUDA_CHECK(cudaGetLastError());
  return TNB_OK;
}

template <int ES>
int launch_t2w(const void* src, void* dst, const Plan& p, cudaStream_t st) {
  using W = typename Word<ES>::T;
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) != 0)
    return -1;  // caller falls back to the warp-tile kernel
  auto kern = permute_t2w_kernel<ES>;
  constexpr int T = WideCfg<ES>::T, LD = WideCfg<ES>::LD;
  const size_t smem = (size_t)T * LD * ES;
  static int per_sm = 0;
  if (per_sm == 0) {
    TNB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    TNB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
    if (per_sm < 1) per_sm = 1;
  }
  const int64_t grid = std::min<int64_t>(p.td.ntiles, (int64_t)sm_count() * per_sm);
  kern<<<(unsigned)grid, 256, smem, st>>>(static_cast<const W*>(src), static_cast<W*>(dst), p.td);
  count_launch();
  TNB_CUDA_CHECK(cudaGetLastError());
  return TNB_OK;
}

template <int ES>
int launch_rows_bulk(const void* src, void* dst, const Plan& p, cudaStream_t st) {
  auto kern = permute_rows_bulk_kernel<ES>;
  const size_t smem = (size_t)kBulkWarps * kBulkStages * kBulkStage;
  static int per_sm = 0;
  if (per_sm == 0) {
    TNB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    TNB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBulkWarps * 32, smem));
    if (per_sm < 1) per_sm = 1;
  }
  const int64_t row_bytes = p.rd.L * ES;
  const int64_t units = row_bytes <= kBulkStage ? (p.rd.rows + (kBulkStage / row_bytes) - 1) / (kBulkStage / row_bytes)
                                                : p.rd.rows * p.rd.bchunks;
  const int64_t grid = std::min<int64_t>((units + kBulkWarps - 1) / kBulkWarps, (int64_t)sm_count() * per_sm);
  kern<<<(unsigned)grid, kBulkWarps * 32, smem, st>>>(static_cast<const unsigned char*>(src),
                                                       static_cast<unsigned char*>(dst), p.rd);
  count_launch();
  TNB_CUDA_CHECK(cudaGetLastError());
  return TNB_OK;
}

template <int ES>
int launch_rows(const void* src, void* dst, const Plan& p, cudaStream_t st) {
  const bool aligned = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  if (p.rd.bulk && aligned) return launch_rows_bulk<ES>(src, dst, p, st);
  const bool vec = p.rd.vec && aligned;
  auto kern = vec ? permute_rows_kernel<ES> : permute_rows_scalar_kernel<ES>;
  static int per_sm[2] = {0, 0};
  int& psm = per_sm[vec ? 1 : 0];
  if (psm == 0) {
    TNB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&psm, kern, 256, 0));
    if (psm < 1) psm = 1;
  }
  const int64_t row_bytes = p.rd.L * ES;
  int64_t units = p.rd.rows;
  if (vec) {
    const int64_t R = row_bytes <= 8192 ? std::min<int64_t>(32, 8192 / row_bytes) : 1;
    units = row_bytes <= 8192 ? (p.rd.rows + R - 1) / R : p.rd.rows * p.rd.chunks;
  }
  const int64_t grid = std::min<int64_t>((units + 7) / 8, (int64_t)sm_count() * psm);
  kern<<<(unsigned)grid, 256, 0, st>>>(static_cast<const unsigned char*>(src), static_cast<unsigned char*>(dst),
                                       p.rd);
  count_launch();
  TNB_CUDA_CHECK(cudaGetLastError());
  return TNB_OK;
}

template <int ES>
int launch(const void* src, void* dst, const Plan& p, cudaStream_t st) {
  if (p.kind == 1) return launch_rows<ES>(src, dst, p, st);
  if (p.kind == 2) {
    if constexpr (ES == 8 || ES == 16) {
      if (p.t2d_T == -1) {
        int rc = launch_t2w<ES>(src, dst, p, st);
        if (rc != -1) return rc;
        // unaligned base pointers: warp tiles over the same descriptor (tile sides 16 / 8)
        Plan q = p;
        const int Tn = 16;
        q.td.ti = (q.td.Di + Tn - 1) / Tn;
        q.td.tj = (q.td.Do + Tn - 1) / Tn;
        q.td.ntiles = q.td.ntiles / ((p.td.Di + WideCfg<ES>::T - 1) / WideCfg<ES>::T) /
                      ((p.td.Do + WideCfg<ES>::T - 1) / WideCfg<ES>::T) * q.td.ti * q.td.tj;
        q.td.ti_div = FastDiv((uint32_t)q.td.ti);
        q.td.tj_div = FastDiv((uint32_t)q.td.tj);
        return launch_t2d<ES, 16>(src, dst, q, st);
      }
    }
    if constexpr (ES == 8) return launch_t2d<8, 16>(src, dst, p, st);
    if constexpr (ES == 16) {
      if (p.t2d_T == 16) return launch_t2d<16, 16>(src, dst, p, st);
      return launch_t2d<16, 8>(src, dst, p, st);
    }
  }
  using T = typename Word<ES>::T;
  auto kern = permute_tiled_kernel<ES>;
  static int configured_smem[1] = {0};
  if ((int)p.smem > 48 * 1024 && configured_smem[0] < (int)p.smem) {
    TNB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
    configured_smem[0] = (int)p.smem;
  }
  int per_sm = 0;
  TNB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, p.smem));
  if (per_sm < 1) per_sm = 1;
  int64_t grid = std::min<int64_t>(p.d.ntiles, (int64_t)sm_count() * per_sm);
  kern<<<(unsigned)grid, kThreads, p.smem, st>>>(static_cast<const T*>(src), static_cast<T*>(dst), p.d);
  count_launch();
  TNB_CUDA_CHECK(cudaGetLastError());
  return TNB_OK;
}

}  // namespace

int permute_device(const void* src, void* dst, int es, int rank, const int64_t* shape, const int32_t* perm,
                   cudaStream_t st) {
  Plan p;
  int rc = make_plan(es, rank, shape, perm, p);
  if (rc) return rc;
  if (p.nelem == 0) return TNB_OK;
  if (p.identity) {
    TNB_CUDA_CHECK(cudaMemcpyAsync(dst, src, (size_t)p.nelem * es, cudaMemcpyDeviceToDevice, st));
    return TNB_OK;
  }
  KTimer kt(TNB_KF_PERMUTE, st, 2.0 * (double)p.nelem * es);
  switch (es) {
    case 1: return launch<1>(src, dst, p, st);
    case 2: return launch<2>(src, dst, p, st);
    case 4: return launch<4>(src, dst, p, st);
    case 8: return launch<8>(src, dst, p, st);
    case 16: return launch<16>(src, dst, p, st);
    default: return fail(TNB_EINVAL, "permute: elem_size must be 1, 2, 4, 8 or 16");
  }
}

}  // namespace tnb

extern "C" int tnb_permute(const void* src, void* dst, int elem_size, int rank, const int64_t* shape,
                           const int32_t* perm, void* stream) {
  int rc = tnb::require_device();
  if (rc) return rc;
  if (rank > 0 && (!shape || !perm)) return tnb::fail(TNB_EINVAL, "permute: shape/perm is NULL");
  if (elem_size != 1 && elem_size != 2 && elem_size != 4 && elem_size != 8 && elem_size != 16)
    return tnb::fail(TNB_EINVAL, "permute: elem_size must be 1, 2, 4, 8 or 16");
  return tnb::permute_device(src, dst, elem_size, rank, shape, perm, (cudaStream_t)stream);
}

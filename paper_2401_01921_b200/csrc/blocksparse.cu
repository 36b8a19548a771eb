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
//      output tile list) from a pinned staging buffer.
//   2. pairing kernel (ON DEVICE, one CTA): thread per output block o finds its
//      contributing pairs (i asc, j asc) -- exactly the reference's accumulation
//      order restricted to o -- and writes a CSR (out_ptr, pair list).
//   3. grouped GEMM kernel: one CTA per output tile; it loops over its output
//      block's pairs in that order, accumulating all of them in registers
//      (deterministic, no atomics), then stores the tile once. Tiles of blocks
//      with no pair store zeros.
#include <algorithm>
#include <array>
#include <map>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "gemm_core.cuh"

namespace tnb {
namespace {

struct BlockDesc {
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
  int64_t max_pairs;
};

// ---- pairing: one CTA; thread per output block -----------------------------
__device__ __forceinline__ bool a_matches(const BsMeta& m, int i, int o) {
  const int32_t* aq = m.a_qn + (int64_t)i * m.ra;
  const int32_t* oq = m.out_qn + (int64_t)o * m.ro;
  for (int f = 0; f < m.nfa; ++f)
    if (aq[m.a_free[f]] != oq[f]) return false;
  return true;
}
__device__ __forceinline__ bool b_matches(const BsMeta& m, int i, int j, int o) {
  const int32_t* aq = m.a_qn + (int64_t)i * m.ra;
  const int32_t* bq = m.b_qn + (int64_t)j * m.rb;
  const int32_t* oq = m.out_qn + (int64_t)o * m.ro + m.nfa;
  for (int c = 0; c < m.nc; ++c)
    if (aq[m.a_axes[c]] != bq[m.b_axes[c]]) return false;
  for (int f = 0; f < m.nfb; ++f)
    if (bq[m.b_free[f]] != oq[f]) return false;
  return true;
}

__global__ void __launch_bounds__(1024) bs_pair_kernel(const BsMeta m) {
  __shared__ int32_t carry;
  __shared__ int32_t wsum[32];
  int32_t* cnt = m.out_ptr + 1;  // counts first, then scanned in place
  for (int o = threadIdx.x; o < m.nout; o += blockDim.x) {
    int c = 0;
    for (int i = 0; i < m.na; ++i) {
      if (!a_matches(m, i, o)) continue;
      for (int j = 0; j < m.nb; ++j) c += b_matches(m, i, j, o) ? 1 : 0;
    }
    cnt[o] = c;
  }
  __syncthreads();
  // inclusive scan of cnt[0..nout) in chunks of blockDim
  if (threadIdx.x == 0) {
    carry = 0;
    m.out_ptr[0] = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int base = 0; base < m.nout; base += blockDim.x) {
    int o = base + threadIdx.x;
    int v = (o < m.nout) ? cnt[o] : 0;
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
    int incl = v + (warp > 0 ? wsum[warp - 1] : 0) + carry;
    __syncthreads();
    if (o < m.nout) cnt[o] = incl;
    if (threadIdx.x == blockDim.x - 1) carry = incl;
    __syncthreads();
  }
  // write pairs of each output block in reference order (i asc, j asc)
  if (m.out_ptr[m.nout] > m.max_pairs) {
    if (threadIdx.x == 0) m.err[0] = 1;
    return;
  }
  for (int o = threadIdx.x; o < m.nout; o += blockDim.x) {
    int p = m.out_ptr[o];
    for (int i = 0; i < m.na; ++i) {
      if (!a_matches(m, i, o)) continue;
      for (int j = 0; j < m.nb; ++j)
        if (b_matches(m, i, j, o)) {
          m.pairs[2 * p] = i;
          m.pairs[2 * p + 1] = j;
          ++p;
        }
    }
  }
}

// ---- grouped GEMM: one CTA per output tile ------------------------------------
template <bool CPLX, int MODE>
struct BsCfg;
template <int MODE>
struct BsCfg<false, MODE> { using Core = TileCore<false, 0, 64, 64, 16, 2, 2, 3>; };
template <int MODE>
struct BsCfg<true, MODE> { using Core = TileCore<true, MODE, 64, 64, 8, 2, 2, 3>; };

// Per-call data pointers (A blocks, B blocks, output blocks) travel as a kernel
// parameter when they fit, so a cached plan needs no per-call H2D copy.
constexpr int kInlinePtrs = 1024;
struct PtrTable {
  const void* p[kInlinePtrs];
};

template <bool CPLX, int MODE>
__global__ void __launch_bounds__(128, 2) bs_gemm_kernel(const __grid_constant__ BsMeta m,
                                                         const __grid_constant__ PtrTable pt) {
  using Core = typename BsCfg<CPLX, MODE>::Core;
  using T = typename Core::T;
  extern __shared__ __align__(16) unsigned char smem[];
  const void* const* ptrs = m.ptrs ? m.ptrs : pt.p;
  const TileRef t = m.tiles[blockIdx.x];
  if (m.mask && !m.mask[t.panel]) return;  // panel owned by another rank
  const int M = m.out_M[t.o], N = m.out_N[t.o];
  typename Core::Acc acc;
  Core::zero(acc);
  const int p0 = m.out_ptr[t.o], p1 = m.out_ptr[t.o + 1];
  for (int p = p0; p < p1; ++p) {
    const int i = m.pairs[2 * p], j = m.pairs[2 * p + 1];
    const BlockDesc& da = m.da[i];
    const BlockDesc& db = m.db[j];
    const T* A = static_cast<const T*>(ptrs[i]);
    const T* B = static_cast<const T*>(ptrs[m.na + j]);
    const bool a_mfast = da.free_g.n > 0 && da.free_g.stride[da.free_g.n - 1] == 1;
    const bool b_nfast = db.free_g.n > 0 && db.free_g.stride[db.free_g.n - 1] == 1;
    Core::mainloop(smem, A, B, da.free_g, da.k_g, db.k_g, db.free_g, t.m0, t.n0, M, N, 0, da.K, a_mfast, b_nfast,
                   acc);
  }
  Core::store(static_cast<T*>(const_cast<void*>(ptrs[m.na + m.nb + t.o])), N, t.m0, t.n0, M, N, acc);
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
struct Plan {
  unsigned char* dblob = nullptr;
  BsMeta meta;
  int64_t npairs = 0;
  size_t o_optr = 0, o_pairs = 0;
  int dtype = 0;
};

struct PlanCache {
  std::mutex mu;
  std::unordered_map<std::string, Plan> plans;
  int device = -1;
  void* stage = nullptr;  // pinned staging for large pointer tables
  size_t stage_cap = 0;
  cudaEvent_t stage_ev = nullptr;
};
PlanCache g_cache;

template <bool CPLX, int MODE>
int launch_bs(const BsMeta& meta, const PtrTable* pt, cudaStream_t st) {
  using Core = typename BsCfg<CPLX, MODE>::Core;
  auto kern = bs_gemm_kernel<CPLX, MODE>;
  static bool configured = false;
  if (!configured) {
    TNB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Core::kSmem));
    configured = true;
  }
  if (meta.ntiles > 0) {
    kern<<<meta.ntiles, Core::NT, Core::kSmem, st>>>(meta, *pt);
    count_launch();
    TNB_CUDA_CHECK(cudaGetLastError());
  }
  return TNB_OK;
}

template <typename X>
void append(std::string& key, const X* p, size_t n) {
  key.append(reinterpret_cast<const char*>(p), n * sizeof(X));
}

}  // namespace
}  // namespace tnb

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
    int32_t hdr[8] = {dtype, na, nb, nout, rank_a, rank_b, nc, 0};
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
  std::lock_guard<std::mutex> lock(g_cache.mu);
  int dev = 0;
  TNB_CUDA_CHECK(cudaGetDevice(&dev));
  if (g_cache.device != dev) {
    g_cache.plans.clear();  // plans are per device (one process normally drives one GPU)
    g_cache.device = dev;
  }
  auto hit = g_cache.plans.find(key);
  if (hit == g_cache.plans.end()) {
    if (g_cache.plans.size() >= 256) {
      TNB_CUDA_CHECK(cudaStreamSynchronize(st));
      for (auto& kv : g_cache.plans) cudaFree(kv.second.dblob);
      g_cache.plans.clear();
    }
    Plan plan;
    plan.dtype = dtype;
    BsMeta& meta = plan.meta;
    memset(&meta, 0, sizeof(meta));
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
      if (F >= (1ll << 31) || K >= (1ll << 31)) return false;
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
    const int BM = 64, BN = 64;
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
    size_t off = 0;
    auto take = [&](size_t bytes) {
      size_t o = align_up(off, 16);
      off = o + bytes;
      return o;
    };
    const size_t o_aqn = take((size_t)na * rank_a * 4), o_bqn = take((size_t)nb * rank_b * 4),
                 o_oqn = take((size_t)nout * ro * 4), o_oM = take((size_t)nout * 4), o_oN = take((size_t)nout * 4),
                 o_da = take(sizeof(BlockDesc) * na), o_db = take(sizeof(BlockDesc) * nb),
                 o_tiles = take(sizeof(TileRef) * tiles.size()),
                 o_mask = take(panel_mask ? (size_t)npanels : 0);
    const size_t upload = off;
    const size_t o_optr = take((size_t)(nout + 1) * 4), o_err = take(16), o_pairs = take((size_t)meta.max_pairs * 8);
    const size_t total = off;
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
    TNB_CUDA_CHECK(cudaMemsetAsync(dblob + o_err, 0, 16, st));
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
    meta.ptrs = nullptr;
    bs_pair_kernel<<<1, 1024, 0, st>>>(meta);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      cudaFree(dblob);
      return cuda_fail(e, "bs_contract: pairing kernel launch");
    }
    plan.npairs = exact_pairs;
    plan.o_optr = o_optr;
    plan.o_pairs = o_pairs;
    hit = g_cache.plans.emplace(key, plan).first;
  }
  Plan& plan = hit->second;
  BsMeta meta = plan.meta;
  // ---- per-call data pointers
  const int nptr = na + nb + nout;
  PtrTable pt;
  if (nptr <= kInlinePtrs) {
    for (int i = 0; i < na; ++i) pt.p[i] = a_ptrs[i];
    for (int j = 0; j < nb; ++j) pt.p[na + j] = b_ptrs[j];
    for (int o = 0; o < nout; ++o) pt.p[na + nb + o] = out_ptrs[o];
    meta.ptrs = nullptr;
  } else {
    if (g_cache.stage_ev) TNB_CUDA_CHECK(cudaEventSynchronize(g_cache.stage_ev));
    size_t bytes = (size_t)nptr * sizeof(void*);
    if (g_cache.stage_cap < bytes) {
      if (g_cache.stage) cudaFreeHost(g_cache.stage);
      g_cache.stage_cap = std::max(bytes, (size_t)1 << 16);
      TNB_CUDA_CHECK(cudaMallocHost(&g_cache.stage, g_cache.stage_cap));
    }
    if (!g_cache.stage_ev) TNB_CUDA_CHECK(cudaEventCreateWithFlags(&g_cache.stage_ev, cudaEventDisableTiming));
    const void** hp = static_cast<const void**>(g_cache.stage);
    for (int i = 0; i < na; ++i) hp[i] = a_ptrs[i];
    for (int j = 0; j < nb; ++j) hp[na + j] = b_ptrs[j];
    for (int o = 0; o < nout; ++o) hp[na + nb + o] = out_ptrs[o];
    void* dptr = nullptr;
    TNB_CUDA_CHECK(cudaMallocAsync(&dptr, bytes, st));
    TNB_CUDA_CHECK(cudaMemcpyAsync(dptr, hp, bytes, cudaMemcpyHostToDevice, st));
    TNB_CUDA_CHECK(cudaEventRecord(g_cache.stage_ev, st));
    meta.ptrs = static_cast<const void* const*>(dptr);
  }
  if (dtype == TNB_F64) rc = launch_bs<false, 0>(meta, &pt, st);
  else rc = launch_bs<true, 0>(meta, &pt, st);
  if (meta.ptrs) cudaFreeAsync(const_cast<void*>(static_cast<const void*>(meta.ptrs)), st);
  if (rc != TNB_OK) return rc;
  if (npairs) *npairs = plan.npairs;
  if (pairs_out) {
    if (max_pairs < plan.npairs) return fail(TNB_EINVAL, "bs_contract: pairs_out too small");
    // bookkeeping readback: CSR grouped by output block -> reference order (i asc, j asc)
    std::vector<int32_t> optr(nout + 1);
    int32_t err = 0;
    TNB_CUDA_CHECK(cudaMemcpyAsync(optr.data(), plan.dblob + plan.o_optr, (size_t)(nout + 1) * 4,
                                   cudaMemcpyDeviceToHost, st));
    TNB_CUDA_CHECK(cudaMemcpyAsync(&err, meta.err, 4, cudaMemcpyDeviceToHost, st));
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

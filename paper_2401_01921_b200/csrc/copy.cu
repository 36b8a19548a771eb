// Batched strided byte copies (tnb_copy2d_batched): the data mover behind the
// block-slab <-> packed-payload conversions of the .utn container
// (pkg/src/tnkit/io.py:56-107: payload = every block's C-order bytes,
// concatenated in block order) and the block <-> sector-matrix scatters of the
// block-sparse matricisation (linalg.py:70-142).
//
// One launch moves every segment: the (segment, row) space is flattened and
// walked by warps; each warp copies one row with the widest aligned vector
// (16/8/4/1 bytes) the row's addresses allow; rows longer than 4 KB are split into 4 KB
// pieces so that a few long rows (packed block payloads) still spread over the whole GPU.
// HBM-bound: 2 x bytes moved.
#include <algorithm>
#include <vector>

#include <cstring>

#include "common.cuh"

namespace tnb {
namespace {

constexpr int kInlineSegs = 256;
constexpr int64_t kChunkBytes = 4096;  // work unit: one 4 KB piece of one row (long rows spread over warps)

struct SegTable {
  TnbCopy2D s[kInlineSegs];
  int64_t row0[kInlineSegs + 1];  // prefix sums of work units (rows x 4 KB pieces)
};

template <typename V>
__device__ __forceinline__ void copy_row(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst,
                                         int64_t bytes, int lane) {
  const int64_t n = bytes / (int64_t)sizeof(V);
  const V* s = reinterpret_cast<const V*>(src);
  V* d = reinterpret_cast<V*>(dst);
#pragma unroll 4
  for (int64_t i = lane; i < n; i += 32) d[i] = s[i];
}

__global__ void __launch_bounds__(256) copy2d_kernel(const unsigned char* __restrict__ src,
                                                     unsigned char* __restrict__ dst, int nseg,
                                                     const __grid_constant__ SegTable tab,
                                                     const TnbCopy2D* __restrict__ gsegs,
                                                     const int64_t* __restrict__ grow0) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const TnbCopy2D* segs = gsegs ? gsegs : tab.s;
  const int64_t* row0 = grow0 ? grow0 : tab.row0;
  const int64_t total = row0[nseg];
  int seg = 0;
  for (int64_t r = warp; r < total; r += nwarps) {
    // rows are visited in increasing order by each warp: advance (or search) the segment
    if (r >= row0[seg + 1] || r < row0[seg]) {
      int lo = 0, hi = nseg - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (row0[mid] <= r) lo = mid;
        else hi = mid - 1;
      }
      seg = lo;
    }
    const TnbCopy2D g = segs[seg];
    const int64_t cpr = (g.row_bytes + kChunkBytes - 1) / kChunkBytes;  // pieces per row
    const int64_t u = r - row0[seg];
    const int64_t k = u / cpr, piece = u - k * cpr;
    const int64_t b0 = piece * kChunkBytes;
    const int64_t bytes = (g.row_bytes - b0) < kChunkBytes ? (g.row_bytes - b0) : kChunkBytes;
    const unsigned char* s = src + g.src_off + k * g.src_pitch + b0;
    unsigned char* d = dst + g.dst_off + k * g.dst_pitch + b0;
    const uintptr_t al = reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d) | (uintptr_t)bytes;
    if ((al & 15) == 0) copy_row<uint4>(s, d, bytes, lane);
    else if ((al & 7) == 0) copy_row<uint2>(s, d, bytes, lane);
    else if ((al & 3) == 0) copy_row<uint32_t>(s, d, bytes, lane);
    else copy_row<unsigned char>(s, d, bytes, lane);
  }
}

}  // namespace
}  // namespace tnb

extern "C" int tnb_copy2d_batched(const void* src, void* dst, int64_t nseg, const TnbCopy2D* segs, void* stream) {
  using namespace tnb;
  int rc = require_device();
  if (rc) return rc;
  if (nseg < 0 || (nseg > 0 && (!segs || !src || !dst))) return fail(TNB_EINVAL, "copy2d: bad arguments");
  if (nseg == 0) return TNB_OK;
  if (nseg >= (1ll << 31)) return fail(TNB_EUNSUP, "copy2d: too many segments");
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int64_t> row0((size_t)nseg + 1, 0);
  double bytes = 0.0;
  for (int64_t i = 0; i < nseg; ++i) {
    const TnbCopy2D& g = segs[i];
    if (g.rows < 0 || g.row_bytes < 0 || g.src_off < 0 || g.dst_off < 0)
      return fail(TNB_EINVAL, "copy2d: negative extent or offset");
    row0[i + 1] = row0[i] + (g.row_bytes > 0 ? g.rows * ((g.row_bytes + kChunkBytes - 1) / kChunkBytes) : 0);
    bytes += 2.0 * (double)g.rows * (double)g.row_bytes;
  }
  const int64_t total = row0[nseg];
  if (total == 0) return TNB_OK;
  SegTable* tab = new SegTable;  // 20 KB: keep it off the stack
  TnbCopy2D* gsegs = nullptr;
  int64_t* grow0 = nullptr;
  void* dmem = nullptr;
  if (nseg <= kInlineSegs) {
    std::copy(segs, segs + nseg, tab->s);
    std::copy(row0.begin(), row0.end(), tab->row0);
  } else {
    const size_t sb = sizeof(TnbCopy2D) * (size_t)nseg, rb = sizeof(int64_t) * ((size_t)nseg + 1);
    // eager: pageable sources are staged before cudaMemcpyAsync returns. Under capture the
    // memcpy node re-reads its source at every replay, so the table goes to pinned memory
    // owned by the graph.
    const void* src_tab = nullptr;
    std::vector<unsigned char> packed;
    if (capturing(st)) {
      void* pin = nullptr;
      int rc2 = capture_pinned(st, sb + rb, &pin);
      if (rc2) {
        delete tab;
        return rc2;
      }
      src_tab = pin;
    } else {
      release_deferred_host();
      packed.resize(sb + rb);
      src_tab = packed.data();
    }
    memcpy(const_cast<void*>(src_tab), segs, sb);
    memcpy(static_cast<char*>(const_cast<void*>(src_tab)) + sb, row0.data(), rb);
    cudaError_t e = cudaMallocAsync(&dmem, sb + rb, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dmem, src_tab, sb + rb, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) {
      delete tab;
      return cuda_fail(e, "copy2d: segment table upload");
    }
    gsegs = static_cast<TnbCopy2D*>(dmem);
    grow0 = reinterpret_cast<int64_t*>(static_cast<char*>(dmem) + sb);
  }
  const int64_t warps = std::min<int64_t>(total, (int64_t)sm_count() * 64);
  const int grid = (int)std::max<int64_t>(1, (warps + 7) / 8);
  {
    KTimer kt(TNB_KF_OTHER, st, bytes);
    copy2d_kernel<<<grid, 256, 0, st>>>(static_cast<const unsigned char*>(src), static_cast<unsigned char*>(dst),
                                        (int)nseg, *tab, gsegs, grow0);
  }
  count_launch();
  cudaError_t e = cudaGetLastError();
  delete tab;
  if (dmem) cudaFreeAsync(dmem, st);
  if (e != cudaSuccess) return cuda_fail(e, "copy2d: launch");
  return TNB_OK;
}

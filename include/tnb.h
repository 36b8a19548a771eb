/*
 * tnb.h -- C ABI of libtnb.so, the B200 (sm_100a) engine for the tensor-operation
 * hot path of the reference `tnkit` package (arxiv 2401.01921, Cytnx paper).
 *
 * The reference is pure Python; its hot path reaches numpy/OpenBLAS at exactly
 * these call sites, which are the seams this ABI replaces:
 *
 *   tnb_permute            <- np.ascontiguousarray(self.view())
 *                             pkg/src/tnkit/storage.py:122 (contiguous),
 *                             storage.py:126 (contiguous_), storage.py:143 (reshape)
 *   tnb_contract_dense     <- np.tensordot(a.view(), b.view(), axes=(a_pos, b_pos))
 *                             + np.ascontiguousarray(res)
 *                             pkg/src/tnkit/contract.py:127-132 (contract_pair, dense)
 *   tnb_bs_contract[_masked]
 *                          <- _contract_pair_blocks, pkg/src/tnkit/contract.py:137-167
 *                             (b_by_key pairing :148-151, per-pair tensordot :157-158,
 *                              ordered += into the output block :162-164)
 *   tnb_zero_flux_blocks   <- _zero_flux_combos, pkg/src/tnkit/unitensor.py:31-45
 *   tnb_optimal_order      <- find_optimal_order, pkg/src/tnkit/contract.py:271-343
 *
 * Conventions (mirroring the reference's error behaviour, README.md:112-114):
 *   - every entry point returns int status: 0 = TNB_OK, otherwise an error code;
 *     tnb_last_error() returns a thread-local message for the last failure.
 *   - structure is validated by the host layer before these calls (ValueError /
 *     TypeError are raised in Python before any arithmetic, contract.py:107-123);
 *     the ABI re-checks what it needs for memory safety and returns
 *     TNB_EINVAL rather than faulting.
 *   - the caller allocates every output buffer; the library never frees caller
 *     memory. Device pointers are plain CUDA device pointers; `stream` is a
 *     cudaStream_t (NULL = legacy default stream). All device work is
 *     asynchronous on `stream`.
 *   - tensors are described in the reference's storage model (storage.py:40-57):
 *     a C-contiguous buffer with storage shape `shape[0..rank)` and a logical
 *     permutation `perm` (logical axis k lives on storage axis perm[k]).
 *   - no CPU fallback: compute entry points return TNB_ENODEV without a GPU.
 */
#ifndef TNB_H_
#define TNB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TNB_MAX_RANK 16

/* status codes */
#define TNB_OK 0
#define TNB_EINVAL 1   /* bad argument (shape, perm, dtype, sizes) */
#define TNB_ECUDA 2    /* CUDA runtime error (launch / async fault) */
#define TNB_ENODEV 3   /* no CUDA device */
#define TNB_ENOMEM 4   /* workspace allocation failed */
#define TNB_EUNSUP 5   /* unsupported dtype / feature (no fallback path) */

/* dtype codes (storage.py:15-20); contraction supports F64 and C128 only */
#define TNB_F64 0
#define TNB_C128 1
#define TNB_I64 2
#define TNB_BOOL 3

/* complex GEMM formulation */
#define TNB_CPLX_4M 0  /* four real DMMA products per complex MAC (exact 4M) */
#define TNB_CPLX_3M 1  /* Gauss/Karatsuba 3M: three real products           */

/* ---- library / device -------------------------------------------------- */
int tnb_version(void);                       /* ABI version, e.g. 100 */
int64_t tnb_launch_count(void);              /* kernels launched by libtnb so far (process-wide) */
const char* tnb_last_error(void);            /* thread-local, never NULL */
int tnb_device_count(int* count);            /* 0 devices is not an error */
int tnb_set_device(int device);
int tnb_synchronize(void* stream);           /* waits; surfaces async faults */
/* 2-D strided copy (cudaMemcpy2DAsync; kind: 1 H2D, 2 D2H, 3 D2D): streams a column
 * panel of a row-major result to (pinned) host memory while later panels compute. */
int tnb_memcpy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch,
                       int64_t width, int64_t height, int kind, void* stream);

/* ---- kernel timer (measurement; bench.py's roofline) ----------------------
 * While enabled, every libtnb kernel launch outside stream capture records a
 * CUDA event pair on the stream it is launched on, plus its algorithmic work
 * (flop for contractions: 2 per real MAC, 8 per complex MAC; bytes read +
 * written for permutes; 0 where the host does not know it).
 * tnb_ktimer_read sums launches, device milliseconds and work of one family
 * since the last reset (it waits for the recorded events). */
#define TNB_KF_GEMM 0        /* stream-K DMMA GEMM (dense contraction)        */
#define TNB_KF_GEMM_SKINNY 1 /* memory-bound narrow/skinny contraction kernels */
#define TNB_KF_PERMUTE 2     /* permute materialisation kernels              */
#define TNB_KF_BS_GEMM 3     /* block-sparse grouped GEMM                    */
#define TNB_KF_BS_PAIR 4     /* block-sparse device pairing                  */
#define TNB_KF_OTHER 5       /* widening, split-K reduce, ...                */
int tnb_ktimer_enable(int on);
int tnb_ktimer_reset(void);
int tnb_ktimer_read(int family, int64_t* launches, double* ms, double* work);

/* ---- a7: permute materialisation (storage.py:114-144) ---------------------
 * dst[row-major over logical shape] = src viewed with storage shape `shape`
 * and logical permutation `perm`; bit-exact data movement for element sizes
 * 1, 2, 4, 8, 16 bytes. src and dst must not overlap. */
int tnb_permute(const void* src, void* dst, int elem_size, int rank,
                const int64_t* shape, const int32_t* perm, void* stream);

/* ---- a11: dense pairwise contraction (contract.py:100-134) ----------------
 * out[a_free..., b_free...] = sum_{shared} A[...] * B[...]
 *   a_* / b_* : storage shape + perm of each operand (lazy permutes are read
 *               in place, never materialised)
 *   nc, a_axes[nc], b_axes[nc]: LOGICAL axes contracted pairwise, in the
 *               order of the shared labels (a's order, contract.py:112-114)
 *   dtype_a/b : TNB_F64 or TNB_C128; out dtype = result_type (C128 if any)
 *   out       : C-contiguous, shape = a_free dims then b_free dims
 *   cplx_mode : TNB_CPLX_4M or TNB_CPLX_3M (ignored for real)
 * Returns TNB_EUNSUP for I64/BOOL (the reference accepts them; the engine
 * has no CPU fallback and says so). */
int tnb_contract_dense(const void* a, int dtype_a, int rank_a,
                       const int64_t* shape_a, const int32_t* perm_a,
                       const void* b, int dtype_b, int rank_b,
                       const int64_t* shape_b, const int32_t* perm_b,
                       int nc, const int32_t* a_axes, const int32_t* b_axes,
                       void* out, int cplx_mode, void* stream);

/* ---- batched strided copies (block slab <-> packed payload / sector matrix)
 * For every segment: rows x row_bytes bytes from src + src_off (row pitch
 * src_pitch) to dst + dst_off (row pitch dst_pitch). Offsets and pitches are in
 * bytes relative to the two base pointers; segments must not overlap in dst.
 * One launch; vector width chosen per row from the alignment. Used by the
 * .utn container I/O (io.py:56-107 payload = blocks' C-order bytes in block
 * order) and the block-sparse matricisation (linalg.py:70-142). */
typedef struct {
  int64_t src_off, dst_off, rows, row_bytes, src_pitch, dst_pitch;
} TnbCopy2D;
int tnb_copy2d_batched(const void* src, void* dst, int64_t nseg, const TnbCopy2D* segs, void* stream);

/* ---- file payload -> HBM (the .utn loader, io.py:83-107's payload read) ----
 * nbytes bytes of the open file fd from byte offset `offset` are read with pread() by up to
 * nthreads threads (the caller's included) in `chunk`-byte pieces into the PINNED host
 * buffer `pinned` (>= nbytes), and each piece is copied to dst (device) with
 * cudaMemcpyAsync on `stream` as soon as it and every earlier piece have landed. Returns
 * once every read is done and every copy is queued; the caller must keep `pinned`
 * untouched until the copies complete (an event on `stream`). TNB_EINVAL on a short read. */
int tnb_file_to_device(int fd, int64_t offset, int64_t nbytes, void* pinned, void* dst, int64_t chunk,
                       int nthreads, void* stream);

/* ---- one Lanczos orthogonalisation step (linalg.py:474-562 vector work) ----
 * q: r basis vectors as ROWS (row pitch ldq elements), w: the matvec result (n elements,
 * overwritten by w - sum_k <q_k, w> q_k), q_next: receives w / |w| (may be NULL);
 * *alpha = Re <q_{r-1}, w> and *beta = |w| are written to DEVICE memory (no host sync).
 * r = 0: only normalises w into q_next. work: tnb_lanczos_work_bytes(r_max, n) bytes,
 * zeroed before first use (the step leaves its counters zeroed). float64 / complex128. */
int64_t tnb_lanczos_work_bytes(int r_max, int64_t n);
int tnb_lanczos_step(int dtype, const void* q, int64_t ldq, int r, void* w, int64_t n, void* q_next,
                     double* alpha, double* beta, void* work, void* stream);

/* ---- batched one-sided Jacobi SVD of sector matrices (linalg.py:246-341) ---
 * Each sector: A (m x n, 1 <= m <= n, row-major, dtype TNB_F64 or TNB_C128; s is
 * float64 either way) in `a` (read only), workspaces b (m x ldb) and q (m x ldq)
 * with ldb = n, ldq = m for complex128 and both rounded up to even for float64
 * (16-byte rows); outputs the thin factors in torch/LAPACK layout
 * u (m x m row-major), s (m, descending), vh (m x n row-major) and *status:
 * sweeps used (> 0) or -1 (not converged within max_sweeps). Rank-deficient
 * sectors (singular values <= rank_tol * max) are handled in the kernel: their
 * vh rows are completed to an orthonormal basis of the complement of the kept
 * rows (two-pass Gram-Schmidt), as LAPACK completes V. A row pair is rotated while
 * |b_p.b_q| > tol * sqrt(n) * eps * |b_p||b_q| (eps = 2^-52).
 * One thread-block cluster per sector, all sectors in one launch. */
typedef struct {
  void *a, *b, *q, *u, *s, *vh;
  int32_t* status;
  int64_t m, n;
} TnbSvdSector;
int tnb_svd_jacobi_batched(int dtype, int nsec, const TnbSvdSector* secs, int max_sweeps, double tol,
                           double rank_tol, void* stream);

/* Same contraction writing a column panel of a wider row-major output: row i of
 * the result lands at out + i * out_ld (out_ld >= the result's column count;
 * 0 = packed). Used to pipeline a contraction with the chunked host upload of
 * its right operand (each chunk of b's outermost free axis = one column panel). */
int tnb_contract_dense_ld(const void* a, int dtype_a, int rank_a,
                          const int64_t* shape_a, const int32_t* perm_a,
                          const void* b, int dtype_b, int rank_b,
                          const int64_t* shape_b, const int32_t* perm_b,
                          int nc, const int32_t* a_axes, const int32_t* b_axes,
                          void* out, int64_t out_ld, int cplx_mode, void* stream);

/* Same contraction writing the output in a chosen PHYSICAL axis order: out_order[p] is the
 * logical output axis (a_free..., b_free...) stored at physical position p (row-major over
 * the physical order); NULL = the logical order (tnb_contract_dense). The result is read
 * back as a lazily permuted tensor. Network launches use it to lay an intermediate out
 * K-major for the long-K contraction that consumes it (network.py:213-244 semantics are
 * unchanged: only the storage order of an intermediate differs). */
int tnb_contract_dense_out(const void* a, int dtype_a, int rank_a,
                           const int64_t* shape_a, const int32_t* perm_a,
                           const void* b, int dtype_b, int rank_b,
                           const int64_t* shape_b, const int32_t* perm_b,
                           int nc, const int32_t* a_axes, const int32_t* b_axes,
                           void* out, const int32_t* out_order, int cplx_mode, void* stream);

/* ---- a3: zero-flux block enumeration (unitensor.py:31-45), host only ------
 * Bonds are given as flattened charge tables:
 *   nbonds, nsyms; nsec[b]; btype[b] (+1 IN, -1 OUT);
 *   charges: for bond b, sector s, symmetry y at
 *            charges[(sec_off[b] + s) * nsyms + y], sec_off = prefix sum of nsec
 *   sym_n[y]: 0 for U(1), n for Z_n
 * Writes up to max_out tuples (row-major enumeration, first bond outermost)
 * into out_qn[count * nbonds] and sets *count to the total number found
 * (call with max_out = 0 to size). */
int tnb_zero_flux_blocks(int nbonds, int nsyms, const int32_t* nsec,
                         const int32_t* btype, const int64_t* charges,
                         const int32_t* sym_n, int64_t max_out,
                         int32_t* out_qn, int64_t* count);

/* ---- a12: U(1)/Z_n block-sparse pairwise contraction (contract.py:137-167)
 * Block metadata is uploaded once per block STRUCTURE (device-resident plan
 * cache); pairing is computed ON DEVICE:
 *   for i in a-block order, for j ascending with key(b_j) == key(a_i):
 *       out[out_idx(i,j)] += A_i . B_j
 * The k-iterations of all output tiles (each tile's pairs concatenated in that
 * order) are split evenly over one persistent CTA per SM (grouped stream-K);
 * a tile split across CTAs is finished by the CTA holding its last k-iteration,
 * which adds the earlier partials in CTA order: deterministic, no atomics.
 *
 * Plan (host -> device):
 *   na, nb, nout      : block counts
 *   rank_a, rank_b    : tensor ranks (every block shares them)
 *   a_qn[na*rank_a], b_qn[nb*rank_b]: qn-index tuples per block (logical order)
 *   a_shape[na*rank_a], b_shape[nb*rank_b]: block STORAGE shapes
 *   a_perm[rank_a], b_perm[rank_b]: the common lazy permutation of the blocks
 *   nc, a_axes, b_axes: contracted logical axes
 *   out_qn[nout*rank_out]: output block qn tuples (zero-flux enumeration)
 *   out_shape[nout*rank_out]: output block shapes
 * Data: a_ptrs[na], b_ptrs[nb], out_ptrs[nout] device pointers (host arrays);
 *       every output block is fully overwritten (blocks without pairs are zeroed).
 * Returns the number of pairs in *npairs. If pairs_out != NULL it must hold
 * 3*max_pairs int32 and receives (i, j, out_idx) triples in reference order
 * (copied back from the device table) for bit-exact bookkeeping checks. */
int tnb_bs_contract(int dtype, int na, int nb, int nout,
                    int rank_a, int rank_b,
                    const int32_t* a_qn, const int64_t* a_shape, const int32_t* a_perm,
                    const int32_t* b_qn, const int64_t* b_shape, const int32_t* b_perm,
                    int nc, const int32_t* a_axes, const int32_t* b_axes,
                    const int32_t* out_qn, const int64_t* out_shape,
                    const void* const* a_ptrs, const void* const* b_ptrs,
                    void* const* out_ptrs,
                    int64_t max_pairs, int32_t* pairs_out, int64_t* npairs,
                    void* stream);

/* Multi-GPU partition of a block-sparse contraction: the output is cut into
 * "panels" of TNB_BS_PANEL_ROWS rows (rows = the a_free part of each output
 * block), enumerated block by block in output-block order. With panel_mask !=
 * NULL only panels whose mask byte is non-zero are computed and written (each
 * panel's full K reduction is local: no cross-GPU reduction); the caller
 * assembles the rest (parallel.py: NCCL all-gather). npanels must equal the
 * panel count. Same semantics as tnb_bs_contract otherwise. */
#define TNB_BS_PANEL_ROWS 64
int tnb_bs_contract_masked(int dtype, int na, int nb, int nout,
                           int rank_a, int rank_b,
                           const int32_t* a_qn, const int64_t* a_shape, const int32_t* a_perm,
                           const int32_t* b_qn, const int64_t* b_shape, const int32_t* b_perm,
                           int nc, const int32_t* a_axes, const int32_t* b_axes,
                           const int32_t* out_qn, const int64_t* out_shape,
                           const void* const* a_ptrs, const void* const* b_ptrs,
                           void* const* out_ptrs, int64_t npanels, const uint8_t* panel_mask,
                           int64_t max_pairs, int32_t* pairs_out, int64_t* npairs,
                           void* stream);

/* Split form of the same operation for repeated calls on one block STRUCTURE
 * (a Lanczos loop, a sweep over equal-structure sites): tnb_bs_plan builds --
 * or finds in the device-resident plan cache -- the plan of a structure (same
 * arguments as tnb_bs_contract_masked minus the data; panel_mask may be NULL)
 * and returns an opaque id; tnb_bs_execute launches the grouped GEMM for one
 * set of block pointers; tnb_bs_plan_pairs reads back the (i, j, out_idx)
 * triples. Ids become stale (TNB_EINVAL) when the cache is flushed (>256
 * structures or a device change): re-plan then. */
int tnb_bs_plan(int dtype, int na, int nb, int nout, int rank_a, int rank_b,
                const int32_t* a_qn, const int64_t* a_shape, const int32_t* a_perm,
                const int32_t* b_qn, const int64_t* b_shape, const int32_t* b_perm,
                int nc, const int32_t* a_axes, const int32_t* b_axes,
                const int32_t* out_qn, const int64_t* out_shape,
                int64_t npanels, const uint8_t* panel_mask,
                int64_t* plan_id, int64_t* npairs, void* stream);
int tnb_bs_execute(int64_t plan_id, const void* const* a_ptrs, const void* const* b_ptrs,
                   void* const* out_ptrs, void* stream);
int tnb_bs_plan_pairs(int64_t plan_id, int64_t max_pairs, int32_t* pairs_out, int64_t* npairs,
                      void* stream);
/* nbatch independent contractions of ONE plan's structure (e.g. the equal-structure
 * sites of a sweep) in one grouped stream-K launch over all their output tiles:
 * a_ptrs[nbatch][na], b_ptrs[nbatch][nb], out_ptrs[nbatch][nout] (row-major). Each
 * contraction's result is the one tnb_bs_execute gives (same per-tile pair order). Not
 * for panel-masked plans (TNB_EUNSUP). No reference counterpart: contract.py:137-167
 * runs one pair at a time; this is the batched form of the same arithmetic. */
int tnb_bs_execute_batched(int64_t plan_id, int64_t nbatch, const void* const* a_ptrs,
                           const void* const* b_ptrs, void* const* out_ptrs, void* stream);

/* ---- a14: optimal contraction order DP (contract.py:271-343), host only ---
 * n tensors (n <= 16). Labels are interned to ints: nlab[t] labels for tensor
 * t at labels[lab_off[t] ..], dims[label_id] their dimensions (int64).
 * names_rank[t]: rank of tensor t's name in the lexicographic order of the
 * rendered strings' alphabet -- the host passes the names themselves:
 * names = concatenated NUL-terminated strings.
 * Output: the rendered order string "((A,B),C)" into out[cap]; *cost the
 * total cost as a decimal string (costs may exceed 64 bits) in cost_out[64].*/
int tnb_optimal_order(int n, const char* names, const int32_t* nlab,
                      const int32_t* labels, const int64_t* dims,
                      char* out, int64_t cap, char* cost_out);

#ifdef __cplusplus
}
#endif
#endif /* TNB_H_ */

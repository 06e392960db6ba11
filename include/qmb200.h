/*
 * qmb200.h -- C ABI of the B200 block-sparse quadtree multiply (libqmb200.so).
 *
 * The reference (arXiv 2011.11762, Python package `quadmat` under pkg/src/quadmat) has no
 * native code and no FFI; its multiply is the recursive task graph
 *   MatrixSession.multiply        session.py:160-171
 *   -> ops.multiply_spec          ops.py:582-608
 *   -> "multiply" task body       ops.py:197-245   (+ "add" ops.py:147-169, "assemble" ops.py:134-139)
 *   -> BlockSparseLeaf.multiply   leaves/block_sparse.py:112-132 (numpy dgemm per block triple)
 * Each entry point below replaces one layer of that stack; the per-function comment names it.
 * A maintainer binding this library from the reference would load it with ctypes and call the
 * functions from a replacement "multiply" task body.
 *
 * Conventions
 *  - All pointers marked (device) are CUDA device pointers owned by the caller; the library never
 *    allocates or frees caller memory and never returns owned allocations. Scratch comes from a
 *    caller-provided workspace (size queried with the *_workspace_bytes functions).
 *  - Every call is stream-ordered on the caller's stream (a cudaStream_t passed as void*; NULL is
 *    the legacy default stream). Only qm_spgemm_count synchronises (it returns sizes to the host).
 *  - Return value: QM_OK (0) or a negative QM_ERR_* code; qm_last_error() returns a thread-local
 *    message for the last failure on the calling thread.
 *  - The library is reentrant: no mutable globals other than the thread-local error string and a
 *    relaxed launch counter.
 *
 * Data layout ("quadtree key" order)
 *  A matrix is nnzb dense bs x bs float64 blocks, row-major (the BlockSparseLeaf block payload,
 *  block_sparse.py:226-231), stored contiguously in ascending order of their uint64 quadtree key
 *      qkey(bi, bj) = morton(bi / nbl, bj / nbl) << (2*lbits) | (bi % nbl) << lbits | (bj % nbl)
 *  where nbl = leaf_dim / bs blocks per leaf side, lbits = ceil(log2(nbl)), and morton() interleaves
 *  the leaf-grid coordinates with the row bit high (NW, NE, SW, SE = quadtree.py:128-129). That is
 *  exactly the order in which canonical_bytes (quadtree.py:293-318) visits the blocks: depth-first
 *  over the tree, then BlockSparseLeaf.encode's sorted (bi, bj) order inside a leaf.
 */
#ifndef QMB200_H
#define QMB200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define QM_API __attribute__((visibility("default")))
#else
#define QM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define QM_ABI_VERSION 2 /* 2: support masks are uint64[3*n] (rows, columns, flags) */

enum qm_status {
  QM_OK = 0,
  QM_ERR_INVALID = -1,     /* bad argument / nonconformant operands (DimensionMismatch, Configuration) */
  QM_ERR_CUDA = -2,        /* a CUDA runtime call or kernel launch failed */
  QM_ERR_WORKSPACE = -3,   /* caller workspace smaller than the queried size */
  QM_ERR_UNSUPPORTED = -4, /* block size / layout not supported by this build */
};

/* Geometry of one quadtree matrix: MatrixParams (quadtree.py:24-44) + BlockSparseLeaf.block_size. */
typedef struct qm_layout {
  int64_t n_logical; /* MatrixParams.n_logical */
  int32_t leaf_dim;  /* MatrixParams.leaf_dim; must be a multiple of block_size */
  int32_t depth;     /* MatrixParams.depth (leaf_dim << depth >= n_logical) */
  int32_t block_size;/* BlockSparseLeaf.block_size */
  int32_t reserved;  /* must be 0 */
} qm_layout;

/* ---- library info --------------------------------------------------------------------------- */
QM_API int qm_abi_version(void);
QM_API const char *qm_last_error(void);
/* Number of kernels this library has launched in this process (relaxed counter; for bench). */
QM_API uint64_t qm_launch_count(void);

/* Reads n (1..8) int64 values from device memory to host memory through a mapped pinned buffer
 * written by a kernel on `stream` (no copy engine, so it never queues behind large in-flight
 * copies), then synchronises `stream`. Used for the small counts the host needs. */
QM_API int qm_read_i64(const int64_t *dev_src /*device*/, int32_t n, int64_t *host_out /*host*/,
                       void *stream);

/* ---- quadtree keys ---------------------------------------------------------------------------- */
/* Replaces the quadrant recursion of build_from_triplets (quadtree.py:112-142) for block placement:
 * keys[i] = qkey(bi[i], bj[i]) on the device. */
QM_API int qm_encode_keys(const qm_layout *layout, const int32_t *bi /*device*/, const int32_t *bj /*device*/,
                   int64_t n, uint64_t *keys /*device*/, void *stream);
/* Inverse: (bi, bj) block coordinates of each key. */
QM_API int qm_decode_keys(const qm_layout *layout, const uint64_t *keys /*device*/, int64_t n,
                   int32_t *bi /*device*/, int32_t *bj /*device*/, void *stream);

/* ---- construction (replaces build_from_triplets + BlockSparseLeaf.from_triplets,
 *      quadtree.py:90-142, block_sparse.py:47-68) ---------------------------------------------- */
QM_API size_t qm_build_workspace_bytes(const qm_layout *layout, int64_t n_entries);
/* Sorts the entries by (block quadtree key, position in block), stably, and counts the distinct
 * blocks touched. Entries outside [0, n_logical) are counted in *n_out_of_range (host) and nothing
 * else is done (the caller raises OutOfRangeError). Synchronises `stream`. */
QM_API int qm_build_count(const qm_layout *layout, const int64_t *rows /*device*/,
                          const int64_t *cols /*device*/, int64_t n, void *ws, size_t ws_bytes,
                          int64_t *n_blocks_out /*host*/, int64_t *n_out_of_range /*host*/, void *stream);
/* Sums duplicate entries in input order starting from +0.0 (np.add.at), writes keys[n_blocks],
 * blocks[n_blocks,bs,bs], sumsq, nonzero flags and counts exactly-zero blocks in *zero_count
 * (device; the caller zeroes it first and compacts with qm_compact when it is nonzero). */
QM_API int qm_build_fill(const qm_layout *layout, const double *vals /*device*/, int64_t n, void *ws,
                         size_t ws_bytes, int64_t n_blocks, uint64_t *keys, double *blocks,
                         double *sumsq, uint8_t *nonzero, int64_t *zero_count, void *stream);
/* qm_build_fill that also writes the blocks' support masks (uint64[3*n_blocks], qm_block_meta's
 * layout; NULL = none) and OR-accumulates the not-full flags into not_full[2] (device, zeroed by
 * the caller; NULL = none) in the same pass over the filled blocks that computes the norms. */
QM_API int qm_build_fill_meta(const qm_layout *layout, const double *vals /*device*/, int64_t n, void *ws,
                              size_t ws_bytes, int64_t n_blocks, uint64_t *keys, double *blocks,
                              double *sumsq, uint8_t *nonzero, int64_t *zero_count, uint64_t *masks,
                              int64_t *not_full, void *stream);

/* ---- symbolic phase (replaces the recursive task expansion, ops.py:197-245 + engine.py:196-326) */
/* Persistent workspace for one product; valid from qm_spgemm_count until qm_spgemm_fill returns. */
QM_API size_t qm_spgemm_workspace_bytes(const qm_layout *layout, int64_t nA, int64_t nB);
/* Builds block-row indexes of A and B inside ws, counts the C blocks of the symbolic product
 * (every (i,j) with some k such that A(i,k) and B(k,j) are stored) and the product triples.
 * Synchronises `stream` and writes the two counts to host memory. */
QM_API int qm_spgemm_count(const qm_layout *layout, const uint64_t *a_keys /*device, sorted*/, int64_t nA,
                    const uint64_t *b_keys /*device, sorted*/, int64_t nB, void *ws, size_t ws_bytes,
                    int64_t *n_c_out /*host*/, int64_t *n_triples_out /*host*/, void *stream);
/* qm_spgemm_count with per-block support masks (NULL = full support): a_cmask[t] / b_rmask[t] are
 * the nonzero-column mask of A block t and the nonzero-row mask of B block t (qm_block_masks). A
 * pair whose masks share no bit multiplies to an exactly-zero block: it yields no triple, and a C
 * block without any surviving triple is not created (it would be an exact-zero block, which
 * _set_block, block_sparse.py:37-41, drops). The fill calls of the same workspace use the masks too.
 * flags & QM_SPGEMM_UPPER: only the C blocks of leaves (li, lj) with li <= lj are enumerated -- the
 * reference's symmetric_square / rank_k never spawn the SW products of diagonal-path nodes
 * (ops.py:214-216). */
#define QM_SPGEMM_UPPER 1 /* flags: only C blocks of leaves (li, lj) with li <= lj (the `upper` variants) */
QM_API int qm_spgemm_count_masked(const qm_layout *layout, const uint64_t *a_keys, const uint64_t *a_cmask,
                                  int64_t nA, const uint64_t *b_keys, const uint64_t *b_rmask, int64_t nB,
                                  int32_t flags, void *ws, size_t ws_bytes, int64_t *n_c_out,
                                  int64_t *n_triples_out, void *stream);
/* The symbolic count of ONE rank of a multi-GPU product (the reference's per-worker task
 * expansion: each worker only expands the tasks it owns, ops.py:197-241 / engine.py:286-300).
 * A cheap global pass over the (all-gathered) structure counts the structural triples of every C
 * tile -- an aligned quadtree subtree, 4^min(depth, 8) of them in Morton order -- at O(nA) cost;
 * the tiles are cut into `world` contiguous ranges of nearly equal work, and this rank's C key range
 * [part_out[0], part_out[1]) is a union of whole subtrees (the ranks' ranges tile the key space in
 * rank order). Only C blocks inside the range are counted here and emitted by the fill calls of the
 * same workspace (keys, offsets and triples local to the rank). part_out (host int64[3]): key range
 * and the total tile work; key_cuts (device uint64[world+1], may be NULL): every rank's range bound.
 * Support masks as in qm_spgemm_count_masked. Synchronises the stream once. */
QM_API int qm_spgemm_count_part(const qm_layout *layout, const uint64_t *a_keys, const uint64_t *a_cmask,
                                int64_t nA, const uint64_t *b_keys, const uint64_t *b_rmask, int64_t nB,
                                int32_t world, int32_t rank, void *ws, size_t ws_bytes, int64_t *n_c_out,
                                int64_t *n_triples_out, int64_t *part_out, uint64_t *key_cuts, void *stream);
/* Row index of one operand (operand metadata, like its norms and masks: built once per block set
 * by qm_row_index_build and kept with it): the block set's entries sorted by (row, column) -- positions
 * `perm`, rows, columns, row pointers [nbg+1] -- plus the support mask each sorted entry brings to a
 * product (the block's column mask when it is the left operand, its row mask as the right one).
 * With it the symbolic phase skips its own row indexing (the decode + radix sort of qm_spgemm_count). */
typedef struct qm_row_index {
  const uint32_t *rowptr; /* device [nbg + 1] */
  const uint32_t *row;    /* device [n] */
  const uint32_t *col;    /* device [n] */
  const uint32_t *perm;   /* device [n]: index of the sorted entry in the block set */
  const uint64_t *mask;   /* device [n] or NULL (full supports); both operands' or neither */
} qm_row_index;
QM_API size_t qm_row_index_workspace_bytes(const qm_layout *layout, int64_t n);
/* masks: the block set's [3, n] support masks or NULL; cmask_sorted / rmask_sorted (optional, [n]):
 * its column / row masks in row-sorted order (the left / right operand roles). */
QM_API int qm_row_index_build(const qm_layout *layout, const uint64_t *keys, int64_t n, const uint64_t *masks, void *ws,
                        size_t ws_bytes, uint32_t *rowptr, uint32_t *row, uint32_t *col, uint32_t *perm,
                        uint64_t *cmask_sorted, uint64_t *rmask_sorted, void *stream);
/* qm_spgemm_count_masked / _part over caller-held row indexes (world = 0: the whole product;
 * world >= 1: rank's share, part_out / key_cuts as qm_spgemm_count_part). Same workspace. */
QM_API int qm_spgemm_count_ix(const qm_layout *layout, const qm_row_index *a, int64_t nA, const qm_row_index *b,
                              int64_t nB, int32_t flags, int32_t world, int32_t rank, void *ws, size_t ws_bytes,
                              int64_t *n_c_out, int64_t *n_triples_out, int64_t *part_out, uint64_t *key_cuts,
                              void *stream);
/* Fill after qm_spgemm_count_ix: C keys + c_tptr (c_keys non-NULL) and/or triples [t_lo, t_hi) (tri
 * non-NULL), with the same row indexes and workspaces. */
QM_API int qm_spgemm_fill_ix(const qm_layout *layout, const qm_row_index *a, int64_t nA, const qm_row_index *b,
                             int64_t nB, int64_t nC, int64_t t_lo, int64_t t_hi, void *ws, size_t ws_bytes,
                             void *fill_ws, size_t fill_ws_bytes, uint64_t *c_keys, int64_t *c_tptr, uint32_t *tri,
                             void *stream);
QM_API size_t qm_spgemm_fill_workspace_bytes(const qm_layout *layout, int64_t nC);
/* Emits the C key set in quadtree-key order (c_keys[nC]), the triple offsets c_tptr[nC+1] and the
 * triples tri[2*nT] = (a_index, b_index) pairs, grouped by C block, k ascending within a group --
 * the order of BlockSparseLeaf.multiply's k loop (block_sparse.py:121-129). */
QM_API int qm_spgemm_fill(const qm_layout *layout, int64_t nA, int64_t nB, int64_t nC, int64_t nT,
                          void *ws, size_t ws_bytes, void *fill_ws, size_t fill_ws_bytes,
                          uint64_t *c_keys /*device*/, int64_t *c_tptr /*device*/,
                          uint32_t *tri /*device*/, void *stream);
/* The two halves of qm_spgemm_fill, for the multi-GPU partition (each rank emits only the triples
 * of its own C range): _keys writes c_keys and c_tptr (fill_ws must then stay untouched until the
 * triples are emitted); _triples writes tri[0 .. t_hi-t_lo) = triples [t_lo, t_hi). */
QM_API int qm_spgemm_fill_keys(const qm_layout *layout, int64_t nA, int64_t nB, int64_t nC, void *ws,
                               size_t ws_bytes, void *fill_ws, size_t fill_ws_bytes,
                               uint64_t *c_keys, int64_t *c_tptr, void *stream);
QM_API int qm_spgemm_fill_triples(const qm_layout *layout, int64_t nA, int64_t nB, int64_t nC, void *ws,
                                  size_t ws_bytes, void *fill_ws, size_t fill_ws_bytes,
                                  const int64_t *c_tptr, int64_t t_lo, int64_t t_hi, uint32_t *tri,
                                  void *stream);

/* ---- numeric phase (replaces BlockSparseLeaf.multiply + add, block_sparse.py:112-152) ------- */
/* c_blocks[m] = sum over t in [c_tptr[m], c_tptr[m+1]) of A[tri[2t]] * B[tri[2t+1]] (fp64),
 * c_sumsq[m] = squared Frobenius norm of the block, c_nonzero[m] = any entry != 0
 * (the np.any test of _set_block, block_sparse.py:37-41). *zero_count (device, int64) is set
 * to the number of exactly-zero C blocks (zeroed on the stream first). Block sizes above the
 * 64x64 CTA tile (bs 128) are computed as (bs/64)^2 tiles whose partial norms go to the caller's
 * workspace (qm_numeric_workspace_bytes) and are combined in a fixed order. nT = c_tptr[nC] (the
 * triple count, known to the caller from qm_spgemm_count) selects the kernel variant: few triples
 * per C block favour deeper prefetch, many favour more resident CTAs. a_keys / c_keys (the A and C
 * quadtree keys) are used for bs 16, where the C blocks of one leaf row (pair) segment are computed
 * together so that they share their A and B blocks (NULL: per-block kernel), and by the optional
 * claim orders of the bs 32/64/128 kernel (QM_UNIT_ORDER=k|lpt; default quadtree-key order). */
QM_API size_t qm_numeric_workspace_bytes(int32_t block_size, int64_t nC, int64_t nT);
QM_API int qm_numeric(const qm_layout *layout, const uint64_t *a_keys, const double *a_blocks, int64_t nA,
               const double *b_blocks, int64_t nB, const uint32_t *tri, const int64_t *c_tptr,
               const uint64_t *c_keys, int64_t nC, int64_t nT, double *c_blocks, double *c_sumsq,
               uint8_t *c_nonzero, int64_t *zero_count, void *ws, size_t ws_bytes, void *stream);
/* qm_numeric with the operands' support masks and virtual transposes. a_masks / b_masks: device
 * uint64[3*n] (row masks, column masks, flags; qm_block_meta) or NULL = full support: for bs 32-128
 * the TMA kernel skips the k panels (16 deep for bs 32/64, 32 for bs 128) of a triple where A's
 * nonzero columns and B's nonzero rows do not meet (they add exactly zero), except when either
 * block's flags mark a NaN/Inf (then every panel runs: 0*Inf is NaN). flags &
 * QM_NUMERIC_TRANSPOSED_REFS: a triple index with bit 31 set names a stored block used transposed
 * -- the reference's virtual transposes (`_virtual_child` / ta / tb, ops.py:100-116) as a TMA box
 * and shared-memory addressing choice, no materialised transpose (bs 32/64/128 only).
 * *panel_count (device int64, may be NULL) receives the k depth executed by the bs 32/64/128
 * kernel, summed over triples (bs per triple without skipping; -1 for other kernels): the executed
 * flops are 2*bs*bs*count. */
#define QM_NUMERIC_TRANSPOSED_REFS 1
QM_API int qm_numeric_masked(const qm_layout *layout, const uint64_t *a_keys, const double *a_blocks,
                             const uint64_t *a_masks, int64_t nA, const double *b_blocks, const uint64_t *b_masks,
                             int64_t nB, int32_t flags, const uint32_t *tri, const int64_t *c_tptr,
                             const uint64_t *c_keys, int64_t nC, int64_t nT, double *c_blocks, double *c_sumsq,
                             uint8_t *c_nonzero, int64_t *zero_count, int64_t *panel_count, void *ws,
                             size_t ws_bytes, void *stream);
/* The numeric phase of a multi-GPU product fused with its halo exchange: operand blocks live in
 * up to 8 pools per operand -- this rank's and the other ranks' block pools mapped into this GPU's
 * address space (CUDA IPC / peer access over NVLink). a_pools / b_pools / a_counts / b_counts are
 * HOST arrays of device pointers and block counts; triple indices are packed
 * (owner << 28) | local_index. The TMA producer reads each block straight from its owner's memory,
 * overlapped with the DMMAs of earlier stages (no separate exchange). bs 32/64/128 only. */
QM_API int qm_numeric_pools(const qm_layout *layout, const double *const *a_pools, const int64_t *a_counts,
                            int32_t n_a_pools, const double *const *b_pools, const int64_t *b_counts,
                            int32_t n_b_pools, const uint32_t *tri, const int64_t *c_tptr, int64_t nC,
                            int64_t nT, double *c_blocks, double *c_sumsq, uint8_t *c_nonzero,
                            int64_t *zero_count, void *ws, size_t ws_bytes, void *stream);
/* CUDA IPC of block pools for qm_numeric_pools (same-node ranks): export writes the 64-byte
 * cudaIpcMemHandle of the allocation containing `ptr` and ptr's byte offset in it; open maps a peer
 * handle (once per handle and process) and returns the allocation base; close unmaps it. */
QM_API int qm_ipc_export(const void *ptr, void *handle_out, int64_t *offset_out);
QM_API int qm_ipc_open(const void *handle, void **base_out);
QM_API int qm_ipc_close(void *base);
/* Halo of a staged multi-GPU product: the blocks one rank reads from its peers' pools. */
#define QM_MAX_RANKS 8
typedef struct qm_halo {
  int32_t world;                      /* ranks (<= QM_MAX_RANKS) */
  int32_t reserved;                   /* must be 0 */
  const uint32_t *index[2];           /* device: global block indices of the A / B halo, ascending */
  int64_t count[2];                   /* entries of index[0] / index[1] */
  double *pool[2];                    /* device: halo pools; block x of index[o] lands at pool[o] + x */
  uint64_t peer_base[2][QM_MAX_RANKS];/* address of rank r's A / B pool (peer memory mapped by qm_ipc_open) */
  int64_t offset[2][QM_MAX_RANKS + 1];/* rank r owns global indices [offset[o][r], offset[o][r+1]) */
  int64_t min_ns;                     /* measurement only: the gather lasts at least this long */
} qm_halo;

/* Staged multi-GPU numeric phase (replaces the remote-operand fetches of the reference's transfer
 * layer, TransferSim.fetch chunkstore.py:188-210, for the blocks one worker's tasks read). As
 * qm_numeric_pools, plus:
 *   mask_tri / a_cmask, a_flags / b_rmask, b_flags: support masks (A's column masks, B's row masks,
 *     NaN/Inf flags; qm_block_meta's rows) indexed by mask_tri (the triples in the masks' index
 *     space, e.g. global block indices), so k panels are skipped as in qm_numeric_masked (all NULL:
 *     no skipping);
 *   order: claim order, one C block index per claim (NULL: key order);
 *   halo (NULL: none): before the numeric kernel, a gather kernel copies the halo blocks from the
 *     peer pools (read over NVLink) into the halo pools with bulk (TMA) copies on a few SMs; the
 *     numeric kernel is launched as its programmatic dependent and runs meanwhile: claims <
 *     gate_units (the local-only C blocks, put first by `order`) go ahead, claims >= gate_units wait
 *     for the gather grid to complete. */
QM_API int qm_numeric_pools_ex(const qm_layout *layout, const double *const *a_pools, const int64_t *a_counts,
                               int32_t n_a_pools, const double *const *b_pools, const int64_t *b_counts,
                               int32_t n_b_pools, const uint32_t *tri, const uint32_t *mask_tri,
                               const uint64_t *a_cmask, const uint64_t *a_flags, const uint64_t *b_rmask,
                               const uint64_t *b_flags, const uint32_t *order, const qm_halo *halo, int64_t gate_units,
                               const int64_t *c_tptr, int64_t nC, int64_t nT, double *c_blocks, double *c_sumsq,
                               uint8_t *c_nonzero, int64_t *zero_count, int64_t *panel_count, void *ws,
                               size_t ws_bytes, void *stream);
/* Staging plan of one rank (device; the host only reads the three counts). tri: the rank's
 * triples in global block indices (uint32 pairs); the rank owns A indices [a_lo, a_hi) of nA and
 * B indices [b_lo, b_hi) of nB (b_is_a: one operand, one halo). Writes
 *   tri_packed[2*nT]: local index, or (1 << 28) | halo position for a block owned by a peer;
 *   order[nC]: C blocks whose triples are all local first, then the others (key order in each);
 *   halo_a / halo_b: the distinct peer-owned indices, ascending (capacity nA - (a_hi - a_lo), ...);
 *   counts_out (host): [local-only C blocks, halo_a entries, halo_b entries]. Synchronises. */
QM_API size_t qm_stage_plan_workspace_bytes(int64_t nA, int64_t nB, int64_t nC, int32_t b_is_a);
QM_API int qm_stage_plan(const uint32_t *tri, int64_t nT, const int64_t *c_tptr, int64_t nC, int64_t a_lo,
                         int64_t a_hi, int64_t nA, int64_t b_lo, int64_t b_hi, int64_t nB, int32_t b_is_a,
                         void *ws, size_t ws_bytes, uint32_t *tri_packed, uint32_t *order, uint32_t *halo_a,
                         uint32_t *halo_b, int64_t *counts_out, void *stream);
/* Which numeric kernel qm_numeric uses for this block size: 2 = TMA + mbarrier warp-specialised
 * DMMA (bs 32/64/128; bs 16 as grouped leaf-row segments when a leaf holds >= 2 blocks per side),
 * 1 = cp.async DMMA (QM_NUMERIC=cpasync, or bs 16 with one block per leaf), 0 = FP64 SIMT. */
QM_API int qm_numeric_path(int32_t block_size);
/* Name of the numeric kernel qm_numeric / qm_numeric_masked launches for a product of nC C blocks and
 * nT triples in this layout (masked: support masks passed; flags as qm_numeric_masked): bs 16
 * groups and bs 32 quads of C blocks are used for products whose C blocks have k lists of some
 * length (>= 4 / >= 8 triples per block on average), the per-block kernels otherwise. Static string. */
QM_API const char *qm_numeric_kernel(const qm_layout *layout, int64_t nC, int64_t nT, int32_t masked,
                                     int32_t flags);

/* ---- exact-zero compaction (replaces _put_leaf / _set_block dropping, ops.py:119-122) --------- */
QM_API size_t qm_compact_workspace_bytes(int64_t nC);
/* Stream-compacts the C blocks whose c_nonzero flag is set into the *_out arrays (order kept). */
QM_API int qm_compact(int32_t block_size, int64_t nC, const uint8_t *c_nonzero, const uint64_t *keys_in,
               const double *blocks_in, const double *sumsq_in, uint64_t *keys_out,
               double *blocks_out, double *sumsq_out, void *ws, size_t ws_bytes, void *stream);

/* ---- per-block statistics, gather (halo packing) ------------------------------------------- */
/* sumsq[i] = sum of squares of block i, nonzero[i] = any entry != 0 (nonzero may be NULL). */
QM_API int qm_block_stats(int32_t block_size, int64_t n, const double *blocks, double *sumsq,
                   uint8_t *nonzero, void *stream);
/* Support masks of n bs x bs blocks: bit b of row_mask[m] / col_mask[m] is set when a row / column r
 * with b = r (bs <= 64) or b = r*64/bs (bs > 64) of block m holds a nonzero; blocks holding NaN or
 * Inf get full masks. */
QM_API int qm_block_masks(int32_t block_size, int64_t n, const double *blocks, uint64_t *row_mask,
                          uint64_t *col_mask, void *stream);
/* All per-block metadata of n blocks in ONE read of the blocks (each output may be NULL):
 * sumsq[i] / nonzero[i] as qm_block_stats (bit-identical sums), *zero_count += exactly-zero blocks,
 * masks = uint64[3*n]: row masks, column masks (as qm_block_masks), flags (bit 0: the block holds a
 * NaN or Inf -- its masks are full and the numeric kernel executes all of its k panels, so 0*Inf
 * still yields the reference's NaN), and not_full[0] / not_full[1] (device int64, zeroed by the
 * caller) become nonzero when some block's row / column mask is not full (all-full operands skip
 * the exact-zero filters entirely). The reference keeps block norms with the leaf
 * (block_sparse.py:41, BlockSparseLeaf.block_norms); masks are the same kind of input metadata. */
QM_API int qm_block_meta(int32_t block_size, int64_t n, const double *blocks, double *sumsq, uint8_t *nonzero,
                         int64_t *zero_count, uint64_t *masks, int64_t *not_full, void *stream);
/* dst[i] = src[idx[i]] for whole bs x bs blocks (packs halo blocks for the NVLink exchange). */
QM_API int qm_gather_blocks(int32_t block_size, const double *src, const int64_t *idx, int64_t n,
                     double *dst, void *stream);

/* dst[i] = src[i]^T per bs x bs block: the materialised form of the reference's virtual transpose
 * (op_view, leaves/base.py:117-118; ta/tb/symmetric children, ops.py:100-116). */
QM_API int qm_transpose_blocks(int32_t block_size, const double *src, int64_t n, double *dst,
                               void *stream);
/* dst[m] = src[idx[m]], transposed where transpose[m] != 0 (transpose may be NULL): a symmetric
 * operand's full block set from its stored upper triangle in one pass (ops.py:100-116's virtual
 * transposes, materialised). */
QM_API int qm_gather_blocks_t(int32_t block_size, const double *src, const int64_t *idx,
                              const uint8_t *transpose, int64_t n, double *dst, void *stream);

/* ---- add / scale / add_scaled_identity (the step after a product) ---------- */
/* out[m] = alpha*A[ia[m]] + beta*B[ib[m]] per block, an operand absent when its index is -1;
 * exact IEEE products and sum (BlockSparseLeaf.add / scale, block_sparse.py:134-160). Optional
 * (NULL = skip) fused statistics of each output block, bit-identical to qm_block_stats on `out`:
 * sum of squares, nonzero flag, and the count of exactly-zero blocks added to *zero_count. */
QM_API int qm_axpby_blocks(int32_t block_size, int64_t n, const int64_t *ia, const int64_t *ib,
                           double alpha, double beta, const double *a_blocks, const double *b_blocks,
                           double *out, double *out_sumsq, uint8_t *out_nonzero, int64_t *zero_count,
                           void *stream);
/* Diagonal blocks of A + c*I with the reference's two leaf cases (ops.py:253-345): mode 0 =
 * A_blk + c*eye, mode 1 = A_blk + identity-from-triplets (logical diagonal only); ia = -1 when the
 * A block is absent, bi = block row. */
QM_API int qm_add_identity_blocks(int32_t block_size, int64_t n, const int64_t *ia, const int64_t *bi,
                                  const int8_t *mode, double c, int64_t n_logical,
                                  const double *a_blocks, double *out, void *stream);

/* ---- approximate multiply: the reference's norm-based pruning ------------- */
/* Node norms of every quadtree level of one operand (the store's id-carried norms,
 * quadtree.py:138-140, block_sparse.py:91-92): level L (0 = root .. depth) occupies
 * codes/norms[L*n, L*n + counts[L]) (caller arrays of (depth+1)*n entries; counts on the host),
 * codes = Morton node codes ascending. Synchronises the stream once per level. */
QM_API size_t qm_node_norms_workspace_bytes(int64_t n);
QM_API int qm_node_norms(const qm_layout *layout, const uint64_t *keys, const double *sumsq, int64_t n,
                         uint64_t *codes, double *norms, int64_t *counts, void *ws, size_t ws_bytes,
                         void *stream);
/* One level of the pruned task recursion (ops.py:197-241 with tau, ops.py:232): the 8 child pairs
 * of every parent pair (packed I<<42 | K<<21 | J; level 0: the root pair, parents unused), kept
 * when both operand nodes exist (a_sym/b_sym: lower nodes read their stored upper mirror;
 * b_transposed: B node (K,J) is stored node (J,K); upper: I <= J). Pairs with
 * norm(A node)*norm(B node) < tau_l are pruned: their bounds go to pruned_out (the prune log,
 * engine.py:273-275); the others to alive_out. Outputs hold up to 8*n_parents entries; counts are
 * returned on the host (synchronises the stream). */
QM_API size_t qm_prune_level_workspace_bytes(int64_t n_parents);
QM_API int qm_prune_level(const qm_layout *layout, int32_t level, double tau_l, const uint64_t *parents,
                          int64_t n_parents, const uint64_t *a_codes, const double *a_norms, int64_t a_count,
                          int32_t a_sym, const uint64_t *b_codes, const double *b_norms, int64_t b_count,
                          int32_t b_sym, int32_t b_transposed, int32_t upper, uint64_t *alive_out,
                          double *pruned_out, int64_t *n_alive, int64_t *n_pruned, void *ws,
                          size_t ws_bytes, void *stream);

/* The whole pruned recursion in ONE launch (cooperative kernel, a grid-wide barrier between
 * levels, no host round trip per level): the same classification as qm_prune_level for every
 * level 0..depth with tau_l = tau / 8^l. Node tables as written by qm_node_norms (level L at
 * codes/norms + L*stride, counts[L] on the host). Surviving leaf-level pairs (packed
 * I<<42 | K<<21 | J, unordered) go to leaf_pairs_out[cap_pairs], prune bounds (unordered) to
 * log_out[cap_log]. counts_out (host, 2*(depth+1)+2 entries): alive and pruned pairs per level,
 * the log total, and an overflow flag (bit 0: a level had more than cap_pairs survivors, bit 1:
 * more than cap_log bounds -- the caller retries with larger capacities). Synchronises the stream
 * once. */
QM_API size_t qm_prune_all_workspace_bytes(int64_t cap_pairs);
QM_API int qm_prune_all(const qm_layout *layout, double tau, const uint64_t *a_codes, const double *a_norms,
                        int64_t a_stride, const int64_t *a_counts, int32_t a_sym, const uint64_t *b_codes,
                        const double *b_norms, int64_t b_stride, const int64_t *b_counts, int32_t b_sym,
                        int32_t b_transposed, int32_t upper, int64_t cap_pairs, uint64_t *leaf_pairs_out,
                        double *log_out, int64_t cap_log, int64_t *counts_out, void *ws, size_t ws_bytes,
                        void *stream);

/* Keeps the triples of a symbolic plan whose leaf pair (li, lk, lj) is in the sorted
 * leaf_pairs codes ((li*w + lk)*w + lj, w = 2^depth): the products of pruned subtrees vanish; C
 * blocks left without triples vanish too (an all-pruned subtree is nil). Order is preserved.
 * Outputs have the input capacities (nT pairs, nC+1 offsets, nC keys); counts returned on the
 * host (synchronises the stream). */
QM_API size_t qm_filter_triples_workspace_bytes(int64_t nC, int64_t nT);
QM_API int qm_filter_triples(const qm_layout *layout, const uint64_t *a_keys, const uint64_t *b_keys,
                             int32_t b_transposed, const uint32_t *tri, const int64_t *c_tptr,
                             const uint64_t *c_keys, int64_t nC, int64_t nT, const uint64_t *leaf_pairs,
                             int64_t n_pairs, uint32_t *tri_out, int64_t *c_tptr_out, uint64_t *c_keys_out,
                             int64_t *nC_out, int64_t *nT_out, void *ws, size_t ws_bytes, void *stream);

/* Ancestor norms of block entries: out[l*n + m] = the norm (from qm_node_norms tables, level L at
 * codes/norms + L*stride, counts[L] on the host) of the level-l quadtree node containing entry
 * m's block, 0 when absent; sym: a lower node reads its stored upper mirror (symmetric operands). */
QM_API int qm_ancestor_norms(const qm_layout *layout, const uint64_t *keys, int64_t n, const uint64_t *codes,
                             const double *norms, int64_t stride, const int64_t *counts, int32_t sym,
                             double *out, void *stream);
/* The approximate multiply's filter in one pass over the triples: a leaf product survives the
 * reference's pruned recursion iff none of its ancestor tasks was pruned, i.e. at every level l
 * norm(A ancestor) * norm(B ancestor) >= tau / 8^l (ops.py:199-204, 232; both ancestors exist
 * because the blocks do). anc_a [(depth+1)*nA] / anc_b from qm_ancestor_norms of the operands as
 * the plan indexes them (bit 31 of a triple index -- a transposed reference -- is ignored).
 * Compacts like qm_filter_triples (C blocks left without triples vanish; counts to the host,
 * one synchronisation). The prune log itself (qm_prune_all) is not needed for the product. */
QM_API int qm_filter_triples_norms(const qm_layout *layout, double tau, const uint32_t *tri, const int64_t *c_tptr,
                                   const uint64_t *c_keys, int64_t nC, int64_t nT, const double *anc_a, int64_t nA,
                                   const double *anc_b, int64_t nB, uint32_t *tri_out, int64_t *c_tptr_out,
                                   uint64_t *c_keys_out, int64_t *nC_out, int64_t *nT_out, void *ws,
                                   size_t ws_bytes, void *stream);

/* ---- synthetic inputs (device side of the block-keyed generator) -------- */
/* For each key, fills the block with numpy's default_rng([seed, matrix_id, bi, bj]).uniform(-1, 1,
 * (bs, bs)) -- bit-identical PCG64 + SeedSequence -- then zeroes entries outside the element
 * pattern: pattern 0 = dense (clipped to n_logical), 1 = band |i - j| <= half_bw, 2 = band of ones
 * (the reference generators' value 1.0, generators.py:251-265; no random draws). */
QM_API int qm_generate_blocks(const qm_layout *layout, const uint64_t *keys, int64_t n, uint64_t seed,
                       uint32_t matrix_id, int32_t pattern, int64_t half_bw, double *blocks,
                       double *sumsq, void *stream);

/* ---- FP64 peak microbenchmarks (roofline denominator; MEASURED_PEAKS.json has no FP64) ------ */
/* Runs `iters` dependent-chain-free DMMA (kind 0) or DFMA (kind 1) steps on `ctas` CTAs of
 * `threads` threads; returns the flop count of the launch in *flops. */
QM_API int qm_fp64_peak_kernel(int kind, int ctas, int threads, int64_t iters, double *sink,
                        double *flops, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* QMB200_H */

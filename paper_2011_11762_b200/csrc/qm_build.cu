// Device construction of a block set from (row, col, value) triplets.
//
// Replaces the host build of the reference: MatrixSession.matrix_from_triplets (session.py:72-104)
// -> quadtree.build_from_triplets (quadtree.py:90-142) -> BlockSparseLeaf.from_triplets
// (leaves/block_sparse.py:47-68): entries are partitioned by quadrant keeping their input order,
// a leaf stable-sorts its entries by block, and np.add.at sums duplicates into a zero block in
// that order; exactly-zero blocks are dropped (_set_block, block_sparse.py:37-41).
//
// Here: one 64-bit sort key per entry = (quadtree key of its block) << pbits | position in the
// block; a stable radix sort groups duplicates of an element in input order; one thread per
// distinct element sums its run sequentially starting from +0.0 (the np.add.at order, so the
// result is bit-identical to the reference); elements are scattered into zeroed blocks; block norms
// and the exact-zero flags come from qm_block_stats, dropped blocks from qm_compact.
#include <cub/cub.cuh>

#include "qm_common.cuh"

namespace qm {
int launch_block_stats(int bs, int64_t n, const double *blocks, double *sumsq, uint8_t *nonzero,
                       int64_t *zero_count, cudaStream_t st);

namespace {

inline int ceil_log2(uint64_t x) {
  int b = 0;
  while ((1ull << b) < x) ++b;
  return b;
}

inline int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (int)g;
}

__global__ void k_entry_keys(const int64_t *rows, const int64_t *cols, int64_t n, int64_t n_logical,
                             int bs, int nbl, int lbits, int pbits, uint64_t *key, uint32_t *iota,
                             unsigned long long *bad) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rows[x], c = cols[x];
    iota[x] = (uint32_t)x;
    if (r < 0 || c < 0 || r >= n_logical || c >= n_logical) {
      atomicAdd(bad, 1ull);
      key[x] = ~0ull;
      continue;
    }
    const uint32_t bi = (uint32_t)(r / bs), bj = (uint32_t)(c / bs);
    const uint64_t pos = (uint64_t)(r - (int64_t)bi * bs) * bs + (uint64_t)(c - (int64_t)bj * bs);
    key[x] = (qkey(bi, bj, nbl, lbits) << pbits) | pos;
  }
}

// head flags of elements (distinct keys) and of blocks (distinct key >> pbits)
__global__ void k_heads(const uint64_t *skey, int64_t n, int pbits, uint32_t *elem_head,
                        uint32_t *blk_head) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = skey[x];
    const bool eh = x == 0 || skey[x - 1] != k;
    const bool bh = x == 0 || (skey[x - 1] >> pbits) != (k >> pbits);
    elem_head[x] = eh;
    blk_head[x] = bh;
  }
}

// One thread per element head: sequential sum of the duplicate run (input order), scatter.
__global__ void k_elements(const uint64_t *skey, const uint32_t *perm, const double *vals, int64_t n,
                           int pbits, int bs, const uint32_t *elem_head, const uint32_t *blk_head,
                           const uint32_t *blk_incl, double *blocks, uint64_t *keys) {
  const uint64_t pmask = (1ull << pbits) - 1ull;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    if (!elem_head[x]) continue;
    const uint64_t k = skey[x];
    double s = 0.0;
    int64_t y = x;
    do {
      s = s + vals[perm[y]];
      ++y;
    } while (y < n && skey[y] == k);
    const int64_t b = (int64_t)blk_incl[x] - 1;  // inclusive scan of block heads
    blocks[(size_t)b * bs * bs + (k & pmask)] = s;
    if (blk_head[x]) keys[b] = k >> pbits;
  }
}

struct BuildWs {
  uint64_t *key, *skey;
  uint32_t *iota, *perm, *elem_head, *blk_head, *blk_incl;
  unsigned long long *bad;
  void *cub;
  size_t cub_bytes;
};

BuildWs carve_build(Carver &cv, int64_t n, int key_bits) {
  BuildWs w;
  w.key = cv.take<uint64_t>(n);
  w.skey = cv.take<uint64_t>(n);
  w.iota = cv.take<uint32_t>(n);
  w.perm = cv.take<uint32_t>(n);
  w.elem_head = cv.take<uint32_t>(n);
  w.blk_head = cv.take<uint32_t>(n);
  w.blk_incl = cv.take<uint32_t>(n);
  w.bad = cv.take<unsigned long long>(1);
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                  (uint32_t *)nullptr, (uint32_t *)nullptr, (int64_t)n, 0, key_bits);
  cub::DeviceScan::InclusiveSum(nullptr, b, (uint32_t *)nullptr, (uint32_t *)nullptr, (int64_t)n);
  w.cub_bytes = std::max(a, b);
  w.cub = cv.take<char>(w.cub_bytes);
  return w;
}

int build_bits(const Geometry &g, int *pbits, int *key_bits) {
  *pbits = std::max(1, ceil_log2((uint64_t)g.bs * g.bs));
  *key_bits = 2 * (g.depth + g.lbits) + *pbits;
  if (*key_bits > 64) {
    set_error("triplet build: %d key bits exceed 64 (layout too large for the device build)", *key_bits);
    return QM_ERR_UNSUPPORTED;
  }
  return QM_OK;
}

}  // namespace
}  // namespace qm

using namespace qm;

extern "C" size_t qm_build_workspace_bytes(const qm_layout *layout, int64_t n_entries) {
  Geometry g;
  int pbits, key_bits;
  if (make_geometry(layout, &g) != QM_OK || build_bits(g, &pbits, &key_bits) != QM_OK) return 0;
  Carver cv(nullptr, 0);
  carve_build(cv, n_entries, key_bits);
  return cv.off;
}

extern "C" int qm_build_count(const qm_layout *layout, const int64_t *rows, const int64_t *cols,
                              int64_t n, void *ws, size_t ws_bytes, int64_t *n_blocks_out,
                              int64_t *n_out_of_range, void *stream) {
  Geometry g;
  int rc = make_geometry(layout, &g);
  if (rc != QM_OK) return rc;
  int pbits, key_bits;
  rc = build_bits(g, &pbits, &key_bits);
  if (rc != QM_OK) return rc;
  if (n < 0 || n >= (int64_t)1 << 32 || !n_blocks_out || !n_out_of_range) {
    set_error("qm_build_count: bad entry count or outputs");
    return QM_ERR_INVALID;
  }
  *n_blocks_out = 0;
  *n_out_of_range = 0;
  if (n == 0) return QM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Carver cv(ws, ws_bytes);
  BuildWs w = carve_build(cv, n, key_bits);
  if (!cv.ok() || !ws) {
    set_error("qm_build_count: workspace %zu < required %zu", ws_bytes, cv.off);
    return QM_ERR_WORKSPACE;
  }
  QM_CUDA_TRY(cudaMemsetAsync(w.bad, 0, sizeof(unsigned long long), st));
  k_entry_keys<<<grid_for(n), 256, 0, st>>>(rows, cols, n, layout->n_logical, g.bs, g.nbl, g.lbits,
                                            pbits, w.key, w.iota, w.bad);
  QM_LAUNCHED("k_entry_keys");
  int64_t bad = 0;
  rc = read_device_i64(w.bad, 1, &bad, st);
  if (rc != QM_OK) return rc;
  if (bad) {
    *n_out_of_range = (int64_t)bad;
    return QM_OK;
  }
  size_t tb = w.cub_bytes;
  QM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.cub, tb, w.key, w.skey, w.iota, w.perm, n, 0, key_bits, st));
  k_heads<<<grid_for(n), 256, 0, st>>>(w.skey, n, pbits, w.elem_head, w.blk_head);
  QM_LAUNCHED("k_heads");
  tb = w.cub_bytes;
  QM_CUDA_TRY(cub::DeviceScan::InclusiveSum(w.cub, tb, w.blk_head, w.blk_incl, n, st));
  // blk_incl is uint32: read the aligned 8-byte word holding the last entry
  const int64_t last = n - 1;
  int64_t word = 0;
  rc = read_device_i64(w.blk_incl + (last & ~1ll), 1, &word, st);
  if (rc != QM_OK) return rc;
  *n_blocks_out = (last & 1) ? (int64_t)((uint64_t)word >> 32) : (int64_t)(uint32_t)word;
  return QM_OK;
}

extern "C" int qm_build_fill_meta(const qm_layout *layout, const double *vals, int64_t n, void *ws,
                                  size_t ws_bytes, int64_t n_blocks, uint64_t *keys, double *blocks,
                                  double *sumsq, uint8_t *nonzero, int64_t *zero_count, uint64_t *masks,
                                  int64_t *not_full, void *stream) {
  Geometry g;
  int rc = make_geometry(layout, &g);
  if (rc != QM_OK) return rc;
  int pbits, key_bits;
  rc = build_bits(g, &pbits, &key_bits);
  if (rc != QM_OK) return rc;
  if (n == 0 || n_blocks == 0) return QM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Carver cv(ws, ws_bytes);
  BuildWs w = carve_build(cv, n, key_bits);
  if (!cv.ok() || !ws) {
    set_error("qm_build_fill: workspace too small");
    return QM_ERR_WORKSPACE;
  }
  QM_CUDA_TRY(cudaMemsetAsync(blocks, 0, (size_t)n_blocks * g.bs * g.bs * sizeof(double), st));
  k_elements<<<grid_for(n), 256, 0, st>>>(w.skey, w.perm, vals, n, pbits, g.bs, w.elem_head, w.blk_head,
                                          w.blk_incl, blocks, keys);
  QM_LAUNCHED("k_elements");
  // norms, nonzero flags and (optionally) support masks in one read of the filled blocks
  return launch_block_meta(g.bs, n_blocks, blocks, sumsq, nonzero, zero_count, masks,
                           masks ? masks + n_blocks : nullptr, masks ? masks + 2 * n_blocks : nullptr, not_full, st);
}

extern "C" int qm_build_fill(const qm_layout *layout, const double *vals, int64_t n, void *ws,
                             size_t ws_bytes, int64_t n_blocks, uint64_t *keys, double *blocks,
                             double *sumsq, uint8_t *nonzero, int64_t *zero_count, void *stream) {
  return qm_build_fill_meta(layout, vals, n, ws, ws_bytes, n_blocks, keys, blocks, sumsq, nonzero, zero_count,
                            nullptr, nullptr, stream);
}

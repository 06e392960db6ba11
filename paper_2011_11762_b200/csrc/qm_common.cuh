// Shared helpers of libqmb200: error reporting, launch accounting, quadtree-key arithmetic.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/qmb200.h"

namespace qm {

// Thread-local last-error message (qm_last_error).
void set_error(const char *fmt, ...);
// Reads n (<= 8) int64 values from device memory into host memory without a copy engine: a tiny
// kernel writes them into a mapped pinned buffer, then `stream` is synchronised. (A D2H
// cudaMemcpyAsync would queue behind large in-flight copies of earlier steps on the copy engine.)
// An optional second source appends one more value (two scattered counts, one synchronisation).
int read_device_i64(const void *dev_src, int n, int64_t *host_out, cudaStream_t stream,
                    const void *dev_src2 = nullptr);
// The calling thread's mapped pinned buffer (8 int64) used by read_device_i64: a kernel may write
// values there itself (device pointer `dev`) and the host read them after synchronising the stream.
int mapped_i64(int64_t **host, int64_t **dev);
// Counts one kernel launch (qm_launch_count).
void note_launch(int n = 1);
// Per-block metadata in one read (k_block_meta, qm_numeric.cu): sums of squares, nonzero flags,
// exact-zero count, support masks (rmask/cmask/flags may be NULL) and the not-full OR flags.
int launch_block_meta(int bs, int64_t n, const double *blocks, double *sumsq, uint8_t *nonzero,
                      int64_t *zero_count, uint64_t *rmask, uint64_t *cmask, uint64_t *flags,
                      int64_t *not_full, cudaStream_t st);

#define QM_CUDA_TRY(expr)                                                                   \
  do {                                                                                      \
    cudaError_t qm_e_ = (expr);                                                             \
    if (qm_e_ != cudaSuccess) {                                                             \
      qm::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(qm_e_), __FILE__,    \
                    __LINE__);                                                              \
      return QM_ERR_CUDA;                                                                   \
    }                                                                                       \
  } while (0)

// Launch check: records the launch and turns a launch error into a QM_ERR_CUDA return.
#define QM_LAUNCHED(name)                                                                   \
  do {                                                                                      \
    qm::note_launch();                                                                      \
    cudaError_t qm_e_ = cudaGetLastError();                                                 \
    if (qm_e_ != cudaSuccess) {                                                             \
      qm::set_error("launch of %s failed: %s", name, cudaGetErrorString(qm_e_));           \
      return QM_ERR_CUDA;                                                                   \
    }                                                                                       \
  } while (0)

// Once-per-device initialisation (cudaFuncSetAttribute applies to the current device only, so a
// process driving several GPUs must configure each). f() returns a qm_status; a failure is retried
// on the next call. Devices are tracked in a 64-bit mask (ordinal & 63).
struct PerDeviceOnce {
  std::atomic<uint64_t> done{0};
  template <class F>
  int run(F f) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return 0;
    const int rc = f();
    if (rc == 0) done.fetch_or(bit, std::memory_order_acq_rel);
    return rc;
  }
};

// An int computed once per device (e.g. a kernel's occupancy: it never changes for a device).
struct PerDeviceInt {
  std::atomic<int> v[64];
  PerDeviceInt() {
    for (auto &x : v) x.store(-1, std::memory_order_relaxed);
  }
  template <class F>
  int get(int *out, F f) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    int x = v[dev & 63].load(std::memory_order_relaxed);
    if (x < 0) {
      const int rc = f(&x);
      if (rc != 0) return rc;
      v[dev & 63].store(x, std::memory_order_relaxed);
    }
    *out = x;
    return 0;
  }
};

// SM count of the current device (cached per device).
inline int device_sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  int n = cache[dev & 63].load(std::memory_order_relaxed);
  if (n <= 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev & 63].store(n, std::memory_order_relaxed);
  }
  return n;
}

// Derived geometry of a qm_layout.
struct Geometry {
  int32_t bs;     // block size
  int32_t nbl;    // blocks per leaf side = leaf_dim / bs
  int32_t lbits;  // bits of the in-leaf coordinate = ceil(log2(nbl))
  int32_t depth;  // quadtree depth
  int64_t nbg;    // blocks per matrix side = nbl << depth
};

// Optional inputs of the numeric kernel beyond the triples: the A keys and layout (for claim
// orders other than quadtree-key order; a_keys = NULL keeps key order), the operands' support masks
// (k panels where A's nonzero columns and B's nonzero rows do not meet are skipped; NULL = all
// panels), whether triple indices carry transpose flags, and where to count the k depth executed.
struct NumericAux {
  const uint64_t *a_keys = nullptr;
  int32_t nbl = 1, lbits = 0;
  int64_t nbg = 1;
  // support masks of the operands' blocks (row masks, column masks, flags with bit 0 = NaN/Inf);
  // the kernels read A's columns and B's rows (their rows / columns only for transposed references)
  const uint64_t *a_rows = nullptr, *a_cols = nullptr, *a_flags = nullptr;
  const uint64_t *b_rows = nullptr, *b_cols = nullptr, *b_flags = nullptr;
  bool masked() const { return a_cols && a_flags && b_rows && b_flags; }
  bool transpose_bits = false;  // triple indices carry a transpose flag in bit 31 (virtual transposes)
  int64_t *panel_count = nullptr;
  // Staged multi-GPU products (qm_numeric_pools_ex): the caller's claim order (one C block per
  // claim, overriding QM_UNIT_ORDER); triple indices into the masks' index space when the operands
  // come from several pools; and the halo gathered by k_halo_gather while the numeric kernel runs,
  // whose claims >= gate_units wait for it.
  const uint32_t *order = nullptr;
  const uint32_t *mask_tri = nullptr;
  const qm_halo *halo = nullptr;
  int64_t gate_units = 0;
};

inline int make_geometry(const qm_layout *l, Geometry *g) {
  if (!l) { set_error("layout is NULL"); return QM_ERR_INVALID; }
  if (l->block_size < 1 || l->leaf_dim < 1 || l->depth < 0 || l->n_logical < 1) {
    set_error("invalid layout (n=%lld leaf_dim=%d depth=%d bs=%d)", (long long)l->n_logical,
              l->leaf_dim, l->depth, l->block_size);
    return QM_ERR_INVALID;
  }
  if (l->leaf_dim % l->block_size != 0) {
    set_error("block size %d must divide leaf dimension %d", l->block_size, l->leaf_dim);
    return QM_ERR_INVALID;
  }
  g->bs = l->block_size;
  g->nbl = l->leaf_dim / l->block_size;
  int lb = 0;
  while ((1 << lb) < g->nbl) ++lb;
  g->lbits = lb;
  g->depth = l->depth;
  g->nbg = (int64_t)g->nbl << l->depth;
  if (2 * (l->depth + lb) > 62 || g->nbg > (int64_t)1 << 30) {
    set_error("layout too large for 64-bit quadtree keys (depth=%d lbits=%d)", l->depth, lb);
    return QM_ERR_UNSUPPORTED;
  }
  return QM_OK;
}

// Interleave: bit b of x -> bit 2b.
__host__ __device__ __forceinline__ uint64_t spread_bits(uint32_t x) {
  uint64_t v = x;
  v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
  v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
  v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}

// Inverse of spread_bits on the even bits of v.
__host__ __device__ __forceinline__ uint32_t compact_bits(uint64_t v) {
  v &= 0x5555555555555555ull;
  v = (v | (v >> 1)) & 0x3333333333333333ull;
  v = (v | (v >> 2)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v >> 4)) & 0x00FF00FF00FF00FFull;
  v = (v | (v >> 8)) & 0x0000FFFF0000FFFFull;
  v = (v | (v >> 16)) & 0x00000000FFFFFFFFull;
  return (uint32_t)v;
}

// Quadtree key of block (bi, bj): Morton over the leaf grid (row bit high, so NW<NE<SW<SE as in
// quadtree.py:128-129), then row-major inside the leaf (BlockSparseLeaf.encode sorts (bi, bj)).
__host__ __device__ __forceinline__ uint64_t qkey(uint32_t bi, uint32_t bj, int nbl, int lbits) {
  uint32_t li = bi / nbl, lj = bj / nbl;
  uint32_t ri = bi - li * nbl, rj = bj - lj * nbl;
  uint64_t m = (spread_bits(li) << 1) | spread_bits(lj);
  return (m << (2 * lbits)) | ((uint64_t)ri << lbits) | rj;
}

__host__ __device__ __forceinline__ void qkey_decode(uint64_t key, int nbl, int lbits, uint32_t *bi,
                                                     uint32_t *bj) {
  uint64_t local = key & ((1ull << (2 * lbits)) - 1ull);
  uint32_t ri = (uint32_t)(local >> lbits);
  uint32_t rj = (uint32_t)(local & ((1ull << lbits) - 1ull));
  uint64_t m = key >> (2 * lbits);
  uint32_t li = compact_bits(m >> 1), lj = compact_bits(m);
  *bi = li * nbl + ri;
  *bj = lj * nbl + rj;
}

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Bump allocator over a caller workspace.
struct Carver {
  char *base;
  size_t cap, off;
  Carver(void *p, size_t c) : base((char *)p), cap(c), off(0) {}
  template <class T> T *take(size_t count) {
    size_t at = align_up(off);
    off = at + align_up(count * sizeof(T));
    return base ? (T *)(base + at) : nullptr;
  }
  bool ok() const { return off <= cap; }
};

}  // namespace qm

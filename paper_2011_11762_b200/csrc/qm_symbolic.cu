// Symbolic phase of C = A*B on quadtree-key-ordered block matrices.
//
// Replaces the reference's recursive task expansion: _multiply_body (ops.py:197-241) spawns, for
// every non-nil (A-node, B-node) pair, C_ij <- A_i0*B_0j + A_i1*B_1j, and nil operands end the
// recursion through _multiply_fallback (ops.py:244-245, engine.py:306-307). The non-nil leaf-level
// multiply tasks are exactly the block triples (i,k,j) with A(i,k) and B(k,j) stored, and the C
// block set is the set of (i,j) reached. Here that set is computed per C block-row with a windowed
// dense accumulator in shared memory:
//   1. one block-row index of A and B (stable radix sort by row; quadtree keys are monotone in the
//      column for a fixed row, so each row comes out k-ascending),
//   2. k_sym_count:    per row i -> #distinct j, #triples,
//   3. k_sym_emit_c:   per row i -> C keys in j order + per-C triple counts,
//   4. radix sort of C keys into quadtree-key order, exclusive scan of counts -> c_tptr,
//   5. k_sym_emit_tri: per row i -> (a_index, b_index) triples at their final positions, k
//      ascending within each C block (BlockSparseLeaf.multiply's k loop, block_sparse.py:121-129).
#include <stdlib.h>

#include <cub/cub.cuh>

#include "qm_common.cuh"

namespace qm {
namespace {

constexpr int kWin = 4096;   // j-window of the per-row accumulator (slots)
constexpr int kNT = 256;     // threads per row CTA
constexpr int kPer = kWin / kNT;

// Row keys of both operands in one array: A entry t -> row(t), B entry t -> nbg + row(t); the
// value carried through the sort is the entry's index within its own operand.
__global__ void k_decode_rows(const uint64_t *a_keys, int64_t nA, const uint64_t *b_keys, int64_t nB,
                              int64_t nbg, int nbl, int lbits, uint32_t *rowkey, uint32_t *val,
                              unsigned int *done) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *done = 0u;  // k_sym_count's completion ticket
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < nA + nB;
       x += (int64_t)gridDim.x * blockDim.x) {
    const bool is_b = x >= nA;
    const int64_t t = is_b ? x - nA : x;
    uint32_t bi, bj;
    qkey_decode(is_b ? b_keys[t] : a_keys[t], nbl, lbits, &bi, &bj);
    rowkey[x] = bi + (is_b ? (uint32_t)nbg : 0u);
    val[x] = (uint32_t)t;
  }
}

// After the stable sort by row key: column of every sorted entry (x < n), and the row pointers
// rp[r] = first sorted position with row key >= r, r in [0, 2*nbg] (A rows, then B rows).
// Also gathers the support mask of every sorted entry (A entries: nonzero-column mask, B entries:
// nonzero-row mask; all ones when the operand has no masks).
__global__ void k_cols_rowptr(const uint64_t *a_keys, const uint64_t *b_keys, const uint32_t *srow,
                              const uint32_t *perm, int64_t n, int64_t nbg, int nbl, int lbits,
                              const uint64_t *a_cmask, const uint64_t *b_rmask, int upper, uint32_t *scol,
                              uint32_t *rp, uint64_t *smask, int *masked) {
  const int64_t span = n > 2 * nbg + 1 ? n : 2 * nbg + 1;
  if (blockIdx.x == 0 && threadIdx.x == 0) *masked = ((a_cmask || b_rmask) ? 1 : 0) | (upper ? 2 : 0);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < span;
       x += (int64_t)gridDim.x * blockDim.x) {
    if (x < n) {
      uint32_t bi, bj;
      const bool is_a = (int64_t)srow[x] < nbg;
      qkey_decode((is_a ? a_keys : b_keys)[perm[x]], nbl, lbits, &bi, &bj);
      scol[x] = bj;
      const uint64_t *m = is_a ? a_cmask : b_rmask;
      if (a_cmask || b_rmask) smask[x] = m ? m[perm[x]] : ~0ull;
    }
    if (x <= 2 * nbg) {
      int64_t lo = 0, hi = n;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if ((int64_t)srow[mid] < x) lo = mid + 1; else hi = mid;
      }
      rp[x] = (uint32_t)lo;
    }
  }
}

// ---- block-level reductions / scans (deterministic, fixed order) ------------------------------

template <class T, class Op>
__device__ T block_reduce(T v, Op op, T *red /* smem[32] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T r = red[0];
  for (int w = 1; w < nw; ++w) r = op(r, red[w]);
  return r;
}

// Exclusive scan of one uint32 per thread; returns the prefix and writes the block total.
__device__ uint32_t block_exclusive_scan(uint32_t v, uint32_t *total, uint32_t *wsum /* smem[32] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  __syncthreads();
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  uint32_t before = 0, tot = 0;
  for (int w = 0; w < nw; ++w) {
    if (w < warp) before += wsum[w];
    tot += wsum[w];
  }
  *total = tot;
  return before + inc - v;
}

// Exclusive scan of one uint64 per thread (block-wide); returns the prefix and the block total.
__device__ uint64_t block_exclusive_scan64(uint64_t v, uint64_t *total, uint64_t *wsum /* smem[32] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint64_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  __syncthreads();
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  uint64_t before = 0, tot = 0;
  for (int w = 0; w < nw; ++w) {
    if (w < warp) before += wsum[w];
    tot += wsum[w];
  }
  *total = tot;
  return before + inc - v;
}

// Exclusive scan of x[0, n) into y by one CTA (contiguous chunk per thread, in index order).
__device__ void cta_exclusive_scan64(const uint64_t *x, uint64_t *y, int64_t n, uint64_t *wsum) {
  const int64_t per = (n + blockDim.x - 1) / blockDim.x;
  const int64_t lo0 = (int64_t)threadIdx.x * per;
  const int64_t lo = lo0 < n ? lo0 : n, hi = lo + per < n ? lo + per : n;
  uint64_t part = 0;
  for (int64_t q = lo; q < hi; ++q) part += x[q];
  uint64_t total;
  uint64_t run = block_exclusive_scan64(part, &total, wsum);
  for (int64_t q = lo; q < hi; ++q) {
    const uint64_t v = x[q];
    y[q] = run;
    run += v;
  }
}

struct RowSpan {
  uint32_t a0, a1;     // A row entries
  uint64_t nt;         // triples of the row
  uint32_t jmin, jmax; // column span of the C row
};

// Triple count and column span of C row i (all threads get the result).
__device__ RowSpan row_span(int64_t i, const uint32_t *a_rp, const uint32_t *a_scol,
                            const uint32_t *b_rp, const uint32_t *b_scol, uint64_t *red64,
                            uint32_t *red32) {
  RowSpan s;
  s.a0 = a_rp[i];
  s.a1 = a_rp[i + 1];
  uint64_t nt = 0;
  uint32_t jmin = 0xffffffffu, jmax = 0;
  for (uint32_t x = s.a0 + threadIdx.x; x < s.a1; x += blockDim.x) {
    uint32_t k = a_scol[x];
    uint32_t b0 = b_rp[k], b1 = b_rp[k + 1];
    if (b1 > b0) {
      nt += b1 - b0;
      jmin = min(jmin, b_scol[b0]);
      jmax = max(jmax, b_scol[b1 - 1]);
    }
  }
  s.nt = block_reduce(nt, [](uint64_t a, uint64_t b) { return a + b; }, red64);
  s.jmin = block_reduce(jmin, [](uint32_t a, uint32_t b) { return min(a, b); }, red32);
  s.jmax = block_reduce(jmax, [](uint32_t a, uint32_t b) { return max(a, b); }, red32);
  return s;
}

// First position in b_scol[b0, b1) with column >= j.
__device__ __forceinline__ uint32_t lower_bound_col(const uint32_t *b_scol, uint32_t b0, uint32_t b1,
                                                    uint32_t j) {
  while (b0 < b1) {
    uint32_t mid = (b0 + b1) >> 1;
    if (b_scol[mid] < j) b0 = mid + 1; else b1 = mid;
  }
  return b0;
}

// Flags word of the symbolic workspace (k_cols_rowptr, k_tile_cut): bit 0 support masks given,
// bit 1 upper variant, bit 2 key-ranged (a multi-GPU rank's own C key range in krange[0..1]).
constexpr int kFlagMasked = 1, kFlagUpper = 2, kFlagRanged = 4;

// Column interval [*jlo, *jhi) of block row i whose quadtree keys lie in [klo, khi): keys are
// monotone in the column for a fixed row, so it is one interval (binary searches over j).
__device__ __forceinline__ void row_key_cols(uint32_t i, uint64_t klo, uint64_t khi, int64_t nbg, int nbl,
                                             int lbits, uint32_t *jlo, uint32_t *jhi) {
  uint32_t lo = 0, hi = (uint32_t)nbg;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (qkey(i, mid, nbl, lbits) < klo) lo = mid + 1; else hi = mid;
  }
  *jlo = lo;
  hi = (uint32_t)nbg;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (qkey(i, mid, nbl, lbits) < khi) lo = mid + 1; else hi = mid;
  }
  *jhi = lo;
}

// Applies the per-row column restrictions of the workspace flags to a row span: the upper variant
// (leaves li <= lj) and a rank's key range (per-row column bounds rb[i] = (jlo, jhi), k_row_bounds).
// Returns false when the row has nothing left; *raised = the first column moved past the row's own
// first column (the pair loops must then binary-search their B rows' start).
__device__ __forceinline__ bool clamp_row(RowSpan &s, int64_t i, int flags, const uint2 *rb, int nbl,
                                          bool *raised) {
  const uint32_t j0 = s.jmin;
  if (flags & kFlagUpper) s.jmin = max(s.jmin, (uint32_t)((i / nbl) * nbl));
  if (flags & kFlagRanged) {
    const uint2 b = rb[i];
    s.jmin = max(s.jmin, b.x);
    if (b.y == 0) return false;
    s.jmax = min(s.jmax, b.y - 1u);
  }
  *raised = s.jmin > j0;
  return s.nt > 0 && s.jmin <= s.jmax;
}

// A ranged row with no column in the rank's key range (skipped before any of its work).
__device__ __forceinline__ bool row_out_of_range(int64_t i, int flags, const uint2 *rb) {
  if (!(flags & kFlagRanged)) return false;
  const uint2 b = rb[i];
  return b.x >= b.y;
}

// Calls f(x, y, j) for every pair (A entry x of the row, B entry y of row k(x)) whose column j is
// inside [wbase, wbase + kWin). Warps take A entries, lanes take B entries; no ordering.
// Only pairs whose supports meet are visited: A(i,k)'s nonzero columns and B(k,j)'s nonzero rows
// (smask) must share a bit, else the block product is exactly zero -- no triple is emitted for it,
// and a C block none of whose products survive is never created (it would be an exact-zero block,
// dropped by _set_block anyway).
template <class F>
__device__ void for_window_pairs(const RowSpan &s, uint32_t wbase, bool multi, const uint32_t *a_scol,
                                 const uint32_t *b_rp, const uint32_t *b_scol, const uint64_t *a_smask,
                                 const uint64_t *b_smask, bool masked, F f) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t wend = min(wbase + (uint32_t)kWin, s.jmax + 1u);  // s.jmax: the row's (clamped) last column
  for (uint32_t x = s.a0 + warp; x < s.a1; x += nw) {
    uint32_t k = a_scol[x];
    const uint64_t am = masked ? a_smask[x] : ~0ull;
    uint32_t b0 = b_rp[k], b1 = b_rp[k + 1];
    if (multi) b0 = lower_bound_col(b_scol, b0, b1, wbase);
    for (uint32_t y = b0 + lane; y < b1; y += 32) {
      uint32_t j = b_scol[y];
      if (j >= wend) break;
      if (!masked || (am & b_smask[y])) f(x, y, j);
    }
  }
}

// Per row i: cnt[i] = C blocks, cnt[nbg + i] = triples. The last CTA to finish (ticket on `done`,
// zeroed by k_decode_rows) scans cnt into off (C-row offsets, then triple-row offsets) and writes
// the totals (nC, nT) into the caller's mapped host buffer -- one launch instead of count + scan +
// read-back.
__global__ void __launch_bounds__(kNT) k_sym_count(const uint32_t *a_rp, const uint32_t *a_scol,
                                                   const uint32_t *b_rp, const uint32_t *b_scol,
                                                   const uint64_t *a_smask, const uint64_t *b_smask,
                                                   const int *masked_flag,
                                                   const uint2 *rb, int64_t nbg, int nbl, int lbits,
                                                   uint64_t *cnt, uint64_t *off, unsigned int *done,
                                                   volatile int64_t *host_tot) {
  __shared__ uint32_t bm[kWin / 32];
  __shared__ uint64_t red64[32];
  __shared__ uint32_t red32[32];
  __shared__ bool last;
  const int flags = *masked_flag;
  const bool masked = (flags & kFlagMasked) != 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt[2 * nbg] = 0;  // exclusive-scan tail
  for (int64_t i = blockIdx.x; i < nbg; i += gridDim.x) {
    uint32_t total = 0;
    uint64_t ntri = 0;  // surviving triples of the row (<= s.nt, the structural count)
    bool raised = false;
    RowSpan s;
    if (!row_out_of_range(i, flags, rb)) s = row_span(i, a_rp, a_scol, b_rp, b_scol, red64, red32);
    else s.nt = 0;
    if (s.nt > 0 && clamp_row(s, i, flags, rb, nbl, &raised)) {
      const bool multi = (s.jmax - s.jmin) >= (uint32_t)kWin;
      for (uint64_t wb = s.jmin; wb <= s.jmax; wb += kWin) {
        const uint32_t wbase = (uint32_t)wb;
        for (int w = threadIdx.x; w < kWin / 32; w += blockDim.x) bm[w] = 0u;
        __syncthreads();
        uint64_t mine = 0;
        for_window_pairs(s, wbase, multi || raised, a_scol, b_rp, b_scol, a_smask, b_smask, masked,
                         [&](uint32_t, uint32_t, uint32_t j) {
          uint32_t o = j - wbase;
          atomicOr(&bm[o >> 5], 1u << (o & 31));
          ++mine;
        });
        __syncthreads();
        uint32_t c = 0;
        for (int w = threadIdx.x; w < kWin / 32; w += blockDim.x) c += __popc(bm[w]);
        total += block_reduce(c, [](uint32_t a, uint32_t b) { return a + b; }, red32);
        ntri += block_reduce(mine, [](uint64_t a, uint64_t b) { return a + b; }, red64);
      }
    }
    if (threadIdx.x == 0) {
      cnt[i] = total;
      cnt[nbg + i] = ntri;
    }
    __syncthreads();
  }
  __threadfence();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  cta_exclusive_scan64((const uint64_t *)cnt, off, 2 * nbg + 1, red64);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t n_c = ((volatile uint64_t *)off)[nbg], tail = ((volatile uint64_t *)off)[2 * nbg];
    host_tot[0] = (int64_t)n_c;
    host_tot[1] = (int64_t)(tail - n_c);
    __threadfence_system();
  }
}

__global__ void __launch_bounds__(kNT) k_sym_emit_c(const uint32_t *a_rp, const uint32_t *a_scol,
                                                    const uint32_t *b_rp, const uint32_t *b_scol,
                                                    const uint64_t *a_smask, const uint64_t *b_smask,
                                                    const int *masked_flag,
                                                    const uint2 *rb, int64_t nbg, int nbl, int lbits,
                                                    const uint64_t *rowC_off, uint64_t *rm_key,
                                                    uint32_t *rm_cnt, uint32_t *rm_iota, unsigned int *done,
                                                    unsigned long long *bitmap) {
  __shared__ uint32_t cnt[kWin];
  __shared__ uint64_t red64[32];
  __shared__ uint32_t red32[32];
  if (blockIdx.x == 0 && threadIdx.x == 0) *done = 0u;  // k_inv_counts' completion ticket
  const int flags = *masked_flag;
  const bool masked = (flags & kFlagMasked) != 0;
  for (int64_t i = blockIdx.x; i < nbg; i += gridDim.x) {
    if (rowC_off[i + 1] == rowC_off[i]) continue;  // no C block in this row (block-uniform)
    RowSpan s = row_span(i, a_rp, a_scol, b_rp, b_scol, red64, red32);
    bool raised = false;
    if (clamp_row(s, i, flags, rb, nbl, &raised)) {
      uint64_t out = rowC_off[i];
      const bool multi = (s.jmax - s.jmin) >= (uint32_t)kWin;
      for (uint64_t wb = s.jmin; wb <= s.jmax; wb += kWin) {
        const uint32_t wbase = (uint32_t)wb;
        for (int w = threadIdx.x; w < kWin; w += blockDim.x) cnt[w] = 0u;
        __syncthreads();
        for_window_pairs(s, wbase, multi || raised, a_scol, b_rp, b_scol, a_smask, b_smask, masked,
                         [&](uint32_t, uint32_t, uint32_t j) { atomicAdd(&cnt[j - wbase], 1u); });
        __syncthreads();
        const int s0 = threadIdx.x * kPer;
        uint32_t mine = 0;
#pragma unroll
        for (int q = 0; q < kPer; ++q) mine += cnt[s0 + q] != 0u;
        uint32_t total;
        uint32_t pos = block_exclusive_scan(mine, &total, red32);
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
          uint32_t c = cnt[s0 + q];
          if (c) {
            const uint64_t key = qkey((uint32_t)i, wbase + s0 + q, nbl, lbits);
            rm_key[out + pos] = key;
            if (bitmap) atomicOr(&bitmap[key >> 6], 1ull << (key & 63ull));  // rank ordering (k_rank_*)
            rm_cnt[out + pos] = c;
            rm_iota[out + pos] = (uint32_t)(out + pos);
            ++pos;
          }
        }
        out += total;
        __syncthreads();
      }
    }
    __syncthreads();
  }
}

// Triples of C row i at their final positions. A entries are taken 32 at a time (a group): every
// pair (A entry x, B entry y) of the group sets bit x-x0 of its C column's slot mask, so the rank of
// a pair among the C block's triples is the cursor plus the set bits below its own -- k order is
// kept without serialising over the A entries.
constexpr int kWinT = 2048;
constexpr int kPerT = kWinT / kNT;  // 8 slots per thread: a byte of one bitmap word
static_assert(kPerT == 8, "slot ownership assumes 8 slots per thread");

__global__ void __launch_bounds__(kNT) k_sym_emit_tri(
    const uint32_t *a_rp, const uint32_t *a_scol, const uint32_t *a_perm, const uint32_t *b_rp,
    const uint32_t *b_scol, const uint32_t *b_perm, const uint64_t *a_smask, const uint64_t *b_smask,
    const int *masked_flag,
    const uint2 *rb, int64_t nbg, int nbl, int lbits, const uint64_t *rowC_off,
    const uint32_t *inv, const int64_t *c_tptr, int64_t t_lo, int64_t t_hi, uint2 *tri) {
  __shared__ uint32_t mask[kWinT];
  __shared__ int64_t cur[kWinT];
  __shared__ uint32_t bm[kWinT / 32];
  __shared__ uint64_t red64[32];
  __shared__ uint32_t red32[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kNT >> 5;
  const int s0 = threadIdx.x * kPerT;
  const bool ranged = t_lo > 0 || t_hi < c_tptr[rowC_off[nbg]];
  const int flags = *masked_flag;
  const bool masked = (flags & kFlagMasked) != 0;
  for (int64_t i = blockIdx.x; i < nbg; i += gridDim.x) {
    if (ranged) {
      // A multi-GPU rank emits one triple range: skip rows none of whose C blocks reach it
      // (their triples are [c_tptr[q], c_tptr[q+1]) for q = inv[row-major index]).
      int64_t lo = INT64_MAX, hi = -1;
      for (uint64_t x = rowC_off[i] + threadIdx.x; x < rowC_off[i + 1]; x += blockDim.x) {
        const uint32_t q = inv[x];
        lo = min(lo, c_tptr[q]);
        hi = max(hi, c_tptr[q + 1]);
      }
      lo = (int64_t)block_reduce((uint64_t)lo, [](uint64_t a, uint64_t b) { return a < b ? a : b; }, red64);
      hi = (int64_t)block_reduce((uint64_t)(hi + 1), [](uint64_t a, uint64_t b) { return a > b ? a : b; },
                                 red64) - 1;
      if (hi <= t_lo || lo >= t_hi) continue;
    }
    if (rowC_off[i + 1] == rowC_off[i]) continue;  // no C block in this row (block-uniform)
    RowSpan s = row_span(i, a_rp, a_scol, b_rp, b_scol, red64, red32);
    bool upper = false;  // the row's first column was raised: binary-search the B rows' start
    if (clamp_row(s, i, flags, rb, nbl, &upper)) {
      uint64_t out = rowC_off[i];
      const bool multi = (s.jmax - s.jmin) >= (uint32_t)kWinT;
      for (uint64_t wb = s.jmin; wb <= s.jmax; wb += kWinT) {
        const uint32_t wbase = (uint32_t)wb;
        const uint32_t wend = min(wbase + (uint32_t)kWinT, s.jmax + 1u);
        if (threadIdx.x < kWinT / 32) bm[threadIdx.x] = 0u;
        __syncthreads();
        // occupied C columns of the window
        for (uint32_t x = s.a0 + warp; x < s.a1; x += nw) {
          uint32_t k = a_scol[x];
          const uint64_t am = masked ? a_smask[x] : ~0ull;
          uint32_t b0 = b_rp[k], b1 = b_rp[k + 1];
          if (multi || upper) b0 = lower_bound_col(b_scol, b0, b1, wbase);
          for (uint32_t y = b0 + lane; y < b1; y += 32) {
            uint32_t j = b_scol[y];
            if (j >= wend) break;
            if (!masked || (am & b_smask[y])) atomicOr(&bm[(j - wbase) >> 5], 1u << ((j - wbase) & 31));
          }
        }
        __syncthreads();
        const uint32_t occ = (bm[s0 >> 5] >> (s0 & 31)) & 0xffu;
        uint32_t total;
        uint32_t pos = block_exclusive_scan((uint32_t)__popc(occ), &total, red32);
#pragma unroll
        for (int q = 0; q < kPerT; ++q)
          if (occ & (1u << q)) cur[s0 + q] = c_tptr[inv[out + pos++]];
        for (uint32_t x0 = s.a0; x0 < s.a1; x0 += 32) {
          const uint32_t xe = min(x0 + 32u, s.a1);
#pragma unroll
          for (int q = 0; q < kPerT; ++q) mask[s0 + q] = 0u;
          __syncthreads();
          for (uint32_t x = x0 + warp; x < xe; x += nw) {
            uint32_t k = a_scol[x];
            const uint64_t am = masked ? a_smask[x] : ~0ull;
            uint32_t b0 = b_rp[k], b1 = b_rp[k + 1];
            if (multi || upper) b0 = lower_bound_col(b_scol, b0, b1, wbase);
            for (uint32_t y = b0 + lane; y < b1; y += 32) {
              uint32_t j = b_scol[y];
              if (j >= wend) break;
              if (!masked || (am & b_smask[y])) atomicOr(&mask[j - wbase], 1u << (x - x0));
            }
          }
          __syncthreads();
          for (uint32_t x = x0 + warp; x < xe; x += nw) {
            const uint32_t k = a_scol[x];
            const uint32_t ai = a_perm[x];
            const uint64_t am = masked ? a_smask[x] : ~0ull;
            const uint32_t below = (1u << (x - x0)) - 1u;
            uint32_t b0 = b_rp[k], b1 = b_rp[k + 1];
            if (multi || upper) b0 = lower_bound_col(b_scol, b0, b1, wbase);
            for (uint32_t y = b0 + lane; y < b1; y += 32) {
              uint32_t j = b_scol[y];
              if (j >= wend) break;
              if (masked && !(am & b_smask[y])) continue;
              const int64_t p = cur[j - wbase] + __popc(mask[j - wbase] & below);
              if (p >= t_lo && p < t_hi) tri[p - t_lo] = make_uint2(ai, b_perm[y]);
            }
          }
          __syncthreads();
#pragma unroll
          for (int q = 0; q < kPerT; ++q)
            if (occ & (1u << q)) cur[s0 + q] += __popc(mask[s0 + q]);
        }
        out += total;
        __syncthreads();
      }
    }
    __syncthreads();
  }
}

// Inverse of the C-key sort permutation and the per-C-block triple counts in quadtree order. For
// small products (scan_tptr) the last CTA to finish also scans the counts into c_tptr (one launch
// instead of this kernel + a CUB scan); `done` is zeroed by k_sym_emit_c.
__global__ void k_inv_counts(const uint32_t *perm, const uint32_t *rm_cnt, int64_t nC, uint32_t *inv,
                             int64_t *cnt_q, int64_t *c_tptr, unsigned int *done) {
  __shared__ uint64_t wsum[32];
  __shared__ bool last;
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt_q[nC] = 0;  // exclusive-scan tail
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nC;
       p += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c = perm[p];
    inv[c] = (uint32_t)p;
    cnt_q[p] = rm_cnt[c];
  }
  if (!c_tptr) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  cta_exclusive_scan64((const uint64_t *)cnt_q, (uint64_t *)c_tptr, nC + 1, wsum);
}

// Rank ordering of the C keys (products whose key space is small: <= 2^22 keys). C keys are
// distinct, so their quadtree order is their rank in the set: k_sym_emit_c marks every key in a bitmap
// of the key space, k_rank_scan turns the bitmap words' popcounts into exclusive prefixes (one
// CTA), and k_rank_place gives every C block its position = prefix of its word + the set bits below
// its own -- the device-wide radix sort's histogram / scan / onesweep passes and memsets (about ten
// launches, ~65 us for C3's 65 K keys) become one memset and two small kernels. Deterministic: the
// result does not depend on the order of the atomics. k_rank_place also writes the per-block
// triple counts in key order and, like k_inv_counts, scans them into c_tptr in its last CTA.
constexpr int kRankMaxBits = 22;
__global__ void __launch_bounds__(1024) k_rank_scan(const unsigned long long *bitmap, int64_t words, uint32_t *prefix) {
  // One CTA; every warp owns a contiguous run of words and reads it 32 words at a time (coalesced).
  __shared__ uint32_t wtot[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int64_t per = ((words + (int64_t)nw * 32 - 1) / ((int64_t)nw * 32)) * 32;
  const int64_t lo = std::min<int64_t>((int64_t)warp * per, words), hi = std::min<int64_t>(lo + per, words);
  uint32_t part = 0;
  for (int64_t q = lo + lane; q < hi; q += 32) part += (uint32_t)__popcll(bitmap[q]);
  part = __reduce_add_sync(0xffffffffu, part);
  if (lane == 0) wtot[warp] = part;
  __syncthreads();
  uint32_t run = 0;
  for (int w = 0; w < warp; ++w) run += wtot[w];
  for (int64_t q0 = lo; q0 < hi; q0 += 32) {
    const int64_t q = q0 + lane;
    const uint32_t c = q < hi ? (uint32_t)__popcll(bitmap[q]) : 0u;
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (q < hi) prefix[q] = run + incl - c;
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
}

__global__ void k_rank_place(const uint64_t *rm_key, const uint32_t *rm_cnt, int64_t nC,
                             const unsigned long long *bitmap, const uint32_t *prefix, uint64_t *c_keys,
                             uint32_t *perm, uint32_t *inv, int64_t *cnt_q, int64_t *c_tptr, unsigned int *done) {
  __shared__ uint64_t wsum[32];
  __shared__ bool last;
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt_q[nC] = 0;  // exclusive-scan tail
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < nC; x += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = rm_key[x];
    const uint64_t w = key >> 6;
    const uint32_t p = prefix[w] + (uint32_t)__popcll(bitmap[w] & ((1ull << (key & 63ull)) - 1ull));
    c_keys[p] = key;
    perm[p] = (uint32_t)x;
    inv[x] = p;
    cnt_q[p] = rm_cnt[x];
  }
  if (!c_tptr) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  cta_exclusive_scan64((const uint64_t *)cnt_q, (uint64_t *)c_tptr, nC + 1, wsum);
}

// Small products (nC <= kSmallSortMax): the C-key sort, the inverse permutation, the per-block
// triple counts and their scan into c_tptr in ONE launch of one CTA (a block radix sort in shared
// memory) instead of the device-wide radix sort's histogram / scan / onesweep passes + memsets +
// k_inv_counts -- about ten launches, which for ~1-8 K C blocks cost more than the sorting itself.
// Stable like the device-wide sort (padding keys sort last), so the order is the same.
constexpr int kSmallSortThreads = 512, kSmallSortItems = 16;
constexpr int64_t kSmallSortMax = (int64_t)kSmallSortThreads * kSmallSortItems;
using SmallSort = cub::BlockRadixSort<uint64_t, kSmallSortThreads, kSmallSortItems, uint32_t>;

__global__ void __launch_bounds__(kSmallSortThreads) k_sort_small(const uint64_t *rm_key, const uint32_t *rm_cnt,
                                                                   int64_t nC, int key_bits, uint64_t *c_keys,
                                                                   uint32_t *perm, uint32_t *inv, int64_t *cnt_q,
                                                                   int64_t *c_tptr) {
  extern __shared__ __align__(16) uint8_t sort_smem[];
  typename SmallSort::TempStorage &temp = *reinterpret_cast<typename SmallSort::TempStorage *>(sort_smem);
  __shared__ uint64_t wsum[32];
  const uint64_t pad = key_bits >= 64 ? ~0ull : ((1ull << key_bits) - 1ull);
  uint64_t keys[kSmallSortItems];
  uint32_t vals[kSmallSortItems];
#pragma unroll
  for (int q = 0; q < kSmallSortItems; ++q) {
    const int64_t x = (int64_t)threadIdx.x * kSmallSortItems + q;  // blocked arrangement
    keys[q] = x < nC ? rm_key[x] : pad;
    vals[q] = (uint32_t)x;
  }
  SmallSort(temp).Sort(keys, vals, 0, key_bits);
#pragma unroll
  for (int q = 0; q < kSmallSortItems; ++q) {
    const int64_t r = (int64_t)threadIdx.x * kSmallSortItems + q;
    if (r < nC) {
      c_keys[r] = keys[q];
      perm[r] = vals[q];
      inv[vals[q]] = (uint32_t)r;
      cnt_q[r] = rm_cnt[vals[q]];
    }
  }
  if (threadIdx.x == 0) cnt_q[nC] = 0;
  __threadfence_block();
  __syncthreads();
  cta_exclusive_scan64((const uint64_t *)cnt_q, (uint64_t *)c_tptr, nC + 1, wsum);
}

// ---- multi-GPU partition of the symbolic phase ------------------------------------------------
// Work per C tile (aligned square of 2^shift leaves per side, Morton tile code). One warp per A
// entry (i, k): the lanes read B row k's entries 32 at a time (coalesced), and since the row's
// columns ascend, the lanes of one tile column form a contiguous run -- one match + reduce per run
// and one atomic per (entry, tile). Weight of a pair: 1 (structural triple) without support masks;
// with masks, the number of 16-row k panels where A(i,k)'s columns and B(k,j)'s rows meet (0: the
// pair is skipped as exactly zero), i.e. the k depth the numeric kernel executes -- so ranks are
// balanced on executed work, not on structural triples. (Balance only: every rank still filters
// its own pairs exactly.) Host twin: distributed.tile_partition.
__device__ __forceinline__ uint32_t panel_groups(uint64_t m) {
  return (uint32_t)((m & 0xffffull) != 0) + (uint32_t)(((m >> 16) & 0xffffull) != 0) +
         (uint32_t)(((m >> 32) & 0xffffull) != 0) + (uint32_t)((m >> 48) != 0);
}

__global__ void k_tile_work(const uint32_t *srow, const uint32_t *a_scol, const uint64_t *a_smask,
                            const int *masked_flag, int64_t nA, const uint32_t *b_rp, const uint32_t *b_scol,
                            const uint64_t *b_smask, int nbl, int shift, uint64_t *tiles) {
  const uint32_t tw = (uint32_t)nbl << shift;  // tile width in blocks
  const bool masked = (*masked_flag & kFlagMasked) != 0;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t x = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); x < nA; x += nwarps) {
    const uint32_t i = srow[x], k = a_scol[x];
    const uint32_t b0 = b_rp[k], b1 = b_rp[k + 1];
    const uint64_t am = masked ? a_smask[x] : ~0ull;
    const uint64_t I = spread_bits((i / (uint32_t)nbl) >> shift) << 1;
    for (uint32_t base = b0; base < b1; base += 32) {
      const uint32_t y = base + lane;
      const bool valid = y < b1;
      const uint32_t J = valid ? b_scol[y] / tw : 0xffffffffu;
      const uint32_t w = !valid ? 0u : masked ? panel_groups(am & b_smask[y]) : 1u;
      const uint32_t peers = __match_any_sync(0xffffffffu, J);
      const uint32_t sum = __reduce_add_sync(peers, w);
      if (valid && sum && lane == __ffs(peers) - 1)
        atomicAdd((unsigned long long *)&tiles[I | spread_bits(J)], (unsigned long long)sum);
    }
  }
}

// One CTA: prefix of the tile work in Morton order, cut into `world` contiguous tile ranges of
// (nearly) equal work (the first tile whose exclusive prefix reaches r*W/world starts rank r, as
// distributed.partition cuts c_tptr), and this rank's C key range [krange[0], krange[1]) -- a union
// of whole quadtree subtrees, so C stays a contiguous Morton range per rank.
__global__ void __launch_bounds__(kNT) k_tile_cut(const uint64_t *prefix, int64_t ntiles,
                                                  int world, int rank, int kshift, uint64_t *krange,
                                                  uint64_t *key_cuts, int *flags, volatile int64_t *host_out) {
  const uint64_t W = prefix[ntiles];  // exclusive prefix of the tile work (tail = total)
  for (int r = threadIdx.x; r <= world; r += blockDim.x) {
    int64_t cut;
    if (r == 0) {
      cut = 0;
    } else if (r == world) {
      cut = ntiles;
    } else {
      const uint64_t target = (uint64_t)((unsigned __int128)W * (unsigned)r / (unsigned)world);
      int64_t lo = 0, hi = ntiles;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (prefix[mid] < target) lo = mid + 1; else hi = mid;
      }
      cut = lo;
    }
    const uint64_t key = (uint64_t)cut << kshift;
    if (key_cuts) key_cuts[r] = key;
    if (r == rank) krange[0] = key;
    if (r == rank + 1) krange[1] = key;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *flags |= kFlagRanged;
    __threadfence();
    host_out[2] = (int64_t)krange[0];
    host_out[3] = (int64_t)krange[1];
    host_out[4] = (int64_t)W;
  }
}

// Per-row column bounds of this rank's key range: rb[i] = (first, end) column of row i whose keys
// lie in [krange[0], krange[1]) -- one interval, keys being monotone in the column.
__global__ void k_row_bounds(const uint64_t *krange, int64_t nbg, int nbl, int lbits, uint2 *rb) {
  const uint64_t klo = krange[0], khi = krange[1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nbg; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t jlo, jhi;
    row_key_cols((uint32_t)i, klo, khi, nbg, nbl, lbits, &jlo, &jhi);
    rb[i] = make_uint2(jlo, jhi);
  }
}

inline int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (int)g;
}

inline int bits_for(uint64_t maxval) {
  int b = 1;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

// Workspace of the count phase (persists into the fill phase). Both operands share one row index:
// sorted entries [0, nA) are A's rows, [nA, nA+nB) B's; rp has 2*nbg+1 entries (a_rp = rp,
// b_rp = rp + nbg); positions index scol/perm of either operand directly.
struct SymWs {
  uint32_t *rowkey, *val, *srow, *perm, *scol, *rp;
  uint64_t *smask;  // support mask of every sorted entry (see k_cols_rowptr)
  int *masked;      // 1 when the count phase was given support masks
  uint64_t *cnt;   // [2*nbg+1]: C blocks per row, triples per row, 0
  uint64_t *off;   // exclusive scan of cnt: rowC_off = off, nC = off[nbg], nT = off[2nbg] - off[nbg]
  unsigned int *done;  // k_sym_count's completion ticket
  uint64_t *krange;    // [2]: this rank's C key range (flag kFlagRanged; qm_spgemm_count_part)
  uint2 *rb;           // [nbg]: per-row column bounds of the key range (k_row_bounds)
  uint64_t *tiles;     // [4^tile_levels]: structural triples per C tile (qm_spgemm_count_part)
  int tile_levels;
  void *cub;
  size_t cub_bytes;
};

size_t cub_bytes_count(int64_t n, int64_t nbg) {
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                  (uint32_t *)nullptr, (uint32_t *)nullptr, (int64_t)n, 0, 32);
  cub::DeviceScan::ExclusiveSum(nullptr, b, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                (int64_t)(2 * nbg + 1));
  return std::max(a, b);
}

// C tiles of the multi-GPU partition: aligned squares of 2^(depth - tile_levels) leaves per side,
// 4^tile_levels of them in Morton order (at most 65536).
constexpr int kMaxTileLevels = 8;
inline int tile_levels_for(const Geometry &g) { return g.depth < kMaxTileLevels ? g.depth : kMaxTileLevels; }

size_t cub_bytes_scan(int64_t ntiles) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (uint64_t *)nullptr, (uint64_t *)nullptr, ntiles + 1);
  return b;
}

SymWs carve_sym(Carver &cv, int64_t nA, int64_t nB, int64_t nbg, int tile_levels) {
  SymWs w;
  const int64_t n = nA + nB;
  w.rowkey = cv.take<uint32_t>(n); w.val = cv.take<uint32_t>(n); w.srow = cv.take<uint32_t>(n);
  w.perm = cv.take<uint32_t>(n); w.scol = cv.take<uint32_t>(n);
  w.smask = cv.take<uint64_t>(n);
  w.masked = cv.take<int>(1);
  w.rp = cv.take<uint32_t>(2 * nbg + 1);
  w.cnt = cv.take<uint64_t>(2 * nbg + 1);
  w.off = cv.take<uint64_t>(2 * nbg + 1);
  w.done = cv.take<unsigned int>(1);
  w.krange = cv.take<uint64_t>(2);
  w.rb = cv.take<uint2>(nbg);
  w.tile_levels = tile_levels;
  w.tiles = cv.take<uint64_t>(2 * ((size_t)1 << (2 * tile_levels)) + 2);  // work [+ tail], prefix
  w.cub_bytes = std::max(cub_bytes_count(n, nbg), cub_bytes_scan((int64_t)1 << (2 * tile_levels)));
  w.cub = cv.take<char>(w.cub_bytes);
  return w;
}

struct FillWs {
  uint64_t *rm_key;
  uint32_t *rm_cnt, *rm_iota, *perm, *inv;
  int64_t *cnt_q;
  unsigned int *done;
  void *cub;
  size_t cub_bytes;
  unsigned long long *bitmap;  // rank ordering: one bit per key of the key space (NULL: not used)
  uint32_t *prefix;
  int64_t words;
};

// QM_RANK_ORDER=0: the C keys are always ordered by a sort (A/B measurements, tests).
bool rank_order_enabled() {
  const char *e = getenv("QM_RANK_ORDER");
  return !(e && e[0] == '0');
}

// QM_SMALL_SORT=0: small products use the device-wide sort too (A/B measurements).
bool small_sort_enabled() {
  const char *e = getenv("QM_SMALL_SORT");
  return !(e && e[0] == '0');
}

// Products with at most this many C blocks scan c_tptr inside k_inv_counts (one CTA).
constexpr int64_t kFusedTptrScanMax = 32768;

FillWs carve_fill(Carver &cv, int64_t nC, int key_bits) {
  FillWs w;
  w.rm_key = cv.take<uint64_t>(nC);
  w.rm_cnt = cv.take<uint32_t>(nC);
  w.rm_iota = cv.take<uint32_t>(nC);
  w.perm = cv.take<uint32_t>(nC);
  w.inv = cv.take<uint32_t>(nC);
  w.cnt_q = cv.take<int64_t>(nC + 1);
  w.done = cv.take<unsigned int>(1);
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                  (uint32_t *)nullptr, (uint32_t *)nullptr, (int64_t)nC, 0, key_bits);
  cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t *)nullptr, (int64_t *)nullptr, (int64_t)nC + 1);
  w.cub_bytes = std::max(a, b);
  w.cub = cv.take<char>(w.cub_bytes);
  // rank ordering: key space of at most 2^22 keys and not much larger than the C set (the bitmap is
  // zeroed and scanned per product); always carved when eligible, so the workspace size does not
  // depend on the environment switches
  w.bitmap = nullptr;
  w.prefix = nullptr;
  w.words = 0;
  if (key_bits <= kRankMaxBits && nC > 0) {
    const int64_t words = ((int64_t)1 << std::max(key_bits, 6)) / 64;
    if (words <= 64 * nC + 1024) {
      w.words = words;
      w.bitmap = cv.take<unsigned long long>(words);
      w.prefix = cv.take<uint32_t>(words);
    }
  }
  return w;
}

// Block-row index of both operands: one stable radix sort by row key (quadtree keys are monotone
// in the column for a fixed row, so every row comes out k-ascending), columns, row pointers.
int build_rows(const uint64_t *a_keys, const uint64_t *a_cmask, int64_t nA, const uint64_t *b_keys,
               const uint64_t *b_rmask, int64_t nB, int upper, const Geometry &g, const SymWs &w, cudaStream_t st) {
  const int64_t n = nA + nB;
  if (n > 0) {
    k_decode_rows<<<grid_for(n), 256, 0, st>>>(a_keys, nA, b_keys, nB, g.nbg, g.nbl, g.lbits,
                                                w.rowkey, w.val, w.done);
    QM_LAUNCHED("k_decode_rows");
    size_t tb = w.cub_bytes;
    QM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.cub, tb, w.rowkey, w.srow, w.val, w.perm, n, 0,
                                                bits_for((uint64_t)(2 * g.nbg - 1)), st));
    QM_CUDA_TRY(cudaGetLastError());
  }
  k_cols_rowptr<<<grid_for(std::max<int64_t>(n, 2 * g.nbg + 1)), 256, 0, st>>>(
      a_keys, b_keys, w.srow, w.perm, n, g.nbg, g.nbl, g.lbits, a_cmask, b_rmask, upper, w.scol, w.rp, w.smask,
      w.masked);
  QM_LAUNCHED("k_cols_rowptr");
  return QM_OK;
}

int row_grid(int64_t nbg) {
  int64_t g = nbg;
  if (g > 148 * 64) g = 148 * 64;
  return (int)std::max<int64_t>(g, 1);
}

// One operand's block-row index (the row-sorted view of a quadtree-ordered block set): positions
// of the sorted entries, their rows and columns, the row pointers, and the support mask each entry
// contributes to a product (its column mask as A, its row mask as B).
struct Ix {
  const uint32_t *rp = nullptr, *row = nullptr, *col = nullptr, *perm = nullptr;
  const uint64_t *mask = nullptr;
};

// The two operands' indexes inside the symbolic workspace (the joint sort of build_rows): A's
// entries are [0, nA), B's follow, and B's row pointers are the second half of rp.
void ws_ix(const SymWs &w, const Geometry &g, int64_t nA, Ix *a, Ix *b) {
  (void)nA;
  a->rp = w.rp;
  a->row = w.srow;
  a->col = w.scol;
  a->perm = w.perm;
  a->mask = w.smask;
  b->rp = w.rp + g.nbg;
  b->row = w.srow;
  b->col = w.scol;
  b->perm = w.perm;
  b->mask = w.smask;
}

Ix from_abi(const qm_row_index *r) {
  Ix x;
  x.rp = r->rowptr;
  x.row = r->row;
  x.col = r->col;
  x.perm = r->perm;
  x.mask = r->mask;
  return x;
}

// Workspace flags and the completion ticket when the row indexes come from the caller (no
// k_decode_rows / k_cols_rowptr to set them).
__global__ void k_sym_init(int *flags, int value, unsigned int *done) {
  *flags = value;
  *done = 0u;
}

// Row index of one operand: columns, rows and the row pointers of the row-sorted entries, and the
// column / row masks in that order (either may be NULL).
__global__ void k_ix_cols(const uint64_t *keys, const uint32_t *srow, const uint32_t *perm, int64_t n, int64_t nbg,
                          int nbl, int lbits, const uint64_t *masks, uint32_t *col, uint32_t *row, uint32_t *rp,
                          uint64_t *cmask_sorted, uint64_t *rmask_sorted) {
  const int64_t span = n > nbg + 1 ? n : nbg + 1;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < span; x += (int64_t)gridDim.x * blockDim.x) {
    if (x < n) {
      uint32_t bi, bj;
      const uint32_t t = perm[x];
      qkey_decode(keys[t], nbl, lbits, &bi, &bj);
      col[x] = bj;
      row[x] = bi;
      if (cmask_sorted) cmask_sorted[x] = masks ? masks[n + t] : ~0ull;
      if (rmask_sorted) rmask_sorted[x] = masks ? masks[t] : ~0ull;
    }
    if (x <= nbg) {
      int64_t lo = 0, hi = n;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)srow[mid] < x) lo = mid + 1; else hi = mid;
      }
      rp[x] = (uint32_t)lo;
    }
  }
}

}  // namespace
}  // namespace qm

using namespace qm;

extern "C" size_t qm_spgemm_workspace_bytes(const qm_layout *layout, int64_t nA, int64_t nB) {
  Geometry g;
  if (make_geometry(layout, &g) != QM_OK) return 0;
  Carver cv(nullptr, 0);
  carve_sym(cv, nA, nB, g.nbg, tile_levels_for(g));
  return cv.off;
}

namespace {
// Count phase over two row indexes (built into the workspace by build_rows, or the caller's).
int count_core(const Geometry &g, const Ix &a, int64_t nA, const Ix &b, int64_t nB, int world, int rank,
               const SymWs &w, int64_t *n_c_out, int64_t *n_triples_out, int64_t *part_out, uint64_t *key_cuts,
               cudaStream_t st) {
  int64_t *host_tot = nullptr, *dev_tot = nullptr;
  int rc = mapped_i64(&host_tot, &dev_tot);
  if (rc != QM_OK) return rc;
  if (world > 0) {  // multi-GPU partition: this rank's C key range from the tile work
    const int tl = w.tile_levels;
    const int64_t ntiles = (int64_t)1 << (2 * tl);
    QM_CUDA_TRY(cudaMemsetAsync(w.tiles, 0, (size_t)(ntiles + 1) * sizeof(uint64_t), st));
    if (nA > 0) {
      k_tile_work<<<grid_for(nA * 32), 256, 0, st>>>(a.row, a.col, a.mask, w.masked, nA, b.rp, b.col, b.mask, g.nbl,
                                                      g.depth - tl, w.tiles);
      QM_LAUNCHED("k_tile_work");
    }
    uint64_t *prefix = w.tiles + ntiles + 1;
    size_t tb = w.cub_bytes;
    QM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(w.cub, tb, w.tiles, prefix, ntiles + 1, st));
    k_tile_cut<<<1, kNT, 0, st>>>(prefix, ntiles, world, rank, 2 * (g.depth - tl) + 2 * g.lbits, w.krange,
                                   key_cuts, w.masked, dev_tot);
    QM_LAUNCHED("k_tile_cut");
    k_row_bounds<<<grid_for(g.nbg), 256, 0, st>>>(w.krange, g.nbg, g.nbl, g.lbits, w.rb);
    QM_LAUNCHED("k_row_bounds");
  }
  k_sym_count<<<row_grid(g.nbg), kNT, 0, st>>>(a.rp, a.col, b.rp, b.col, a.mask, b.mask, w.masked, w.rb, g.nbg,
                                               g.nbl, g.lbits, w.cnt, w.off, w.done, dev_tot);
  QM_LAUNCHED("k_sym_count");
  QM_CUDA_TRY(cudaStreamSynchronize(st));
  volatile int64_t *ht = (volatile int64_t *)host_tot;
  uint64_t tot[2] = {(uint64_t)ht[0], (uint64_t)ht[1]};
  if (tot[0] >= (1ull << 32)) {
    set_error("product has %llu C blocks; this build indexes C with 32 bits", (unsigned long long)tot[0]);
    return QM_ERR_UNSUPPORTED;
  }
  *n_c_out = (int64_t)tot[0];
  *n_triples_out = (int64_t)tot[1];
  if (part_out) {
    part_out[0] = ht[2];
    part_out[1] = ht[3];
    part_out[2] = ht[4];
  }
  return QM_OK;
}

int count_setup(const qm_layout *layout, int64_t nA, int64_t nB, void *ws, size_t ws_bytes, int64_t *n_c_out,
                int64_t *n_triples_out, Geometry *g, SymWs *w) {
  int rc = make_geometry(layout, g);
  if (rc != QM_OK) return rc;
  if (nA < 0 || nB < 0 || nA + nB >= (int64_t)1 << 32 || !n_c_out || !n_triples_out) {
    set_error("qm_spgemm_count: bad sizes or output pointers");
    return QM_ERR_INVALID;
  }
  Carver cv(ws, ws_bytes);
  *w = carve_sym(cv, nA, nB, g->nbg, tile_levels_for(*g));
  if (!cv.ok() || !ws) {
    set_error("qm_spgemm_count: workspace %zu bytes < required %zu", ws_bytes, cv.off);
    return QM_ERR_WORKSPACE;
  }
  *n_c_out = 0;
  *n_triples_out = 0;
  return QM_OK;
}

int count_impl(const qm_layout *layout, const uint64_t *a_keys, const uint64_t *a_cmask, int64_t nA,
               const uint64_t *b_keys, const uint64_t *b_rmask, int64_t nB, int32_t flags, int world, int rank,
               void *ws, size_t ws_bytes, int64_t *n_c_out, int64_t *n_triples_out, int64_t *part_out,
               uint64_t *key_cuts, void *stream) {
  Geometry g;
  SymWs w;
  int rc = count_setup(layout, nA, nB, ws, ws_bytes, n_c_out, n_triples_out, &g, &w);
  if (rc != QM_OK) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  rc = build_rows(a_keys, a_cmask, nA, b_keys, b_rmask, nB, (flags & QM_SPGEMM_UPPER) ? 1 : 0, g, w, st);
  if (rc != QM_OK) return rc;
  if (nA + nB == 0) QM_CUDA_TRY(cudaMemsetAsync(w.done, 0, sizeof(unsigned int), st));  // no k_decode_rows
  Ix a, b;
  ws_ix(w, g, nA, &a, &b);
  return count_core(g, a, nA, b, nB, world, rank, w, n_c_out, n_triples_out, part_out, key_cuts, st);
}
}  // namespace

extern "C" int qm_spgemm_count_masked(const qm_layout *layout, const uint64_t *a_keys, const uint64_t *a_cmask,
                                      int64_t nA, const uint64_t *b_keys, const uint64_t *b_rmask, int64_t nB,
                                      int32_t flags, void *ws, size_t ws_bytes, int64_t *n_c_out,
                                      int64_t *n_triples_out, void *stream) {
  return count_impl(layout, a_keys, a_cmask, nA, b_keys, b_rmask, nB, flags, 0, 0, ws, ws_bytes, n_c_out,
                    n_triples_out, nullptr, nullptr, stream);
}

extern "C" int qm_spgemm_count_part(const qm_layout *layout, const uint64_t *a_keys, const uint64_t *a_cmask,
                                    int64_t nA, const uint64_t *b_keys, const uint64_t *b_rmask, int64_t nB,
                                    int32_t world, int32_t rank, void *ws, size_t ws_bytes, int64_t *n_c_out,
                                    int64_t *n_triples_out, int64_t *part_out, uint64_t *key_cuts, void *stream) {
  if (world < 1 || rank < 0 || rank >= world || !part_out) {
    set_error("qm_spgemm_count_part: bad world %d / rank %d", world, rank);
    return QM_ERR_INVALID;
  }
  return count_impl(layout, a_keys, a_cmask, nA, b_keys, b_rmask, nB, 0, world, rank, ws, ws_bytes, n_c_out,
                    n_triples_out, part_out, key_cuts, stream);
}

extern "C" int qm_spgemm_count(const qm_layout *layout, const uint64_t *a_keys, int64_t nA,
                               const uint64_t *b_keys, int64_t nB, void *ws, size_t ws_bytes,
                               int64_t *n_c_out, int64_t *n_triples_out, void *stream) {
  return qm_spgemm_count_masked(layout, a_keys, nullptr, nA, b_keys, nullptr, nB, 0, ws, ws_bytes, n_c_out,
                                n_triples_out, stream);
}

// ---- caller-held row indexes (operand metadata: built once per block set, reused by products) ----
extern "C" size_t qm_row_index_workspace_bytes(const qm_layout *layout, int64_t n) {
  Geometry g;
  if (make_geometry(layout, &g) != QM_OK) return 0;
  Carver cv(nullptr, 0);
  cv.take<uint32_t>(std::max<int64_t>(n, 1));  // row keys
  cv.take<uint32_t>(std::max<int64_t>(n, 1));  // iota
  cv.take<uint32_t>(std::max<int64_t>(n, 1));  // sorted rows
  size_t cb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cb, (uint32_t *)nullptr, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                  (uint32_t *)nullptr, std::max<int64_t>(n, 1), 0, 32);
  cv.take<char>(cb);
  cv.take<unsigned int>(1);
  return cv.off;
}

extern "C" int qm_row_index_build(const qm_layout *layout, const uint64_t *keys, int64_t n, const uint64_t *masks,
                            void *ws, size_t ws_bytes, uint32_t *rowptr, uint32_t *row, uint32_t *col, uint32_t *perm,
                            uint64_t *cmask_sorted, uint64_t *rmask_sorted, void *stream) {
  Geometry g;
  int rc = make_geometry(layout, &g);
  if (rc != QM_OK) return rc;
  if (n < 0 || n >= ((int64_t)1 << 32) || !rowptr || (n > 0 && (!keys || !row || !col || !perm))) {
    set_error("qm_row_index_build: bad arguments");
    return QM_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  Carver cv(ws, ws_bytes);
  uint32_t *rowkey = cv.take<uint32_t>(std::max<int64_t>(n, 1));
  uint32_t *iota = cv.take<uint32_t>(std::max<int64_t>(n, 1));
  uint32_t *srow = cv.take<uint32_t>(std::max<int64_t>(n, 1));
  size_t cb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cb, (uint32_t *)nullptr, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                  (uint32_t *)nullptr, std::max<int64_t>(n, 1), 0, 32);
  void *cub_tmp = cv.take<char>(cb);
  unsigned int *done = cv.take<unsigned int>(1);
  if (!cv.ok() || !ws) {
    set_error("qm_row_index_build: workspace %zu bytes < required %zu", ws_bytes, cv.off);
    return QM_ERR_WORKSPACE;
  }
  if (n > 0) {
    k_decode_rows<<<grid_for(n), 256, 0, st>>>(keys, n, nullptr, 0, g.nbg, g.nbl, g.lbits, rowkey, iota, done);
    QM_LAUNCHED("k_decode_rows");
    QM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(cub_tmp, cb, rowkey, srow, iota, perm, n, 0,
                                                bits_for((uint64_t)std::max<int64_t>(g.nbg - 1, 1)), st));
  }
  k_ix_cols<<<grid_for(std::max<int64_t>(n, g.nbg + 1)), 256, 0, st>>>(keys, srow, perm, n, g.nbg, g.nbl, g.lbits,
                                                                        masks, col, row, rowptr, cmask_sorted,
                                                                        rmask_sorted);
  QM_LAUNCHED("k_ix_cols");
  return QM_OK;
}

extern "C" int qm_spgemm_count_ix(const qm_layout *layout, const qm_row_index *a, int64_t nA, const qm_row_index *b,
                                  int64_t nB, int32_t flags, int32_t world, int32_t rank, void *ws, size_t ws_bytes,
                                  int64_t *n_c_out, int64_t *n_triples_out, int64_t *part_out, uint64_t *key_cuts,
                                  void *stream) {
  if (!a || !b || (world > 0 && (rank < 0 || rank >= world || !part_out)) || world < 0) {
    set_error("qm_spgemm_count_ix: bad arguments");
    return QM_ERR_INVALID;
  }
  if ((a->mask == nullptr) != (b->mask == nullptr)) {
    set_error("qm_spgemm_count_ix: give both operands' masks or neither");
    return QM_ERR_INVALID;
  }
  Geometry g;
  SymWs w;
  int rc = count_setup(layout, nA, nB, ws, ws_bytes, n_c_out, n_triples_out, &g, &w);
  if (rc != QM_OK) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  k_sym_init<<<1, 1, 0, st>>>(w.masked, (a->mask ? kFlagMasked : 0) | ((flags & QM_SPGEMM_UPPER) ? kFlagUpper : 0),
                              w.done);
  QM_LAUNCHED("k_sym_init");
  return count_core(g, from_abi(a), nA, from_abi(b), nB, world, rank, w, n_c_out, n_triples_out, part_out, key_cuts,
                    st);
}

extern "C" size_t qm_spgemm_fill_workspace_bytes(const qm_layout *layout, int64_t nC) {
  Geometry g;
  if (make_geometry(layout, &g) != QM_OK) return 0;
  Carver cv(nullptr, 0);
  carve_fill(cv, nC, 2 * (g.depth + g.lbits) > 0 ? 2 * (g.depth + g.lbits) : 1);
  return cv.off;
}

namespace {
// Shared prologue of the fill entry points: carve both workspaces.
int fill_setup(const qm_layout *layout, int64_t nA, int64_t nB, int64_t nC, void *ws, size_t ws_bytes,
               void *fill_ws, size_t fill_ws_bytes, Geometry *g, SymWs *w, FillWs *f, int *key_bits) {
  int rc = make_geometry(layout, g);
  if (rc != QM_OK) return rc;
  Carver cv(ws, ws_bytes);
  *w = carve_sym(cv, nA, nB, g->nbg, tile_levels_for(*g));
  if (!cv.ok() || !ws) {
    set_error("qm_spgemm_fill: workspace too small");
    return QM_ERR_WORKSPACE;
  }
  *key_bits = std::max(1, 2 * (g->depth + g->lbits));
  Carver fv(fill_ws, fill_ws_bytes);
  *f = carve_fill(fv, nC, *key_bits);
  if (!fv.ok() || (nC > 0 && !fill_ws)) {
    set_error("qm_spgemm_fill: fill workspace %zu bytes < required %zu", fill_ws_bytes, fv.off);
    return QM_ERR_WORKSPACE;
  }
  return QM_OK;
}

int fill_keys_core(const Geometry &g, const Ix &a, const Ix &b, int64_t nC, const SymWs &w, const FillWs &f,
                   int key_bits, uint64_t *c_keys, int64_t *c_tptr, cudaStream_t st) {
  if (nC == 0) return cudaMemsetAsync(c_tptr, 0, sizeof(int64_t), st) == cudaSuccess ? QM_OK : QM_ERR_CUDA;
  // (single-CTA sort for the smallest products, rank ordering when the key space is small, else the
  // device-wide radix sort)
  const bool small = nC <= kSmallSortMax && small_sort_enabled();
  const bool rank = f.bitmap != nullptr && rank_order_enabled() && !(small && nC <= 2048);
  if (rank) QM_CUDA_TRY(cudaMemsetAsync(f.bitmap, 0, (size_t)f.words * sizeof(unsigned long long), st));
  k_sym_emit_c<<<row_grid(g.nbg), kNT, 0, st>>>(a.rp, a.col, b.rp, b.col, a.mask, b.mask, w.masked, w.rb, g.nbg,
                                                g.nbl, g.lbits, w.off, f.rm_key, f.rm_cnt, f.rm_iota, f.done,
                                                rank ? f.bitmap : nullptr);
  QM_LAUNCHED("k_sym_emit_c");
  if (rank) {
    k_rank_scan<<<1, 1024, 0, st>>>(f.bitmap, f.words, f.prefix);
    QM_LAUNCHED("k_rank_scan");
    const bool fused = nC <= kFusedTptrScanMax;
    k_rank_place<<<grid_for(nC), 256, 0, st>>>(f.rm_key, f.rm_cnt, nC, f.bitmap, f.prefix, c_keys, f.perm, f.inv,
                                               f.cnt_q, fused ? c_tptr : nullptr, f.done);
    QM_LAUNCHED("k_rank_place");
    if (!fused) {
      size_t tb = f.cub_bytes;
      QM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(f.cub, tb, f.cnt_q, c_tptr, nC + 1, st));
    }
    return QM_OK;
  }
  if (nC <= kSmallSortMax && small_sort_enabled()) {
    static PerDeviceOnce once;
    int rc = once.run([]() -> int {
      QM_CUDA_TRY(cudaFuncSetAttribute(k_sort_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(typename SmallSort::TempStorage)));
      return (int)QM_OK;
    });
    if (rc != QM_OK) return rc;
    k_sort_small<<<1, kSmallSortThreads, sizeof(typename SmallSort::TempStorage), st>>>(
        f.rm_key, f.rm_cnt, nC, key_bits, c_keys, f.perm, f.inv, f.cnt_q, c_tptr);
    QM_LAUNCHED("k_sort_small");
    return QM_OK;
  }
  size_t tb = f.cub_bytes;
  QM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(f.cub, tb, f.rm_key, c_keys, f.rm_iota, f.perm, nC, 0,
                                              key_bits, st));
  const bool fused = nC <= kFusedTptrScanMax;
  k_inv_counts<<<grid_for(nC), 256, 0, st>>>(f.perm, f.rm_cnt, nC, f.inv, f.cnt_q, fused ? c_tptr : nullptr,
                                             f.done);
  QM_LAUNCHED("k_inv_counts");
  if (!fused) {
    tb = f.cub_bytes;
    QM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(f.cub, tb, f.cnt_q, c_tptr, nC + 1, st));
  }
  return QM_OK;
}

int fill_triples_core(const Geometry &g, const Ix &a, const Ix &b, int64_t nC, const SymWs &w, const FillWs &f,
                      const int64_t *c_tptr, int64_t t_lo, int64_t t_hi, uint32_t *tri, cudaStream_t st) {
  if (nC == 0 || t_hi <= t_lo) return QM_OK;
  k_sym_emit_tri<<<row_grid(g.nbg), kNT, 0, st>>>(a.rp, a.col, a.perm, b.rp, b.col, b.perm, a.mask, b.mask,
                                                  w.masked, w.rb, g.nbg, g.nbl, g.lbits, w.off, f.inv, c_tptr, t_lo,
                                                  t_hi, (uint2 *)tri);
  QM_LAUNCHED("k_sym_emit_tri");
  return QM_OK;
}
}  // namespace

extern "C" int qm_spgemm_fill_keys(const qm_layout *layout, int64_t nA, int64_t nB, int64_t nC,
                                   void *ws, size_t ws_bytes, void *fill_ws, size_t fill_ws_bytes,
                                   uint64_t *c_keys, int64_t *c_tptr, void *stream) {
  Geometry g;
  SymWs w;
  FillWs f;
  int key_bits;
  int rc = fill_setup(layout, nA, nB, nC, ws, ws_bytes, fill_ws, fill_ws_bytes, &g, &w, &f, &key_bits);
  if (rc != QM_OK) return rc;
  Ix a, b;
  ws_ix(w, g, nA, &a, &b);
  return fill_keys_core(g, a, b, nC, w, f, key_bits, c_keys, c_tptr, (cudaStream_t)stream);
}

extern "C" int qm_spgemm_fill_triples(const qm_layout *layout, int64_t nA, int64_t nB, int64_t nC,
                                      void *ws, size_t ws_bytes, void *fill_ws, size_t fill_ws_bytes,
                                      const int64_t *c_tptr, int64_t t_lo, int64_t t_hi, uint32_t *tri,
                                      void *stream) {
  Geometry g;
  SymWs w;
  FillWs f;
  int key_bits;
  int rc = fill_setup(layout, nA, nB, nC, ws, ws_bytes, fill_ws, fill_ws_bytes, &g, &w, &f, &key_bits);
  if (rc != QM_OK) return rc;
  Ix a, b;
  ws_ix(w, g, nA, &a, &b);
  return fill_triples_core(g, a, b, nC, w, f, c_tptr, t_lo, t_hi, tri, (cudaStream_t)stream);
}

extern "C" int qm_spgemm_fill(const qm_layout *layout, int64_t nA, int64_t nB, int64_t nC, int64_t nT,
                              void *ws, size_t ws_bytes, void *fill_ws, size_t fill_ws_bytes,
                              uint64_t *c_keys, int64_t *c_tptr, uint32_t *tri, void *stream) {
  int rc = qm_spgemm_fill_keys(layout, nA, nB, nC, ws, ws_bytes, fill_ws, fill_ws_bytes, c_keys, c_tptr,
                               stream);
  if (rc != QM_OK) return rc;
  return qm_spgemm_fill_triples(layout, nA, nB, nC, ws, ws_bytes, fill_ws, fill_ws_bytes, c_tptr, 0, nT,
                                tri, stream);
}

extern "C" int qm_spgemm_fill_ix(const qm_layout *layout, const qm_row_index *a, int64_t nA, const qm_row_index *b,
                                 int64_t nB, int64_t nC, int64_t t_lo, int64_t t_hi, void *ws, size_t ws_bytes,
                                 void *fill_ws, size_t fill_ws_bytes, uint64_t *c_keys, int64_t *c_tptr, uint32_t *tri,
                                 void *stream) {
  if (!a || !b) {
    set_error("qm_spgemm_fill_ix: NULL row index");
    return QM_ERR_INVALID;
  }
  Geometry g;
  SymWs w;
  FillWs f;
  int key_bits;
  int rc = fill_setup(layout, nA, nB, nC, ws, ws_bytes, fill_ws, fill_ws_bytes, &g, &w, &f, &key_bits);
  if (rc != QM_OK) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const Ix ia = from_abi(a), ib = from_abi(b);
  if (c_keys) {  // keys + c_tptr (c_keys NULL: triples only, c_tptr already filled)
    rc = fill_keys_core(g, ia, ib, nC, w, f, key_bits, c_keys, c_tptr, st);
    if (rc != QM_OK) return rc;
  }
  if (tri) return fill_triples_core(g, ia, ib, nC, w, f, c_tptr, t_lo, t_hi, tri, st);
  return QM_OK;
}

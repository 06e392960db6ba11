// Numeric phase for 16x16 blocks (the reference API's default block_size): grouped C blocks.
//
// A 16x16 triple is 8 KFLOP for 4 KB of operands, 2 flop/byte: with one C block per work unit the
// kernel streams every A and B block from L2 once per triple and is bound by L2->SM bandwidth
// (the cp.async kernel reaches ~50% of the DMMA peak). Here a work unit is a *group*: the C blocks
// of R block rows (R = 2 when a leaf has <= 8 blocks per side, else 1) x up to 8 aligned block
// columns of one leaf -- consecutive in quadtree-key order, since a leaf stores its blocks
// row-major (BlockSparseLeaf.encode). A triple (r,k,c) exists iff A(r,k) and B(k,c) do, so one
// pipeline stage per k carries the group's A(r,k) and B(k,c) blocks and feeds every member
// product at that k: up to 16 products for 20 KB (R = 2; 6.6 flop/byte) -- each B block serves
// both rows and each A block all 8 columns.
//
//   merge: the members' k-ascending triple lists are merged into the group's union of k (one
//     entry per k: R A indices and 8 B indices, absent = 0xffffffff) by the kernel's producer warp
//     itself, one entry per pipeline stage (k_group_merge, one warp per group writing an entries
//     array, is the earlier separate pass: QM_G16_MERGE=kernel);
//   k_numeric_group16: warp-specialised like k_numeric_tma (one TMA producer warp, mbarrier ring),
//     4 consumer warps, warp w owns columns w, w+4 of every group row: R x 2 accumulators of
//     16x16 fed only by the entries where both its A row and B column are present (so each C
//     block sums exactly its own triples, k ascending -- the order of BlockSparseLeaf.multiply,
//     block_sparse.py:121-129), and writes the blocks, their sums of squares and exact-zero flags
//     (_set_block, block_sparse.py:37-41) when the group ends.
#include <stdlib.h>
#include <string.h>

#include <cub/cub.cuh>

#include "qm_common.cuh"
#include "qm_tma.cuh"

namespace qm {
namespace {

constexpr int kG = 8;                         // block columns per group
constexpr int kBlk = 16;                      // block size
constexpr int kBlkBytes = kBlk * kBlk * 8;    // 2 KB
constexpr int kCW = 4;                        // consumer warps: warp w owns columns w, w+4 (gcol)
constexpr uint32_t kAbsent = 0xffffffffu;

// Columns of consumer warp w: w and w + 4. At the ends of a group's k range only a contiguous run
// of its columns has a B block; interleaving spreads that run over the warps (= the SM's four
// sub-partitions), so the busiest warp of a partial stage has half the work it would have with
// adjacent columns 2w, 2w+1 (-DQM_EXP_G16_PAIRED; +3 % with the specialised partial stages below,
// -4 % before them, when every partial stage took a guarded slow path). Mirroring the ownership in
// the second row (columns 3 - w, 7 - w: a run of present columns then loads the warps from both ends)
// needs separate B fragments per row -- 12 instead of 8 fragment loads per k step -- and measured
// 2.5 % slower.
#ifdef QM_EXP_G16_PAIRED
__device__ __forceinline__ int gcol(int warp, int q) { return 2 * warp + q; }
__device__ __forceinline__ uint32_t gcols_present(uint32_t pm, int warp) { return (pm >> (2 * warp)) & 3u; }
#else
__device__ __forceinline__ int gcol(int warp, int q) { return warp + 4 * q; }
__device__ __forceinline__ uint32_t gcols_present(uint32_t pm, int warp) {
  return ((pm >> warp) & 1u) | (((pm >> (warp + 4)) & 1u) << 1);
}
#endif

// R = block rows per group (1, or 2 when a leaf row pair is contiguous in key order: <= 8 blocks per
// leaf side). A group is R x 8 member slots, slot = r * 8 + c, in key order.
template <int R>
struct GCfg {
  static constexpr int M = R * kG;                       // member slots
  static constexpr int EW = R + kG;                      // words per entry: a[R], b[8]
#ifndef QM_G16_STAGES2
#define QM_G16_STAGES2 3
#endif
#ifndef QM_G16_MINB2
#define QM_G16_MINB2 3
#endif
  static constexpr int STAGES = R == 1 ? 3 : QM_G16_STAGES2;
  static constexpr int STAGE_BYTES = (R + kG) * kBlkBytes;
  static constexpr int THREADS = 32 * (kCW + 1);
  static constexpr int MINB = R == 1 ? 4 : QM_G16_MINB2;
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + 4 * STAGES * 8 + 64;
};

// Group of a C block: its key without the member bits (same leaf; same block row, or the same
// aligned pair of block rows for R = 2; aligned runs of up to 8 block columns).
template <int R>
__device__ __forceinline__ uint64_t group_code(uint64_t key, int lbits, int mbits) {
  return R == 2 ? key >> (lbits + 1) : key >> mbits;
}
template <int R>
__device__ __forceinline__ int member_slot(uint64_t key, int lbits, int mbits) {
  if (R == 2) return (int)((((key >> lbits) & 1ull) << 3) | (key & ((1ull << lbits) - 1ull)));
  return (int)(key & ((1ull << mbits) - 1ull));
}

template <int R>
__global__ void k_group_heads(const uint64_t *c_keys, int64_t nC, int lbits, int mbits, int64_t *head) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= nC; c += (int64_t)gridDim.x * blockDim.x)
    head[c] = (c < nC && (c == 0 || group_code<R>(c_keys[c], lbits, mbits) !=
                                        group_code<R>(c_keys[c - 1], lbits, mbits))) ? 1 : 0;
}

// First C block of every group (a scatter of the heads through their exclusive scan) and the
// group count.
__global__ void k_group_first(const int64_t *head, const int64_t *gidx, int64_t nC, int64_t *gfirst,
                              int64_t *n_groups) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= nC; c += (int64_t)gridDim.x * blockDim.x) {
    if (c < nC && head[c]) gfirst[gidx[c]] = c;
    if (c == nC) *n_groups = gidx[nC];
  }
}

// One warp per group (grid-stride over the groups, so every warp of the launch has work): lane s owns the member in slot s (if any) and walks
// its k-ascending triple list; each step takes the smallest head k over the lanes (warp min), and
// the lanes holding it supply the entry's A index of their row and B index of their column (a
// triple (r,k,c) exists iff A(r,k) and B(k,c) do, so one entry per k describes every member's
// product at that k). The group's entries go to its own triple range [c_tptr[first], ...): the
// union of the members' k is never longer than their triple lists together, so no count pass.
template <int R>
__global__ void k_group_merge(const uint64_t *c_keys, const int64_t *c_tptr, const uint2 *tri, const uint64_t *a_keys,
                              int64_t nC, int nbl, int lbits, int mbits, const int64_t *gfirst,
                              const int64_t *n_groups, int64_t *ucount, uint32_t *gmask, uint32_t *entries) {
  constexpr int M = GCfg<R>::M, EW = GCfg<R>::EW;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  // writer lanes: [0, R) the A index of row `lane`, [R, R+8) the B index of column lane-R
  const int wr = lane < R ? lane : 0;
  const int wc = (lane >= R && lane < EW) ? lane - R : 0;
  const uint32_t rowsel = 0xffu << (8 * wr);
  const uint32_t colsel = R == 2 ? (0x101u << wc) : (1u << wc);
  const int64_t nG = *n_groups;
  for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < nG; g += warps) {
    const int64_t c0 = gfirst[g];
    const int nm = (int)((g + 1 < nG ? gfirst[g + 1] : nC) - c0);
    int64_t pos = 0, end = 0;
    uint32_t mask = 0;
    for (int m = 0; m < nm; ++m) {
      const int sl = member_slot<R>(c_keys[c0 + m], lbits, mbits);
      mask |= 1u << sl;
      if (lane == sl) {
        pos = c_tptr[c0 + m];
        end = c_tptr[c0 + m + 1];
      }
    }
    uint32_t *out = entries + (size_t)c_tptr[c0] * EW;
    int64_t cnt = 0;
    // The lane's next kD triples and their k (block column of the A block), prefetched kD deep so
    // the dependent tri -> a_keys loads of a lane overlap the merge steps in between.
    constexpr int kD = 4;
    uint2 t[kD];
    uint32_t kq[kD];
#pragma unroll
    for (int d = 0; d < kD; ++d) {
      kq[d] = 0xffffffffu;
      t[d] = make_uint2(0u, 0u);
      if (lane < M && pos + d < end) {
        uint32_t bi;
        t[d] = tri[pos + d];
        qkey_decode(a_keys[t[d].x], nbl, lbits, &bi, &kq[d]);
      }
    }
    while (true) {
      const uint32_t kmin = __reduce_min_sync(0xffffffffu, kq[0]);
      if (kmin == 0xffffffffu) break;
      const bool hit = kq[0] == kmin;
      const uint32_t hits = __ballot_sync(0xffffffffu, hit);
      const uint32_t sa = hits & rowsel, sb = hits & colsel;
      const uint32_t a = __shfl_sync(0xffffffffu, t[0].x, sa ? __ffs(sa) - 1 : 0);
      const uint32_t b = __shfl_sync(0xffffffffu, t[0].y, sb ? __ffs(sb) - 1 : 0);
      if (lane < R) out[cnt * EW + lane] = sa ? a : kAbsent;
      else if (lane < EW) out[cnt * EW + lane] = sb ? b : kAbsent;
      if (hit) {
#pragma unroll
        for (int d = 0; d + 1 < kD; ++d) {
          t[d] = t[d + 1];
          kq[d] = kq[d + 1];
        }
        kq[kD - 1] = 0xffffffffu;
        if (++pos + kD - 1 < end) {
          uint32_t bi;
          t[kD - 1] = tri[pos + kD - 1];
          qkey_decode(a_keys[t[kD - 1].x], nbl, lbits, &bi, &kq[kD - 1]);
        }
      }
      ++cnt;
    }
    if (lane == 0) {
      ucount[g] = cnt;
      gmask[g] = mask;
    }
  }
}

// One stage of a consumer warp: the products of its two columns with every present A row.
// ONA / ONB = the present A rows / B columns of the warp as compile-time masks: each of the (at most
// nine) combinations is its own straight-line code without per-product guards, so the loads of the
// next k step can be scheduled under the DMMAs of this one for partial stages too (the ends of a
// group's k range, where only some of its columns have a B block). Returns the OR of the stage's
// last fragments (the stage-release dependency, see k_numeric_tma).
template <int R, uint32_t ONA, uint32_t ONB>
__device__ __forceinline__ uint64_t group_stage(const uint8_t *sa, int warp, const uint32_t (&aoff)[4],
                                                const uint32_t (&boff)[4][2], double (&acc)[R][2][2][2][2]) {
  uint64_t dep = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double af[R][2], bf[2][2];
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (ONA & (1u << r))
#pragma unroll
        for (int i = 0; i < 2; ++i) af[r][i] = *(const double *)(sa + r * kBlkBytes + i * 8 * 128 + aoff[j]);
#pragma unroll
    for (int q = 0; q < 2; ++q)
      if (ONB & (1u << q)) {
        const uint8_t *sb = sa + (R + gcol(warp, q)) * kBlkBytes;
#pragma unroll
        for (int n = 0; n < 2; ++n) bf[q][n] = *(const double *)(sb + boff[j][n]);
      }
    if (j == 3) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (ONA & (1u << r))
#pragma unroll
          for (int i = 0; i < 2; ++i) dep |= (uint64_t)__double_as_longlong(af[r][i]);
#pragma unroll
      for (int q = 0; q < 2; ++q)
        if (ONB & (1u << q))
#pragma unroll
          for (int n = 0; n < 2; ++n) dep |= (uint64_t)__double_as_longlong(bf[q][n]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int q = 0; q < 2; ++q)
        if ((ONA & (1u << r)) && (ONB & (1u << q)))
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int n = 0; n < 2; ++n) dmma(acc[r][q][i][n][0], acc[r][q][i][n][1], af[r][i], bf[q][n]);
  }
  return dep;
}

// Dispatch on the warp's present columns for a compile-time set of A rows.
template <int R, uint32_t ONA>
__device__ __forceinline__ uint64_t group_stage_b(const uint8_t *sa, int warp, uint32_t onb, const uint32_t (&aoff)[4],
                                                  const uint32_t (&boff)[4][2], double (&acc)[R][2][2][2][2]) {
  if (onb == 3u) return group_stage<R, ONA, 3u>(sa, warp, aoff, boff, acc);
  if (onb == 1u) return group_stage<R, ONA, 1u>(sa, warp, aoff, boff, acc);
  return group_stage<R, ONA, 2u>(sa, warp, aoff, boff, acc);
}

// The members' triple lists of a group as the inline-merge producer reads them (INLINE = true: the
// producer warp merges the lists itself, one entry per stage, instead of reading k_group_merge's
// entries).
struct GroupSrc {
  const uint64_t *c_keys, *a_keys;
  const uint2 *tri;
  int64_t nC;
  int nbl, lbits, mbits;
};

template <int R, bool INLINE>
__global__ void __launch_bounds__(GCfg<R>::THREADS, GCfg<R>::MINB)
    k_numeric_group16(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                      const uint32_t *__restrict__ entries, const int64_t *__restrict__ c_tptr,
                      const int64_t *__restrict__ ucount,
                      const int64_t *__restrict__ gfirst, const uint32_t *__restrict__ gmask,
                      const int64_t *__restrict__ n_groups_dev, double *__restrict__ C, double *__restrict__ csq,
                      uint8_t *__restrict__ cnz, int64_t *__restrict__ zero_count,
                      unsigned long long *__restrict__ counter, uint64_t zmask, const GroupSrc src) {
  using Cfg = GCfg<R>;
  constexpr int STAGES = Cfg::STAGES, EW = Cfg::EW;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *full = (uint64_t *)(smem + (size_t)STAGES * Cfg::STAGE_BYTES);
  uint64_t *empty = full + STAGES;
  volatile int64_t *meta = (volatile int64_t *)(empty + STAGES);       // unit*2 + last, -1 = end
  volatile uint32_t *pmask = (volatile uint32_t *)(meta + STAGES);     // bits 0-7 B columns, 8.. A rows
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nG = INLINE ? 0 : *n_groups_dev;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == kCW) {
    // ---------------- producer warp: one stage per entry; lane c < 8 loads column c's B block,
    // lane 8 + r row r's A block, so the up to 8 + R TMA loads of a stage issue together. The entry
    // of the next stage (and the next claimed group) is loaded one stage ahead.
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&map_a) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&map_b) : "memory");
    }
    const bool loader = lane < kG + R;
    if constexpr (INLINE) {
      // ---- inline merge: lane s < M owns the member in slot s and walks its k-ascending triple
      // list (its next kD triples and their k prefetched); every stage takes the smallest head k
      // over the lanes, and the lanes holding it supply the A index of their row and the B index
      // of their column to the loader lanes -- k_group_merge's step, done here once per stage, so
      // there is no merge pass, no entries array and no per-group metadata read by the consumers
      // (the stage word carries the group's first C block, member mask, present blocks and the
      // last-stage flag).
      // Work is claimed in chunks of 16 consecutive C blocks: the groups that START in a chunk are
      // its claimer's (a group has at most 16 members, so every chunk holds a start), found by
      // comparing neighbouring keys' group codes -- no pre-pass over the C keys at all. The next
      // group (and, when the chunk is used up, the next chunk) is taken when at most kAhead entries
      // of some member remain: just in time for L2 locality, early enough to hide its header loads.
      constexpr int M = Cfg::M, kD = 4, kAhead = 6;
      constexpr uint32_t kNone = 0xffffffffu;
      const int slot = lane < kG ? R + lane : lane - kG;
      const uint32_t sel = lane < kG ? (R == 2 ? (0x101u << lane) : (1u << lane))       // B column `lane`
                                     : (loader ? (0xffu << (8 * (lane - kG))) : 0u);     // A row lane - 8
      const int64_t nQ = (src.nC + 15) >> 4;
      int64_t pos = 0, end = 0, npos = 0, nend = 0;
      int64_t chunk = blockIdx.x, first = -1, nfirst = -1;
      uint32_t heads = 0, mask = 0, nmask = 0;
      bool claimed = false;
      uint2 t[kD];
      uint32_t kq[kD];
      auto chunk_heads = [&](int64_t q) -> uint32_t {
        const int64_t c = (q << 4) + lane;
        bool head = false;
        if (lane < 16 && c < src.nC)
          head = c == 0 || group_code<R>(src.c_keys[c], src.lbits, src.mbits) !=
                               group_code<R>(src.c_keys[c - 1], src.lbits, src.mbits);
        return __ballot_sync(0xffffffffu, head);
      };
      // First C block of the next group of this CTA (-1: no work left); claims chunks as needed.
      auto next_group = [&]() -> int64_t {
        while (heads == 0u) {
          unsigned long long got = 0;
          if (lane == 0) got = atomicAdd(counter, 1ull);
          chunk = (int64_t)gridDim.x + (int64_t)__shfl_sync(0xffffffffu, got, 0);
          if (chunk >= nQ) return -1;
          heads = chunk_heads(chunk);
        }
        const int h = __ffs(heads) - 1;
        heads &= heads - 1u;
        return (chunk << 4) + h;
      };
      // Members of the group starting at C block c0 (the run of keys with its group code), their
      // slots and this lane's triple range.
      auto header = [&](int64_t c0, int64_t &p, int64_t &e, uint32_t &mk) {
        p = e = 0;
        mk = 0;
        if (c0 < 0) return;
        const bool in = lane < 16 && c0 + lane < src.nC;
        const uint64_t key = in ? src.c_keys[c0 + lane] : 0ull;
        const uint64_t code = group_code<R>(key, src.lbits, src.mbits);
        const uint64_t code0 = __shfl_sync(0xffffffffu, code, 0);
        const uint32_t eq = __ballot_sync(0xffffffffu, in && code == code0);
        const int nm = __ffs(~eq) - 1;  // length of the run of equal codes from lane 0
        mk = __reduce_or_sync(0xffffffffu, lane < nm ? 1u << member_slot<R>(key, src.lbits, src.mbits) : 0u);
        if (lane < M && ((mk >> lane) & 1u)) {  // members are in key order = slot order
          const int m = __popc(mk & ((1u << lane) - 1u));
          p = c_tptr[c0 + m];
          e = c_tptr[c0 + m + 1];
        }
      };
      auto fetch = [&](int d, int64_t at) {
        kq[d] = kNone;
        t[d] = make_uint2(0u, 0u);
        if (at < end) {
          uint32_t bi;
          t[d] = src.tri[at];
          qkey_decode(src.a_keys[t[d].x], src.nbl, src.lbits, &bi, &kq[d]);
        }
      };
      if (chunk < nQ) {
        heads = chunk_heads(chunk);
        first = next_group();
      }
      header(first, pos, end, mask);
#pragma unroll
      for (int d = 0; d < kD; ++d) fetch(d, pos + d);
      uint32_t kmin = __reduce_min_sync(0xffffffffu, kq[0]);
      int s = 0;
      uint32_t phase = 0;
      while (true) {
        if (first < 0) {
          if (lane == 0) {
            mbar_wait(&empty[s], phase ^ 1u);
            meta[s] = -1;
            mbar_arrive(&full[s]);
          }
          break;
        }
        if (!claimed) {
          const uint32_t rem = __reduce_max_sync(0xffffffffu, (uint32_t)(end - pos));
          if (rem <= (uint32_t)kAhead) {
            nfirst = next_group();
            header(nfirst, npos, nend, nmask);
            claimed = true;
          }
        }
        const bool hit = kq[0] == kmin;
        const uint32_t hits = __ballot_sync(0xffffffffu, hit);
        const uint32_t mine = hits & sel;
        const int from = mine ? __ffs(mine) - 1 : 0;
        const uint32_t av = __shfl_sync(0xffffffffu, t[0].x, from), bv = __shfl_sync(0xffffffffu, t[0].y, from);
        const uint32_t cur = mine ? (lane < kG ? bv : av) : kAbsent;
        if (hit) {
#pragma unroll
          for (int d = 0; d + 1 < kD; ++d) {
            t[d] = t[d + 1];
            kq[d] = kq[d + 1];
          }
          ++pos;
          fetch(kD - 1, pos + kD - 1);
        }
        const uint32_t knext = __reduce_min_sync(0xffffffffu, kq[0]);
        const bool last = knext == kNone;
        if (lane == 0) mbar_wait(&empty[s], phase ^ 1u);
        __syncwarp();
        const uint32_t pm = __ballot_sync(0xffffffffu, cur != kAbsent);
        uint8_t *st = smem + (size_t)s * Cfg::STAGE_BYTES;
        if (lane == 0) {
          meta[s] = (first << 32) | (int64_t)(mask << 16) | (int64_t)(pm << 1) | (last ? 1 : 0);
          mbar_expect_tx(&full[s], (uint32_t)__popc(pm) * kBlkBytes);
        }
        __syncwarp();
        if (cur != kAbsent)
          tma_load_2d(st + slot * kBlkBytes, lane < kG ? &map_b : &map_a, 0, (int)(cur * kBlk), &full[s]);
        if (++s == STAGES) {
          s = 0;
          phase ^= 1u;
        }
        kmin = knext;
        if (last) {  // next group (taken above: a finished group has no entries left)
          if (!claimed) {
            nfirst = next_group();
            header(nfirst, npos, nend, nmask);
          }
          first = nfirst;
          pos = npos;
          end = nend;
          mask = nmask;
          claimed = false;
#pragma unroll
          for (int d = 0; d < kD; ++d) fetch(d, pos + d);
          kmin = __reduce_min_sync(0xffffffffu, kq[0]);
        }
      }
      return;
    }
    const int word = lane < kG ? R + lane : lane - kG;  // Entry layout: a[R], b[8]
    // smem slot of this lane's block: A rows first, then the 8 B columns
    const int slot = lane < kG ? R + lane : lane - kG;
    int64_t unit = blockIdx.x, e = 0, e1 = 0;
    uint32_t cur = kAbsent;
    if (unit < nG) {
      e = c_tptr[gfirst[unit]];
      e1 = e + ucount[unit];
      if (loader) cur = entries[e * EW + word];
    }
    int s = 0;
    uint32_t phase = 0;
    while (true) {
      int64_t nunit = unit, ne = e + 1, ne1 = e1;
      uint32_t nxt = kAbsent;
      if (unit < nG) {
        if (ne == e1) {  // next group, claimed just in time
          unsigned long long got = 0;
          if (lane == 0) got = atomicAdd(counter, 1ull);
          nunit = (int64_t)gridDim.x + (int64_t)__shfl_sync(0xffffffffu, got, 0);
          if (nunit < nG) {
            ne = c_tptr[gfirst[nunit]];
            ne1 = ne + ucount[nunit];
          }
        }
        if (nunit < nG && loader) nxt = entries[ne * EW + word];
      }
      if (lane == 0) mbar_wait(&empty[s], phase ^ 1u);
      __syncwarp();
      if (unit >= nG) {
        if (lane == 0) {
          meta[s] = -1;
          mbar_arrive(&full[s]);
        }
        break;
      }
      const uint32_t pm = __ballot_sync(0xffffffffu, loader && cur != kAbsent);
      uint8_t *st = smem + (size_t)s * Cfg::STAGE_BYTES;
      if (lane == 0) {
        meta[s] = unit * 2 + (e + 1 == e1 ? 1 : 0);
        pmask[s] = pm;
        mbar_expect_tx(&full[s], (uint32_t)__popc(pm) * kBlkBytes);
      }
      __syncwarp();
      if (loader && cur != kAbsent)
        tma_load_2d(st + slot * kBlkBytes, lane < kG ? &map_b : &map_a, 0, (int)(cur * kBlk), &full[s]);
      unit = nunit;
      e = ne;
      e1 = ne1;
      cur = nxt;
      if (++s == STAGES) {
        s = 0;
        phase ^= 1u;
      }
    }
    return;
  }

  // -------- consumers: warp w = columns w, w+4 (gcol) of every group row (R*16 x 32: each A fragment
  // serves both columns, each B fragment every row) --------
  const int g = lane >> 2, tq = lane & 3;
  uint32_t aoff[4], boff[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int kk = kperm(tq, j);
    aoff[j] = g * 128 + (((kk >> 1) ^ g) << 4) + (kk & 1) * 8;
#pragma unroll
    for (int h = 0; h < 2; ++h) boff[j][h] = kk * 128 + ((((h * 4) + (g >> 1)) ^ (kk & 7)) << 4) + (g & 1) * 8;
  }
  double acc[R][2][2][2][2];  // [row][column of the pair][i][n][2]
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int n = 0; n < 2; ++n) acc[r][q][i][n][0] = acc[r][q][i][n][1] = 0.0;
  int s = 0;
  uint32_t phase = 0;
  int32_t cur_unit = -1, c_first = 0;  // (32-bit: fewer live registers across the stage loop)
  uint32_t gm = 0;
  while (true) {
    mbar_wait(&full[s], phase);  // (testing the next stage's barrier early, under this stage's DMMAs: -0.7 %)
    const int64_t mt = meta[s];
    if (mt < 0) break;
    uint32_t pm;
    if constexpr (INLINE) {  // stage word: first C block << 32 | member mask << 16 | present << 1 | last
      c_first = (int32_t)(mt >> 32);
      gm = ((uint32_t)mt >> 16) & 0xffffu;
      pm = ((uint32_t)mt >> 1) & 0x7fffu;
    } else {
      const int32_t mt_unit = (int32_t)(mt >> 1);
      if (mt_unit != cur_unit) {  // a group's first stage: fetch its epilogue metadata now,
        cur_unit = mt_unit;       // so the loads complete under the group's DMMAs
        gm = gmask[cur_unit];
        c_first = (int32_t)gfirst[cur_unit];
      }
      pm = pmask[s];
    }
    const uint32_t onb = gcols_present(pm, warp);
    const uint32_t ona = (pm >> kG) & ((1u << R) - 1u);
    uint64_t dep = 0;
    const uint8_t *stg = smem + (size_t)s * Cfg::STAGE_BYTES;
    if (onb && ona) {
      if (ona == (1u << R) - 1u) {
        dep = group_stage_b<R, (1u << R) - 1u>(stg, warp, onb, aoff, boff, acc);
#ifdef QM_EXP_G16_REPEAT  // experiment (wrong results): twice the DMMAs per stage, same stage overhead
        dep |= group_stage_b<R, (1u << R) - 1u>(stg, warp, onb, aoff, boff, acc);
#endif
      } else if (R == 2) {
        dep = ona == 1u ? group_stage_b<R, 1u>(stg, warp, onb, aoff, boff, acc)
                        : group_stage_b<R, (R == 2 ? 2u : 1u)>(stg, warp, onb, aoff, boff, acc);
      }
    }
    // release once this warp's fragments are in registers (see k_numeric_tma)
    dep &= zmask;
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s] + (uint32_t)dep);
    if (++s == STAGES) {
      s = 0;
      phase ^= 1u;
    }
    if (mt & 1) {
      // (No branch on "does this member exist" around the accumulator reads: ptxas renames the
      // accumulators around such a branch -- DMMAs with D != C and ~50 register moves per stage.
      // An absent member's accumulators are zero; the same code runs with its stores and result
      // writes predicated off.)
      const uint64_t c_policy = l2_evict_first_policy();  // (created here: one register less in the loop)
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int mb = r * kG + gcol(warp, q);
          const bool member = ((gm >> mb) & 1u) != 0u;
          const int64_t c = (int64_t)c_first + __popc(gm & ((1u << mb) - 1u));
          double *cb = C + (size_t)c * (kBlk * kBlk);
          double ss0 = 0.0, ss1 = 0.0;
          bool nz = false;
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int n = 0; n < 2; ++n) {
              const double v0 = acc[r][q][i][n][0], v1 = acc[r][q][i][n][1];
              if (member) st_evict_first(cb + (size_t)(i * 8 + g) * kBlk + n * 8 + 2 * tq, v0, v1, c_policy);
              ss0 = fma(v0, v0, ss0);
              ss1 = fma(v1, v1, ss1);
              nz |= (v0 != 0.0) | (v1 != 0.0);
              acc[r][q][i][n][0] = acc[r][q][i][n][1] = 0.0;
            }
          double ss = ss0 + ss1;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
          const bool wnz = __any_sync(0xffffffffu, nz);
          if (member && lane == 0) {
            csq[c] = ss;
            cnz[c] = (uint8_t)wnz;
            if (!wnz && zero_count) atomicAdd((unsigned long long *)zero_count, 1ull);
          }
        }
    }
  }
}

inline int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (int)g;
}

size_t scan_bytes(int64_t n) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t *)nullptr, (int64_t *)nullptr, n);
  return b;
}

struct GroupWs {
  int64_t *head, *gidx, *ucount, *gfirst, *n_groups;
  uint32_t *gmask;
  unsigned long long *counter;
  uint32_t *entries;
  void *cub;
  size_t cub_bytes;
};

// Entries are sized for the widest layout (R = 2: 10 words), one per triple at most.
// QM_G16_MERGE=kernel: the separate merge pass (k_group_merge + entries array) instead of the
// producer's inline merge (A/B measurements).
bool inline_merge() {
  const char *e = getenv("QM_G16_MERGE");
  return !(e && strcmp(e, "kernel") == 0);
}

GroupWs carve_group(Carver &cv, int64_t nC, int64_t nT) {
  GroupWs w;
  w.head = cv.take<int64_t>(nC + 1);
  w.gidx = cv.take<int64_t>(nC + 1);
  w.ucount = cv.take<int64_t>(nC + 1);
  w.gfirst = cv.take<int64_t>(nC + 1);
  w.n_groups = cv.take<int64_t>(1);
  w.gmask = cv.take<uint32_t>(nC + 1);
  w.counter = cv.take<unsigned long long>(1);
  w.entries = cv.take<uint32_t>(inline_merge() ? 1 : std::max<int64_t>(nT, 1) * GCfg<2>::EW);  // <= one entry per triple
  w.cub_bytes = scan_bytes(nC + 1);
  w.cub = cv.take<char>(w.cub_bytes);
  return w;
}

// Rows per group: 2 when a leaf has <= 8 blocks per side (a leaf row pair is then contiguous in
// key order), else 1. QM_GROUP_ROWS=1 forces single-row groups (A/B measurements).
int group_rows(const Geometry &g) {
  const char *e = getenv("QM_GROUP_ROWS");
  if (e && strcmp(e, "1") == 0) return 1;
  return g.lbits <= 3 ? 2 : 1;
}

template <int R, bool INLINE>
int launch_group(const Geometry &g, const double *A, int64_t nA, const double *B, int64_t nB,
                 const uint64_t *a_keys, const uint2 *t2, const int64_t *c_tptr, const uint64_t *c_keys,
                 int64_t nC, int64_t nT, double *C, double *csq, uint8_t *cnz, int64_t *zc, const GroupWs &w,
                 cudaStream_t st) {
  using Cfg = GCfg<R>;
  const int mbits = std::min(g.lbits, 3);
  if (!INLINE) {
    k_group_heads<R><<<grid_for(nC + 1), 256, 0, st>>>(c_keys, nC, g.lbits, mbits, w.head);
    QM_LAUNCHED("k_group_heads");
    size_t tb = w.cub_bytes;
    QM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(w.cub, tb, w.head, w.gidx, nC + 1, st));
    k_group_first<<<grid_for(nC + 1), 256, 0, st>>>(w.head, w.gidx, nC, w.gfirst, w.n_groups);
    QM_LAUNCHED("k_group_first");
  }
  if (!INLINE) {
    const int merge_grid = (int)std::min<int64_t>((nC + 7) / 8, (int64_t)device_sm_count() * 8);
    k_group_merge<R><<<merge_grid, 256, 0, st>>>(c_keys, c_tptr, t2, a_keys, nC, g.nbl, g.lbits, mbits, w.gfirst,
                                                 w.n_groups, w.ucount, w.gmask, w.entries);
    QM_LAUNCHED("k_group_merge");
  }
  CUtensorMap ma, mb;
  int rc = make_map(&ma, A, nA, kBlk, kBlk);
  if (rc != QM_OK) return rc;
  rc = make_map(&mb, B, nB, kBlk, kBlk);
  if (rc != QM_OK) return rc;
  static PerDeviceOnce once;
  rc = once.run([]() -> int {
    QM_CUDA_TRY(cudaFuncSetAttribute(k_numeric_group16<R, INLINE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)Cfg::SMEM));
    return (int)QM_OK;
  });
  if (rc != QM_OK) return rc;
  QM_CUDA_TRY(cudaMemsetAsync(w.counter, 0, sizeof(unsigned long long), st));
  int per_sm = 0;
  static PerDeviceInt occupancy;  // cudaOccupancy* costs microseconds of host time per call
  rc = occupancy.get(&per_sm, [](int *x) -> int {
    QM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(x, k_numeric_group16<R, INLINE>, Cfg::THREADS, Cfg::SMEM));
    return (int)QM_OK;
  });
  if (rc != QM_OK) return rc;
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)device_sm_count() * per_sm;
  const int64_t units = INLINE ? (nC + 15) / 16 : nC;  // chunks of 16 C blocks; groups <= C blocks
  if (grid > units) grid = units;
  const GroupSrc src{c_keys, a_keys, t2, nC, g.nbl, g.lbits, mbits};
  k_numeric_group16<R, INLINE><<<(int)grid, Cfg::THREADS, Cfg::SMEM, st>>>(
      ma, mb, w.entries, c_tptr, w.ucount, w.gfirst, w.gmask, w.n_groups, C, csq, cnz, zc, w.counter,
      /*zmask=*/0ull, src);
  QM_LAUNCHED("k_numeric_group16");
  return QM_OK;
}

}  // namespace

size_t numeric_group16_ws_bytes(int64_t nC, int64_t nT) {
  Carver cv(nullptr, 0);
  carve_group(cv, nC, nT);
  return cv.off;
}

// Whether a bs 16 product runs as groups of C blocks. Groups pay when a stage's k is shared by
// several members: k lists of some length (banded, decay). With about one triple per C block
// (random patterns) nearly every stage serves a single member -- 1 of up to 16 products -- and the
// per-block cp.async kernel is 2-3x faster (measured: random, 8 / 32 blocks per row: 8.4 / 10.4
// against 2.8 / 5.7 TFLOP/s). The average k-list length decides; QM_G16_GROUPS=1 / 0 forces groups /
// the per-block kernel.
bool group16_selected(const Geometry &g, int64_t nC, int64_t nT) {
  if (g.bs != kBlk || g.nbl < 2 || nC >= ((int64_t)1 << 31)) return false;
  const char *e = getenv("QM_G16_GROUPS");
  if (e && e[0] == '0') return false;
  return (e && e[0] == '1') || nT >= 4 * nC;
}

// bs 16 with at least two blocks per leaf side; QM_ERR_UNSUPPORTED otherwise (caller falls back).
int launch_numeric_group16(const Geometry &g, const double *A, int64_t nA, const double *B, int64_t nB,
                           const uint64_t *a_keys, const uint32_t *tri, const int64_t *c_tptr,
                           const uint64_t *c_keys, int64_t nC, int64_t nT, double *C, double *csq,
                           uint8_t *cnz, int64_t *zc, void *ws, size_t ws_bytes, cudaStream_t st) {
  if (!a_keys || !c_keys || !group16_selected(g, nC, nT)) return QM_ERR_UNSUPPORTED;
  Carver cv(ws, ws_bytes);
  GroupWs w = carve_group(cv, nC, nT);
  if (!cv.ok() || !ws) {
    set_error("qm_numeric: workspace %zu < required %zu (bs 16 groups)", ws_bytes, cv.off);
    return QM_ERR_WORKSPACE;
  }
  if (nA * (int64_t)kBlk >= ((int64_t)1 << 31) || nB * (int64_t)kBlk >= ((int64_t)1 << 31)) {
    set_error("qm_numeric: pool exceeds TMA's int32 row coordinate");
    return QM_ERR_UNSUPPORTED;
  }
  const uint2 *t2 = (const uint2 *)tri;
  const bool il = inline_merge();
  if (group_rows(g) == 2)
    return il ? launch_group<2, true>(g, A, nA, B, nB, a_keys, t2, c_tptr, c_keys, nC, nT, C, csq, cnz, zc, w, st)
              : launch_group<2, false>(g, A, nA, B, nB, a_keys, t2, c_tptr, c_keys, nC, nT, C, csq, cnz, zc, w, st);
  return il ? launch_group<1, true>(g, A, nA, B, nB, a_keys, t2, c_tptr, c_keys, nC, nT, C, csq, cnz, zc, w, st)
            : launch_group<1, false>(g, A, nA, B, nB, a_keys, t2, c_tptr, c_keys, nC, nT, C, csq, cnz, zc, w, st);
}

}  // namespace qm

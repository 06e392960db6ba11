// Numeric phase for 32x32 blocks: quads of C blocks.
//
// With one 32x32 C block per work unit (k_numeric_tma's bs-32 configuration) a pipeline stage is one
// triple: 16 KB of operands for 64 KFLOP, four warps of 16x16, 32 DMMAs per warp and stage hand-off.
// Here a work unit is a *quad*: the up to four C blocks (2r..2r+1, 2c..2c+1) -- consecutive in
// quadtree-key order when a leaf is one block (the key is the Morton code of the block coordinates)
// or 2x2 blocks (the leaf-local part of the key is row-major). A triple (r,k,c) reads A(r,k) and
// B(k,c), so one stage per k carries the quad's A(2r,k), A(2r+1,k), B(k,2c), B(k,2c+1) -- 32 KB
// for up to four products (half the operand bytes per flop) -- laid out exactly like a 64x64 tile's
// stage of k_numeric_tma (A: two 16-double k sub-panels of 64 rows, B: four 16-column sub-panels of
// 32 k rows), so the four consumer warps run the bs-64 kernel's 32x32 warp tile: 16 DMMAs per 8
// fragment loads and k step, 128 DMMAs per stage. Warp w IS member slot w (block row w >> 1, block
// column w & 1 of the quad); it executes a stage iff its own member has a triple at that k (the
// stage word carries the hit mask -- a pruned plan, approximate.py, can drop single members'
// triples), so every C block sums exactly its own triples in ascending k with the same per-triple
// DMMA order as the per-block kernel: the blocks are bitwise identical, and the squared norms are
// accumulated per 16x16 sub-tile in the per-block kernel's order and combined in its order too.
//
// The producer warp merges the members' k-ascending triple lists itself, one entry per stage
// (lane s < 4 owns member slot s), and claims chunks of 4 consecutive C blocks whose quads it finds
// from neighbouring keys -- as in k_numeric_group16 (qm_numeric_group.cu), no pre-pass.
// Replaces BlockSparseLeaf.multiply + add (block_sparse.py:112-152) and _set_block's exact-zero
// test (block_sparse.py:37-41) for bs 32, like the kernels it stands in for.
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "qm_common.cuh"
#include "qm_tma.cuh"

namespace qm {
namespace {

constexpr int kQB = 32;                       // block size
constexpr int kQBlkElems = kQB * kQB;
constexpr int kQKP = 32;                      // k depth of a stage = one block
constexpr int kQASP = 64 * 128;               // A sub-panel: 64 rows x 16 doubles
constexpr int kQBSP = kQKP * 128;             // B sub-panel: 32 k rows x 16 doubles
constexpr int kQABytes = 2 * kQASP;           // two k sub-panels
constexpr int kQBBytes = 4 * kQBSP;           // four column sub-panels
constexpr int kQStage = kQABytes + kQBBytes;  // 32 KB
constexpr int kQLoad = 32 * 128;              // one TMA box: 32 rows x 16 doubles
constexpr int kQCW = 4;                       // consumer warps = member slots
constexpr uint32_t kQNone = 0xffffffffu;

template <int STAGES_, int MINB_>
struct QCfg {
  static constexpr int STAGES = STAGES_, MINB = MINB_;
  static constexpr int THREADS = 32 * (kQCW + 1);
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * kQStage + 3 * STAGES * 8 + 64;
};

struct QuadSrc {
  const uint64_t *c_keys, *a_keys;
  const uint2 *tri;
  const int64_t *c_tptr;
  int64_t nC;
  int nbl, lbits;
};

// The producer warp (its own function, so that its walk state does not take registers from the
// math warps' loop).
template <class Cfg>
__device__ __noinline__ void quad_producer(const CUtensorMap *map_a, const CUtensorMap *map_b, const QuadSrc &src,
                                           uint8_t *smem, uint64_t *full, uint64_t *empty, volatile int64_t *meta,
                                           unsigned long long *counter) {
  constexpr int STAGES = Cfg::STAGES;
  const int lane = threadIdx.x & 31;
    // ---------------- producer warp ----------------
    // Loader lanes: 0..3 = A block of quad row (lane >> 1), k sub-panel (lane & 1);
    // 4..7 = B block of quad column ((lane - 4) >> 1), column half ((lane - 4) & 1).
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(map_a) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(map_b) : "memory");
    }
    constexpr int kD = 4, kAhead = 4, kChunk = 4;  // (a chunk of 4 C blocks holds at least one quad start)
    const bool is_a = lane < 4, loader = lane < 8;
    const int part = is_a ? lane >> 1 : (lane - 4) >> 1;  // quad row / column served
    const int sub = lane & 1;                             // k sub-panel (A) / column half (B)
    // member slots (row << 1 | column) that read this lane's block
    const uint32_t sel = !loader ? 0u : is_a ? (0x3u << (2 * part)) : (0x5u << part);
    const uint32_t dst_off = is_a ? (uint32_t)(sub * kQASP + part * kQLoad)
                                  : (uint32_t)(kQABytes + (part * 2 + sub) * kQBSP);
    const int64_t nQ = (src.nC + kChunk - 1) / kChunk;
    // A member's walk over its k-ascending triple list: its next kD triples and the raw A keys of
    // the first kD - 1 of them. The two dependent loads (triple -> key of its A block) are issued one
    // advance apart and a key is only decoded when its triple becomes the head, two advances later,
    // so the producer never waits on a load it has just issued.
    struct Walk {
      int64_t pos, end;
      uint2 t[kD];
      uint64_t rk[kD - 1];
    };
    Walk w, nw;
    int64_t chunk = blockIdx.x, first = -1, nfirst = -1;
    uint32_t heads = 0, mask = 0, nmask = 0;
    bool claimed = false;
    auto chunk_heads = [&](int64_t q) -> uint32_t {
      const int64_t c = q * kChunk + lane;
      bool head = false;
      if (lane < kChunk && c < src.nC) head = c == 0 || (src.c_keys[c] >> 2) != (src.c_keys[c - 1] >> 2);
      return __ballot_sync(0xffffffffu, head);
    };
    auto next_quad = [&]() -> int64_t {  // first C block of this CTA's next quad (-1: none left)
      while (heads == 0u) {
        unsigned long long got = 0;
        if (lane == 0) got = atomicAdd(counter, 1ull);
        chunk = (int64_t)gridDim.x + (int64_t)__shfl_sync(0xffffffffu, got, 0);
        if (chunk >= nQ) return -1;
        heads = chunk_heads(chunk);
      }
      const int h = __ffs(heads) - 1;
      heads &= heads - 1u;
      return chunk * kChunk + h;
    };
    // Members of the quad starting at C block c0, and the start of this lane's walk.
    auto open = [&](int64_t c0, Walk &x, uint32_t &mk) {
      x.pos = x.end = 0;
      mk = 0;
      if (c0 >= 0) {
        const bool in = lane < 4 && c0 + lane < src.nC;
        const uint64_t key = in ? src.c_keys[c0 + lane] : 0ull;
        const uint64_t code0 = __shfl_sync(0xffffffffu, key >> 2, 0);
        const uint32_t eq = __ballot_sync(0xffffffffu, in && (key >> 2) == code0);
        const int nm = __ffs(~eq) - 1;  // run of keys with the quad's code from lane 0
        mk = __reduce_or_sync(0xffffffffu, lane < nm ? 1u << (uint32_t)(key & 3ull) : 0u);
        if (lane < 4 && ((mk >> lane) & 1u)) {  // members are in key order = slot order
          const int m = __popc(mk & ((1u << lane) - 1u));
          x.pos = src.c_tptr[c0 + m];
          x.end = src.c_tptr[c0 + m + 1];
        }
      }
#pragma unroll
      for (int d = 0; d < kD; ++d) x.t[d] = x.pos + d < x.end ? src.tri[x.pos + d] : make_uint2(0u, 0u);
#pragma unroll
      for (int d = 0; d + 1 < kD; ++d) x.rk[d] = x.pos + d < x.end ? src.a_keys[x.t[d].x] : 0ull;
    };
    auto head_k = [&](const Walk &x) -> uint32_t {
      uint32_t bi, bj = kQNone;
      if (x.pos < x.end) qkey_decode(x.rk[0], src.nbl, src.lbits, &bi, &bj);
      return bj;
    };
    if (chunk < nQ) {
      heads = chunk_heads(chunk);
      first = next_quad();
    }
    open(first, w, mask);
    uint32_t k0 = head_k(w);
    uint32_t kmin = __reduce_min_sync(0xffffffffu, k0);
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
        const uint32_t rem = __reduce_max_sync(0xffffffffu, (uint32_t)(w.end - w.pos));
        if (rem <= (uint32_t)kAhead) {
          nfirst = next_quad();
          open(nfirst, nw, nmask);
          claimed = true;
        }
      }
      const bool hit = k0 == kmin;
      const uint32_t hits = __ballot_sync(0xffffffffu, hit) & 0xfu;
      const uint32_t mine = hits & sel;
      const int from = mine ? __ffs(mine) - 1 : 0;
      const uint32_t av = __shfl_sync(0xffffffffu, w.t[0].x, from), bv = __shfl_sync(0xffffffffu, w.t[0].y, from);
      const uint32_t cur = mine ? (is_a ? av : bv) : kQNone;
      if (hit) {
#pragma unroll
        for (int d = 0; d + 1 < kD; ++d) w.t[d] = w.t[d + 1];
#pragma unroll
        for (int d = 0; d + 2 < kD; ++d) w.rk[d] = w.rk[d + 1];
        ++w.pos;
        w.t[kD - 1] = w.pos + kD - 1 < w.end ? src.tri[w.pos + kD - 1] : make_uint2(0u, 0u);
        w.rk[kD - 2] = w.pos + kD - 2 < w.end ? src.a_keys[w.t[kD - 2].x] : 0ull;  // t[kD-2]: loaded an advance ago
        k0 = head_k(w);
      }
      const uint32_t knext = __reduce_min_sync(0xffffffffu, k0);
      const bool last = knext == kQNone;
      if (lane == 0) mbar_wait(&empty[s], phase ^ 1u);
      __syncwarp();
      const uint32_t pm = __ballot_sync(0xffffffffu, cur != kQNone);
      uint8_t *st = smem + (size_t)s * kQStage;
      if (lane == 0) {
        meta[s] = (first << 32) | (int64_t)(mask << 8) | (int64_t)(hits << 1) | (last ? 1 : 0);
        mbar_expect_tx(&full[s], (uint32_t)__popc(pm) * kQLoad);
      }
      __syncwarp();
      if (cur != kQNone)
        tma_load_2d(st + dst_off, is_a ? map_a : map_b, sub * 16, (int)(cur * kQB), &full[s]);
      if (++s == STAGES) {
        s = 0;
        phase ^= 1u;
      }
      kmin = knext;
      if (last) {
        if (!claimed) {
          nfirst = next_quad();
          open(nfirst, nw, nmask);
        }
        first = nfirst;
        w = nw;
        mask = nmask;
        claimed = false;
        k0 = head_k(w);
        kmin = __reduce_min_sync(0xffffffffu, k0);
      }
    }
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB)
    k_numeric_quad32(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     const QuadSrc src, double *__restrict__ C, double *__restrict__ csq, uint8_t *__restrict__ cnz,
                     int64_t *__restrict__ zero_count, unsigned long long *__restrict__ counter, uint64_t zmask) {
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *full = (uint64_t *)(smem + (size_t)STAGES * kQStage);
  uint64_t *empty = full + STAGES;
  // per stage: first C block << 32 | member mask << 8 | hit mask << 1 | last; -1 = end
  volatile int64_t *meta = (volatile int64_t *)(empty + STAGES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kQCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == kQCW) {
    quad_producer<Cfg>(&map_a, &map_b, src, smem, full, empty, meta, counter);
    return;
  }

  // ---------------- consumers: warp w = member slot w, a 32x32 tile (4 x 4 m8n8 accumulators) ----------------
  const int g = lane >> 2, tq = lane & 3;
  const int wm0 = (warp >> 1) * 32, wn0 = (warp & 1) * 32;
  // (the fragment's second 8-column half, h = 1, is the first one's offset with bit 6 flipped:
  // ((4 + (g >> 1)) ^ (kk & 7)) << 4 = (((g >> 1) ^ (kk & 7)) << 4) ^ 64 -- four offsets fewer to keep)
  uint32_t aoff[4], boff[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int kk = kperm(tq, j);
    aoff[j] = g * 128 + (((kk >> 1) ^ g) << 4) + (kk & 1) * 8;
    boff[j] = kk * 128 + (((g >> 1) ^ (kk & 7)) << 4) + (g & 1) * 8;
  }
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int n = 0; n < 4; ++n) acc[i][n][0] = acc[i][n][1] = 0.0;
  int s = 0;
  uint32_t phase = 0;
  while (true) {
    mbar_wait(&full[s], phase);
    const int64_t mt = meta[s];
    if (mt < 0) break;
    uint64_t dep = 0;
    if (((uint32_t)mt >> (1 + warp)) & 1u) {  // this member has a triple at the stage's k
      const uint8_t *sa = smem + (size_t)s * kQStage;
      const uint8_t *sb = sa + kQABytes;
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
        const uint8_t *pa = sa + kb * kQASP + wm0 * 128;
        const uint8_t *pb = sb + kb * 16 * 128;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          double af[4], bf[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) af[i] = *(const double *)(pa + i * 8 * 128 + aoff[j]);
#pragma unroll
          for (int n = 0; n < 4; ++n) {
            const int col = wn0 + n * 8;
            bf[n] = *(const double *)(pb + (col >> 4) * kQBSP + (boff[j] ^ (uint32_t)(((col & 15) >> 3) << 6)));
          }
          if (kb == 1 && j == 3) {
#pragma unroll
            for (int i = 0; i < 4; ++i) dep |= (uint64_t)__double_as_longlong(af[i]);
#pragma unroll
            for (int n = 0; n < 4; ++n) dep |= (uint64_t)__double_as_longlong(bf[n]);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int n = 0; n < 4; ++n) dmma(acc[i][n][0], acc[i][n][1], af[i], bf[n]);
        }
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
      // (No branch on "is this warp's member present" around the accumulator reads: ptxas renames the
      // accumulators around such a branch -- DMMAs with D != C, moves and spills in the stage loop.
      // An absent member's warp has all-zero accumulators; it runs the same code with its stores
      // and result writes predicated off.)
      const uint32_t gm = ((uint32_t)mt >> 8) & 0xfu;
      const bool member = ((gm >> warp) & 1u) != 0u;
      const int64_t c = (mt >> 32) + __popc(gm & ((1u << warp) - 1u));
      double *cb = C + (size_t)c * kQBlkElems;
      const uint64_t c_policy = l2_evict_first_policy();  // (created here: fewer live registers in the loop)
      // Squared norm in the per-block kernel's order: one partial per 16x16 sub-tile (that kernel's
      // warp tile: same lane <-> element map, same in-lane order, same shuffle tree), the four
      // partials then summed in k_combine_tiles' order -- bitwise the same norm.
      double sum = 0.0;
      bool nz = false;
#pragma unroll
      for (int wi = 0; wi < 2; ++wi)
#pragma unroll
        for (int wn = 0; wn < 2; ++wn) {
          double ss0 = 0.0, ss1 = 0.0;
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int n = 0; n < 2; ++n) {
              const double v0 = acc[2 * wi + i][2 * wn + n][0], v1 = acc[2 * wi + i][2 * wn + n][1];
              if (member)
                st_evict_first(cb + (size_t)((2 * wi + i) * 8 + g) * kQB + (2 * wn + n) * 8 + 2 * tq, v0, v1, c_policy);
              ss0 = fma(v0, v0, ss0);
              ss1 = fma(v1, v1, ss1);
              nz |= (v0 != 0.0) | (v1 != 0.0);
              acc[2 * wi + i][2 * wn + n][0] = acc[2 * wi + i][2 * wn + n][1] = 0.0;
            }
          double ss = ss0 + ss1;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
          sum += ss;  // ((0 + p00) + p01) + p10) + p11
        }
      const bool wnz = __any_sync(0xffffffffu, nz);
      if (member && lane == 0) {
        csq[c] = sum;
        cnz[c] = (uint8_t)wnz;
        if (!wnz && zero_count) atomicAdd((unsigned long long *)zero_count, 1ull);
      }
    }
  }
}

template <class Cfg>
int launch_quad(const CUtensorMap &ma, const CUtensorMap &mb, const QuadSrc &src, double *C, double *csq,
                uint8_t *cnz, int64_t *zc, unsigned long long *counter, cudaStream_t st) {
  static PerDeviceOnce once;
  int rc = once.run([]() -> int {
    QM_CUDA_TRY(cudaFuncSetAttribute(k_numeric_quad32<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)Cfg::SMEM));
    return (int)QM_OK;
  });
  if (rc != QM_OK) return rc;
  int per_sm = 0;
  static PerDeviceInt occupancy;
  rc = occupancy.get(&per_sm, [](int *x) -> int {
    QM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(x, k_numeric_quad32<Cfg>, Cfg::THREADS, Cfg::SMEM));
    return (int)QM_OK;
  });
  if (rc != QM_OK) return rc;
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)device_sm_count() * per_sm;
  const int64_t chunks = (src.nC + 3) / 4;
  if (grid > chunks) grid = chunks;
  k_numeric_quad32<Cfg><<<(int)grid, Cfg::THREADS, Cfg::SMEM, st>>>(ma, mb, src, C, csq, cnz, zc, counter,
                                                                      /*zmask=*/0ull);
  QM_LAUNCHED("k_numeric_quad32");
  return QM_OK;
}

}  // namespace

// QM_QUAD32=0: bs 32 products use the per-block kernel (A/B measurements, bitwise comparison).
// Measured on B200 (R2): C5-32 numeric 255.4 ms against 260.8 ms per block (0.956 vs 0.936 of the
// DMMA peak); banded n = 32768 0.612 vs 0.607 ms. (The first version was 2 % SLOWER than the
// per-block kernel: its epilogue branched on "is this warp's member present" around the accumulator
// reads, and ptxas then renamed the accumulators in the stage loop -- 16-28 of the 128 DMMAs with
// D != C, register moves before every stage and 128 B of spills. With the stores predicated
// instead, the loop is k_numeric_tma's: in-place accumulation, no moves, no spills.)
bool quad32_enabled() {
  const char *e = getenv("QM_QUAD32");
  return !(e && e[0] == '0');
}

// Whether a bs 32 product of nC blocks / nT triples (no support masks, no transposed references, one
// pool per operand) runs as quads. Quads pay when a stage's k is shared by most members: long k
// lists (banded, decay). With about one triple per C block (random patterns) every stage serves a
// single member -- one warp of four working -- and the per-block kernel is twice as fast (measured:
// 21 vs 9 TFLOP/s). The average k-list length decides (QM_QUAD32=1 forces quads, 0 disables them).
bool quad32_selected(const Geometry &g, int64_t nC, int64_t nT) {
  if (g.bs != kQB || g.lbits > 1 || !quad32_enabled() || nC >= ((int64_t)1 << 31)) return false;
  const char *e = getenv("QM_QUAD32");
  return (e && e[0] == '1') || nT >= 8 * nC;
}

// bs 32, one pool per operand, no support masks / transposed references, a leaf of 1 or 2x2 blocks;
// QM_ERR_UNSUPPORTED otherwise (the caller falls back to k_numeric_tma). The workspace only needs
// its first 8 bytes (the chunk counter).
int launch_numeric_quad32(const Geometry &g, const double *A, int64_t nA, const double *B, int64_t nB,
                          const uint64_t *a_keys, const uint32_t *tri, const int64_t *c_tptr,
                          const uint64_t *c_keys, int64_t nC, int64_t nT, double *C, double *csq, uint8_t *cnz,
                          int64_t *zc, void *ws, size_t ws_bytes, cudaStream_t st) {
  if (!a_keys || !c_keys || !ws || ws_bytes < 256 || !quad32_selected(g, nC, nT)) return QM_ERR_UNSUPPORTED;
  if (nA * (int64_t)kQB >= ((int64_t)1 << 31) || nB * (int64_t)kQB >= ((int64_t)1 << 31)) return QM_ERR_UNSUPPORTED;
  CUtensorMap ma, mb;
  int rc = make_map(&ma, A, nA, kQB, kQB);
  if (rc != QM_OK) return rc;
  rc = make_map(&mb, B, nB, kQB, kQB);
  if (rc != QM_OK) return rc;
  unsigned long long *counter = (unsigned long long *)ws;
  QM_CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st));
  const QuadSrc src{c_keys, a_keys, (const uint2 *)tri, c_tptr, nC, g.nbl, g.lbits};
  // Three CTAs per SM with two stages (C5-32 255.4 ms; two CTAs with three stages, QM_QUAD32_VARIANT=deep:
  // 260.2 ms).
  const char *v = getenv("QM_QUAD32_VARIANT");
  const bool deep = v ? strcmp(v, "deep") == 0 : false;
  if (deep) return launch_quad<QCfg<3, 2>>(ma, mb, src, C, csq, cnz, zc, counter, st);
  return launch_quad<QCfg<2, 3>>(ma, mb, src, C, csq, cnz, zc, counter, st);
}

}  // namespace qm

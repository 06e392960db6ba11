// Numeric phase for 16x16 blocks (the reference API's default block_size): grouped C blocks.
//
// A 16x16 triple is 8 KFLOP for 4 KB of operands, 2 flop/byte: with one C block per work unit the
// kernel streams every A and B block from L2 once per triple and is bound by L2->SM bandwidth
// (the cp.async kernel reaches ~50% of the DMMA peak). Here a work unit is a *group*: the up to 8
// C blocks of one leaf row segment (same block row i, consecutive in quadtree-key order, since a
// leaf stores its blocks row-major -- BlockSparseLeaf.encode). They share the A blocks A(i,k), so a
// pipeline stage carries one A block and the B blocks B(k, j) of the members that have that k:
// up to 8 products for 18 KB, 3.6 flop/byte.
//
//   k_group_merge: one warp per group merges the members' k-ascending triple lists into the
//     group's union of k (one entry per k: the A index and up to 8 B indices, absent =
//     0xffffffff), stored in the group's own triple range;
//   k_numeric_group16: warp-specialised like k_numeric_tma (one TMA producer warp, mbarrier ring),
//     8 consumer warps, warp w owns member w: a 16x16 accumulator fed only by the entries that
//     contain its k (so each C block sums exactly its own triples, k ascending -- the order of
//     BlockSparseLeaf.multiply, block_sparse.py:121-129), and writes the block, its sum of squares
//     and exact-zero flag (_set_block, block_sparse.py:37-41) when the group ends.
#include <cub/cub.cuh>

#include "qm_common.cuh"
#include "qm_tma.cuh"

namespace qm {
namespace {

constexpr int kG = 8;                         // members per group
constexpr int kBlk = 16;                      // block size
constexpr int kBlkBytes = kBlk * kBlk * 8;    // 2 KB
constexpr int kMPW = 2;                       // members per consumer warp (16x32 warp tile)
constexpr int kCW = kG / kMPW;                // consumer warps
constexpr int kStages = 3;
constexpr int kStageBytes = (1 + kG) * kBlkBytes;
constexpr int kThreads = 32 * (kCW + 1);
constexpr int kMinBlocks = 4;
constexpr size_t kSmem = 1024 + (size_t)kStages * kStageBytes + 4 * kStages * 8 + 64;
constexpr uint32_t kAbsent = 0xffffffffu;

struct Entry {
  uint32_t a;
  uint32_t b[kG];
};

// Group of C block c: its key without the low member bits (same leaf, same block row, aligned runs
// of up to 8 block columns); member slot = those low bits.
__device__ __forceinline__ uint64_t group_code(uint64_t key, int mbits) { return key >> mbits; }

__global__ void k_group_heads(const uint64_t *c_keys, int64_t nC, int mbits, int64_t *head) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= nC; c += (int64_t)gridDim.x * blockDim.x)
    head[c] = (c < nC && (c == 0 || group_code(c_keys[c], mbits) != group_code(c_keys[c - 1], mbits))) ? 1 : 0;
}

// k (block column of the A block) of every triple.
__global__ void k_triple_k(const uint2 *tri, int64_t nT, const uint64_t *a_keys, int nbl, int lbits, uint32_t *tk) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nT; t += (int64_t)gridDim.x * blockDim.x) {
    uint32_t bi, bj;
    qkey_decode(a_keys[tri[t].x], nbl, lbits, &bi, &bj);
    tk[t] = bj;
  }
}

// One warp per group (at its head C block): lane s owns the member in slot s (if any) and walks
// its k-ascending triple list; each step takes the smallest head k over the lanes (warp min) and
// every lane holding it contributes its B index to the entry (9 words written by 9 lanes). The
// group's entries go to its own triple range [c_tptr[first], ...): the union of the members' k
// is never longer than their triple lists together, so no count pass is needed.
__global__ void k_group_merge(const uint64_t *c_keys, const int64_t *c_tptr, const uint2 *tri, const uint32_t *tk,
                              int64_t nC, int mbits, const int64_t *head, const int64_t *gidx, int64_t *ucount,
                              int64_t *gfirst, uint32_t *gmask, Entry *entries, int64_t *n_groups) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t c0 = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c0 < nC; c0 += warps) {
    if (!head[c0]) continue;  // warp-uniform
    const int64_t g = gidx[c0];
    int nm = 1;
    while (nm < kG && c0 + nm < nC && !head[c0 + nm]) ++nm;
    int64_t pos = 0, end = 0;
    uint32_t mask = 0;
    for (int m = 0; m < nm; ++m) {
      const int sl = (int)(c_keys[c0 + m] & ((1ull << mbits) - 1ull));
      mask |= 1u << sl;
      if (lane == sl) {
        pos = c_tptr[c0 + m];
        end = c_tptr[c0 + m + 1];
      }
    }
    Entry *out = entries + c_tptr[c0];
    int64_t cnt = 0;
    while (true) {
      const uint32_t myk = (lane < kG && pos < end) ? tk[pos] : 0xffffffffu;
      const uint32_t kmin = __reduce_min_sync(0xffffffffu, myk);
      if (kmin == 0xffffffffu) break;
      const bool hit = myk == kmin;
      const unsigned hits = __ballot_sync(0xffffffffu, hit);
      const uint32_t my_a = hit ? tri[pos].x : 0u;
      const uint32_t a = __shfl_sync(0xffffffffu, my_a, __ffs(hits) - 1);
      uint32_t *ew = reinterpret_cast<uint32_t *>(out + cnt);
      if (lane == kG) ew[0] = a;  // Entry::a
      if (lane < kG) ew[1 + lane] = hit ? tri[pos].y : kAbsent;
      if (hit) ++pos;
      ++cnt;
    }
    if (lane == 0) {
      ucount[g] = cnt;
      gfirst[g] = c0;
      gmask[g] = mask;
      if (c0 + nm == nC) *n_groups = g + 1;
    }
  }
}

__global__ void __launch_bounds__(kThreads, kMinBlocks)
    k_numeric_group16(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                      const Entry *__restrict__ entries, const int64_t *__restrict__ c_tptr,
                      const int64_t *__restrict__ ucount,
                      const int64_t *__restrict__ gfirst, const uint32_t *__restrict__ gmask,
                      const int64_t *__restrict__ n_groups_dev, double *__restrict__ C, double *__restrict__ csq,
                      uint8_t *__restrict__ cnz, int64_t *__restrict__ zero_count,
                      unsigned long long *__restrict__ counter, uint64_t zmask) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *full = (uint64_t *)(smem + (size_t)kStages * kStageBytes);
  uint64_t *empty = full + kStages;
  volatile int64_t *meta = (volatile int64_t *)(empty + kStages);       // unit*2 + last, -1 = end
  volatile uint32_t *pmask = (volatile uint32_t *)(meta + kStages);     // members present in the entry
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nG = *n_groups_dev;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == kCW) {
    // ---------------- producer warp: one stage per entry; lane m < 8 loads member m's B block,
    // lane 8 the A block, so the up to 9 TMA loads of a stage issue together. The entry of the
    // next stage (and the next claimed group) is loaded one stage ahead.
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&map_a) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&map_b) : "memory");
    }
    const uint32_t *ew = reinterpret_cast<const uint32_t *>(entries);
    const int word = lane < kG ? 1 + lane : 0;  // Entry layout: a, b[0..7]
    int64_t unit = blockIdx.x, e = 0, e1 = 0;
    uint32_t cur = kAbsent;
    if (unit < nG) {
      e = c_tptr[gfirst[unit]];
      e1 = e + ucount[unit];
      if (lane <= kG) cur = ew[e * (1 + kG) + word];
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
        if (nunit < nG && lane <= kG) nxt = ew[ne * (1 + kG) + word];
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
      const uint32_t pm = __ballot_sync(0xffffffffu, lane < kG && cur != kAbsent);
      uint8_t *st = smem + (size_t)s * kStageBytes;
      if (lane == 0) {
        meta[s] = unit * 2 + (e + 1 == e1 ? 1 : 0);
        pmask[s] = pm;
        mbar_expect_tx(&full[s], (uint32_t)(1 + __popc(pm)) * kBlkBytes);
      }
      __syncwarp();
      if (lane == kG) tma_load_2d(st, &map_a, 0, (int)(cur * kBlk), &full[s]);
      else if (lane < kG && cur != kAbsent)
        tma_load_2d(st + (1 + lane) * kBlkBytes, &map_b, 0, (int)(cur * kBlk), &full[s]);
      unit = nunit;
      e = ne;
      e1 = ne1;
      cur = nxt;
      if (++s == kStages) {
        s = 0;
        phase ^= 1u;
      }
    }
    return;
  }

  // -------- consumers: warp w = members 2w, 2w+1 (16x32: the A fragments serve both) --------
  const int g = lane >> 2, tq = lane & 3;
  uint32_t aoff[4], boff[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int kk = kperm(tq, j);
    aoff[j] = g * 128 + (((kk >> 1) ^ g) << 4) + (kk & 1) * 8;
#pragma unroll
    for (int h = 0; h < 2; ++h) boff[j][h] = kk * 128 + ((((h * 4) + (g >> 1)) ^ (kk & 7)) << 4) + (g & 1) * 8;
  }
  const uint64_t c_policy = l2_evict_first_policy();
  double acc[kMPW][2][2][2];
#pragma unroll
  for (int q = 0; q < kMPW; ++q)
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int n = 0; n < 2; ++n) acc[q][i][n][0] = acc[q][i][n][1] = 0.0;
  int s = 0;
  uint32_t phase = 0;
  while (true) {
    mbar_wait(&full[s], phase);
    const int64_t mt = meta[s];
    if (mt < 0) break;
    const uint32_t on = (pmask[s] >> (kMPW * warp)) & ((1u << kMPW) - 1u);
    uint64_t dep = 0;
    if (on) {
      const uint8_t *sa = smem + (size_t)s * kStageBytes;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double af[2], bf[kMPW][2];
#pragma unroll
        for (int i = 0; i < 2; ++i) af[i] = *(const double *)(sa + i * 8 * 128 + aoff[j]);
#pragma unroll
        for (int q = 0; q < kMPW; ++q)
          if (on & (1u << q)) {
            const uint8_t *sb = sa + (1 + kMPW * warp + q) * kBlkBytes;
#pragma unroll
            for (int n = 0; n < 2; ++n) bf[q][n] = *(const double *)(sb + boff[j][n]);
          }
        if (j == 3) {
#pragma unroll
          for (int i = 0; i < 2; ++i) dep |= (uint64_t)__double_as_longlong(af[i]);
#pragma unroll
          for (int q = 0; q < kMPW; ++q)
            if (on & (1u << q))
#pragma unroll
              for (int n = 0; n < 2; ++n) dep |= (uint64_t)__double_as_longlong(bf[q][n]);
        }
#pragma unroll
        for (int q = 0; q < kMPW; ++q)
          if (on & (1u << q))
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
              for (int n = 0; n < 2; ++n) dmma(acc[q][i][n][0], acc[q][i][n][1], af[i], bf[q][n]);
      }
    }
    // release once this warp's fragments are in registers (see k_numeric_tma)
    dep &= zmask;
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s] + (uint32_t)dep);
    if (++s == kStages) {
      s = 0;
      phase ^= 1u;
    }
    if (mt & 1) {
      const int64_t unit = mt >> 1;
      const uint32_t gm = gmask[unit];
#pragma unroll
      for (int q = 0; q < kMPW; ++q) {
        const int mb = kMPW * warp + q;
        if ((gm >> mb) & 1u) {
          const int64_t c = gfirst[unit] + __popc(gm & ((1u << mb) - 1u));
          double *cb = C + (size_t)c * (kBlk * kBlk);
          double ss0 = 0.0, ss1 = 0.0;
          bool nz = false;
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int n = 0; n < 2; ++n) {
              const double v0 = acc[q][i][n][0], v1 = acc[q][i][n][1];
              st_evict_first(cb + (size_t)(i * 8 + g) * kBlk + n * 8 + 2 * tq, v0, v1, c_policy);
              ss0 = fma(v0, v0, ss0);
              ss1 = fma(v1, v1, ss1);
              nz |= (v0 != 0.0) | (v1 != 0.0);
            }
          double ss = ss0 + ss1;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
          const bool wnz = __any_sync(0xffffffffu, nz);
          if (lane == 0) {
            csq[c] = ss;
            cnz[c] = (uint8_t)wnz;
            if (!wnz && zero_count) atomicAdd((unsigned long long *)zero_count, 1ull);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < kMPW; ++q)
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int n = 0; n < 2; ++n) acc[q][i][n][0] = acc[q][i][n][1] = 0.0;
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
  Entry *entries;
  uint32_t *tk;
  void *cub;
  size_t cub_bytes;
};

GroupWs carve_group(Carver &cv, int64_t nC, int64_t nT) {
  GroupWs w;
  w.head = cv.take<int64_t>(nC + 1);
  w.gidx = cv.take<int64_t>(nC + 1);
  w.ucount = cv.take<int64_t>(nC + 1);
  w.gfirst = cv.take<int64_t>(nC + 1);
  w.n_groups = cv.take<int64_t>(1);
  w.gmask = cv.take<uint32_t>(nC + 1);
  w.counter = cv.take<unsigned long long>(1);
  w.entries = cv.take<Entry>(std::max<int64_t>(nT, 1));  // one entry per distinct k: <= triples
  w.tk = cv.take<uint32_t>(std::max<int64_t>(nT, 1));
  w.cub_bytes = scan_bytes(nC + 1);
  w.cub = cv.take<char>(w.cub_bytes);
  return w;
}

}  // namespace

size_t numeric_group16_ws_bytes(int64_t nC, int64_t nT) {
  Carver cv(nullptr, 0);
  carve_group(cv, nC, nT);
  return cv.off;
}

// bs 16 with at least two blocks per leaf side; QM_ERR_UNSUPPORTED otherwise (caller falls back).
int launch_numeric_group16(const Geometry &g, const double *A, int64_t nA, const double *B, int64_t nB,
                           const uint64_t *a_keys, const uint32_t *tri, const int64_t *c_tptr,
                           const uint64_t *c_keys, int64_t nC, int64_t nT, double *C, double *csq,
                           uint8_t *cnz, int64_t *zc, void *ws, size_t ws_bytes, cudaStream_t st) {
  if (g.bs != kBlk || g.nbl < 2 || !a_keys || !c_keys) return QM_ERR_UNSUPPORTED;
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
  const int mbits = std::min(g.lbits, 3);
  const uint2 *t2 = (const uint2 *)tri;
  k_group_heads<<<grid_for(nC + 1), 256, 0, st>>>(c_keys, nC, mbits, w.head);
  QM_LAUNCHED("k_group_heads");
  size_t tb = w.cub_bytes;
  QM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(w.cub, tb, w.head, w.gidx, nC + 1, st));
  k_triple_k<<<grid_for(nT), 256, 0, st>>>(t2, nT, a_keys, g.nbl, g.lbits, w.tk);
  QM_LAUNCHED("k_triple_k");
  const int merge_grid = (int)std::min<int64_t>((nC + 7) / 8, 148 * 64);
  k_group_merge<<<merge_grid, 256, 0, st>>>(c_keys, c_tptr, t2, w.tk, nC, mbits, w.head, w.gidx, w.ucount,
                                            w.gfirst, w.gmask, w.entries, w.n_groups);
  QM_LAUNCHED("k_group_merge");
  CUtensorMap ma, mb;
  int rc = make_map(&ma, A, nA, kBlk, kBlk);
  if (rc != QM_OK) return rc;
  rc = make_map(&mb, B, nB, kBlk, kBlk);
  if (rc != QM_OK) return rc;
  static PerDeviceOnce once;
  rc = once.run([]() -> int {
    QM_CUDA_TRY(cudaFuncSetAttribute(k_numeric_group16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
    return (int)QM_OK;
  });
  if (rc != QM_OK) return rc;
  QM_CUDA_TRY(cudaMemsetAsync(w.counter, 0, sizeof(unsigned long long), st));
  int per_sm = 0;
  QM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_numeric_group16, kThreads, kSmem));
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)device_sm_count() * per_sm;
  if (grid > nC) grid = nC;  // groups <= C blocks
  k_numeric_group16<<<(int)grid, kThreads, kSmem, st>>>(ma, mb, w.entries, c_tptr, w.ucount, w.gfirst, w.gmask,
                                                         w.n_groups,
                                                         C, csq, cnz, zc, w.counter, /*zmask=*/0ull);
  QM_LAUNCHED("k_numeric_group16");
  return QM_OK;
}

}  // namespace qm

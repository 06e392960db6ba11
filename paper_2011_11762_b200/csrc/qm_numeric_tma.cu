// Numeric phase v2: warp-specialised TMA + mbarrier pipeline feeding FP64 DMMA.
//
// Same contract as k_numeric_dmma (qm_numeric.cu): each C block is owned by one CTA for its whole
// k list, accumulated in registers in a fixed order, with the fused norm / exact-zero epilogue of
// _set_block (block_sparse.py:37-41) -- the replacement of BlockSparseLeaf.multiply + add
// (block_sparse.py:112-152). What changes is how operands reach the tensor cores:
//
//  * one producer warp per CTA walks the CTA's stage stream (C block -> triple -> k panel) and
//    issues 2-D TMA loads (cp.async.bulk.tensor, SWIZZLE_128B, 16-double = 128-byte sub-panels)
//    into a ring of shared-memory stages, signalling `full[s]` with complete_tx;
//  * consumer warps wait on `full[s]`, run their DMMAs, and release the stage with one arrive on
//    `empty[s]` per warp -- no CTA-wide barrier in the main loop, no LDGSTS or address math in the
//    math warps;
//  * the 4 k values of each m8n8k4 step are a permutation of the 16-double panel chosen so that the
//    A fragment (8 rows x 4 k) and the B fragment (4 k x 8 columns) both hit 16 distinct 8-byte
//    slots of the 128-byte swizzle row per half-warp: bank-conflict free without padding.
//      lane t=0: k = 2j           t=1: k = 8 + 2((j+1)&3)
//      lane t=2: k = 2((j+2)&3)+1 t=3: k = 9 + 2((j+3)&3)      (j = k step 0..3 in the panel)
//    Each k in 0..15 is used exactly once per panel, so the sum is unchanged.
#include <algorithm>

#include <cub/cub.cuh>

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include "qm_common.cuh"
#include "qm_tma.cuh"

namespace qm {
namespace {

// A CTA computes one TILE x TILE tile of a C block (TILE = BS, or 64 for BS = 128: the block is
// then NQ = (BS/TILE)^2 work units whose partial norms are combined in a fixed order afterwards).
// EW (epilogue warp): the consumers write a finished tile into the stage holding the unit's last
// k panel (32 KB = one bs-64 tile) instead of storing it themselves; an extra warp TMA-stores it
// (cp.async.bulk.tensor, SASS UTMASTG) and computes its norm / exact-zero flag from shared memory,
// then hands the stage back to the producer. The math warps' epilogue shrinks to a barrier and 16
// shared stores -- for units of one or two triples (random patterns) it was ~7% of the kernel.
// EW_ = 2: the consumers still compute the norms / flags from registers (only the stores move).
template <int BS_, int TILE_, int WARPS_M_, int WARPS_N_, int KP_, int STAGES_, int MINB_, int EW_ = 0>
struct TmaCfg {
  static constexpr int BS = BS_, TILE = TILE_, WARPS_M = WARPS_M_, WARPS_N = WARPS_N_, KP = KP_;
  static constexpr int STAGES = STAGES_, MINB = MINB_;
  static constexpr bool EW = EW_ != 0, EW_NORM = EW_ == 1;
  static constexpr int NQN = BS / TILE, NQ = NQN * NQN;  // tiles per C block
  static constexpr int NCW = WARPS_M * WARPS_N;         // consumer warps
  static constexpr int NTHR = 32 * (NCW + 1 + (EW ? 1 : 0));  // + one producer warp (+ the epilogue warp)
  static constexpr int NPART = EW_NORM ? 1 : NCW;       // partial norms per work unit
  static constexpr int TM = TILE / WARPS_M, TN = TILE / WARPS_N;
  static constexpr int MT = TM / 8, NT = TN / 8;
  static constexpr int NP = BS / KP;                    // k panels per triple
  static constexpr int KSP = KP / 16;                   // 16-wide k sub-panels per stage (A)
  static constexpr int NSP = TILE / 16;                 // 16-wide column sub-panels (B)
  static constexpr int A_SP_BYTES = TILE * 128;         // one A sub-panel: TILE rows x 16 doubles
  static constexpr int B_SP_BYTES = KP * 128;           // one B sub-panel: KP rows x 16 doubles
  static constexpr int A_BYTES = KSP * A_SP_BYTES;
  static constexpr int B_BYTES = NSP * B_SP_BYTES;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + 5 * STAGES * 8 + 2 * 32 * 8;
  static_assert(!EW || (size_t)TILE * TILE * 8 <= (size_t)STAGE_BYTES, "EW: a C tile must fit in one stage");
  static_assert(KP % 16 == 0 && BS % KP == 0 && TILE % 16 == 0 && BS % TILE == 0, "panels");
  static_assert(TM % 8 == 0 && TN % 8 == 0, "warp tile");
  static_assert(A_SP_BYTES % 1024 == 0 && B_SP_BYTES % 1024 == 0, "swizzle-128B atoms need 1 KB alignment");
};

// Tensor maps of the operand block pools. NPOOL = 1: one local pool per operand. NPOOL > 1: the
// pools of every rank of a multi-GPU product, mapped into this GPU's address space (CUDA IPC /
// peer access); a triple index then packs (owner << kOwnerShift) | local index, and the producer's
// TMA reads the block straight from its owner's HBM over NVLink -- the halo exchange fused into the
// numeric kernel, overlapped with the DMMAs of earlier stages.
constexpr int kOwnerShift = 28;
constexpr uint32_t kLocalMask = (1u << kOwnerShift) - 1u;
constexpr int kMaxPools = 8;

template <int NPOOL, bool TR = false>
struct __align__(64) TmaMaps {
  CUtensorMap a[NPOOL];
  CUtensorMap b[NPOOL];
  CUtensorMap c;  // the C pool (EW variants: TMA stores of finished tiles)
};
// TR: triple indices may carry a transpose flag (bit 31): the stored block is used transposed, the
// reference's virtual transposes (ops.py:100-116) as TMA box / shared-memory addressing choices.
// `at` views the A pool with the B box (KP rows x 16 columns), `bt` the B pool with the A box.
template <int NPOOL>
struct __align__(64) TmaMaps<NPOOL, true> {
  CUtensorMap a[NPOOL];
  CUtensorMap b[NPOOL];
  CUtensorMap c;
  CUtensorMap at, bt;
};
constexpr uint32_t kTransposed = 1u << 31;

// Stage cursor over work units u = m * NQ + q (C block m, tile q), triple t, k panel p.
// `unit` is the claim index; `mu` the work unit it maps to (C block order[unit / NQ], tile unit % NQ;
// order = NULL: the identity, quadtree-key order). `sm` = the k panels of triple t that can
// contribute (tri_sm[t], from the operands' support masks; all NP panels when tri_sm is NULL):
// a panel where A's columns or B's rows are all zero adds exactly zero and is skipped.
struct Cur {
  int64_t unit, mu, t, tend;
  int p;
  uint32_t sm;
};

template <class Cfg>
__device__ __forceinline__ uint32_t triple_panels(const uint8_t *tri_sm, int64_t t) {
  return tri_sm ? (uint32_t)tri_sm[t] : (1u << Cfg::NP) - 1u;
}

template <class Cfg>
__device__ __forceinline__ void cur_start(Cur &c, int64_t unit, int64_t nU, const int64_t *tptr,
                                          const uint32_t *order, const uint8_t *tri_sm) {
  c.unit = unit;
  if (unit < nU) {
    const int64_t m = order ? (int64_t)order[unit / Cfg::NQ] : unit / Cfg::NQ;
    c.mu = m * Cfg::NQ + unit % Cfg::NQ;
    c.t = tptr[m];
    c.tend = tptr[m + 1];
    c.sm = triple_panels<Cfg>(tri_sm, c.t);
  } else {
    c.mu = c.t = c.tend = 0;
    c.sm = 1u;
  }
  c.p = __ffs(c.sm) - 1;
}

// True when the cursor's stage is the unit's last (no later panel of this triple, no later triple:
// every triple has at least one panel).
__device__ __forceinline__ bool cur_last(const Cur &c) {
  return (c.sm & ~((2u << c.p) - 1u)) == 0u && c.t + 1 == c.tend;
}

// Advances the producer's cursor; a finished unit is replaced by the next one claimed from the
// global work counter just in time (claiming a unit ahead widened the window of units in flight
// and raised DRAM re-reads of A/B by 2x with 3 CTAs/SM).
// ahead: the next claim is taken one unit early (*next holds it), so the counter's round trip
// overlaps the current unit's loads instead of stalling the producer between units -- for units of
// one or two stages (about one triple per C block) that latency is a visible share of the unit.
template <class Cfg>
__device__ __forceinline__ void cur_next(Cur &c, int64_t nU, const int64_t *tptr, const uint32_t *order,
                                         const uint8_t *tri_sm, unsigned long long *counter, bool ahead,
                                         int64_t *next) {
  const uint32_t rest = c.sm & ~((2u << c.p) - 1u);
  if (rest) {
    c.p = __ffs(rest) - 1;
  } else if (++c.t == c.tend) {
    if (ahead) {
      const int64_t u = *next;
      *next = u < nU ? (int64_t)gridDim.x + (int64_t)atomicAdd(counter, 1ull) : u;
      cur_start<Cfg>(c, u, nU, tptr, order, tri_sm);
    } else {
      cur_start<Cfg>(c, (int64_t)gridDim.x + (int64_t)atomicAdd(counter, 1ull), nU, tptr, order, tri_sm);
    }
  } else {
    c.sm = triple_panels<Cfg>(tri_sm, c.t);
    c.p = __ffs(c.sm) - 1;
  }
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Halo gather of a staged multi-GPU product: copies the halo blocks from the peer pools (read over
// NVLink) into the local halo pools with bulk copies through shared memory -- the TMA engine moves
// the bytes; kGatherLanes lanes per CTA each keep two chunks in flight (bulk async-groups are
// per thread). It lets the numeric kernel launch right away (programmatic dependent launch); that
// kernel's claims reading the halo execute griddepcontrol.wait, i.e. wait for this grid to finish.
// min_ns (measurement only): the grid does not finish before min_ns after it started (emulates a
// slower link on a one-GPU box).
constexpr int kGatherChunk = 8192, kGatherLanes = 8, kGatherCtas = 32;
constexpr int kGatherSmem = kGatherLanes * 2 * kGatherChunk;

struct GatherArgs {
  const uint32_t *index[2];
  int64_t count[2];
  double *pool[2];
  uint64_t base[2][QM_MAX_RANKS];
  int64_t off[2][QM_MAX_RANKS + 1];
  int32_t world;
  int64_t block_bytes, min_ns;
};

__global__ void __launch_bounds__(32) k_halo_gather(const __grid_constant__ GatherArgs ga) {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  extern __shared__ __align__(128) uint8_t gbuf[];
  __shared__ __align__(8) uint64_t bar[kGatherLanes][2];
  const int lane = threadIdx.x;
  if (lane >= kGatherLanes) return;
  const uint64_t t0 = global_ns();
  mbar_init(&bar[lane][0], 1);
  mbar_init(&bar[lane][1], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  const int64_t cpb = (ga.block_bytes + kGatherChunk - 1) / kGatherChunk;  // chunks per block
  const int64_t jobs = (ga.count[0] + ga.count[1]) * cpb;
  const int64_t first = (int64_t)blockIdx.x * kGatherLanes + lane, step = (int64_t)gridDim.x * kGatherLanes;
  uint8_t *buf[2] = {gbuf + (lane * 2) * kGatherChunk, gbuf + (lane * 2 + 1) * kGatherChunk};
  // chunk j: (source, destination, bytes)
  auto where = [&](int64_t j, uint64_t *src, uint64_t *dst) -> uint32_t {
    int64_t x = j / cpb;
    const int64_t co = (j % cpb) * kGatherChunk;
    const int o = x < ga.count[0] ? 0 : 1;
    if (o) x -= ga.count[0];
    const int64_t gi = ga.index[o][x];
    int r = 0;
    while (r + 1 < ga.world && gi >= ga.off[o][r + 1]) ++r;
    *src = ga.base[o][r] + (uint64_t)(gi - ga.off[o][r]) * (uint64_t)ga.block_bytes + (uint64_t)co;
    *dst = (uint64_t)ga.pool[o] + (uint64_t)x * (uint64_t)ga.block_bytes + (uint64_t)co;
    const int64_t rest = ga.block_bytes - co;
    return (uint32_t)(rest < kGatherChunk ? rest : (int64_t)kGatherChunk);
  };
  auto load = [&](int64_t j, int b) {
    uint64_t src, dst;
    const uint32_t bytes = where(j, &src, &dst);
    mbar_expect_tx(&bar[lane][b], bytes);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(buf[b])),
        "l"(src), "r"(bytes), "r"(smem_u32(&bar[lane][b]))
        : "memory");
  };
  if (first < jobs) load(first, 0);
  if (first + step < jobs) load(first + step, 1);
  for (int64_t k = 0; first + k * step < jobs; ++k) {
    const int b = (int)(k & 1);
    mbar_wait(&bar[lane][b], (uint32_t)((k >> 1) & 1));
    uint64_t src, dst;
    const uint32_t bytes = where(first + k * step, &src, &dst);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(buf[b])),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    if (first + (k + 2) * step < jobs) {
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // buf b has been read out
      load(first + (k + 2) * step, b);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  while (ga.min_ns > 0 && global_ns() - t0 < (uint64_t)ga.min_ns) __nanosleep(1000);
}

template <class Cfg, int NPOOL, bool TR>
__global__ void __launch_bounds__(Cfg::NTHR, Cfg::MINB)
    k_numeric_tma(const __grid_constant__ TmaMaps<NPOOL, TR> maps,
                  const uint2 *__restrict__ tri, const int64_t *__restrict__ tptr, int64_t nC,
                  double *__restrict__ C, double *__restrict__ csq, uint8_t *__restrict__ cnz,
                  int64_t *__restrict__ zero_count, double *__restrict__ part_sq,
                  uint8_t *__restrict__ part_nz, unsigned long long *__restrict__ counter,
                  const uint32_t *__restrict__ order, const uint8_t *__restrict__ tri_sm, uint64_t zmask,
                  bool claim_ahead, int64_t gate_units) {
  constexpr int BS = Cfg::BS, MT = Cfg::MT, NT = Cfg::NT, STAGES = Cfg::STAGES;
  const int64_t nU = nC * Cfg::NQ;
  // Align to 1 KB (SWIZZLE_128B atoms) by offsetting the __shared__ array itself: the pointer keeps
  // the shared address space, so fragment loads are LDS (not generic LD) and stay ordered before
  // the stage-release mbarrier arrive.
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *full = (uint64_t *)(smem + (size_t)STAGES * Cfg::STAGE_BYTES);
  uint64_t *empty = full + STAGES;
  volatile int64_t *meta = (volatile int64_t *)(empty + STAGES);  // per stage: unit*2 + last, -1 = end
  // EW: finished tiles queued for the epilogue warp: slot j holds (unit << 4 | stage), -1 = end
  uint64_t *cfull = (uint64_t *)(meta + STAGES);
  volatile int64_t *cq = (volatile int64_t *)(cfull + STAGES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::NCW);
      if constexpr (Cfg::EW) mbar_init(&cfull[s], Cfg::NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if constexpr (Cfg::EW) {
    if (warp == Cfg::NCW + 1) {
      // ------------------------------ epilogue warp ------------------------------
      // Per finished tile (in the consumers' order): TMA-store it from its stage (4 column
      // sub-panels of TILE rows x 16 doubles, the SWIZZLE_128B layout the consumers wrote), sum
      // its squares / test it for exact zero from shared memory meanwhile (fixed order: lane =
      // row within each 32-row group, chunks in order, then a fixed shuffle tree), and give the
      // stage back to the producer once the store has read it.
      if (lane == 0) asm volatile("prefetch.tensormap [%0];\n" ::"l"(&maps.c) : "memory");
      const uint64_t c_policy = l2_evict_first_policy();
      for (int64_t j = 0;; ++j) {
        const int q = (int)(j % STAGES);
        mbar_wait(&cfull[q], (uint32_t)((j / STAGES) & 1));
        const int64_t e = cq[q];
        if (e < 0) break;
        const int64_t unit = e >> 4;
        const int s = (int)(e & 15);
        const uint8_t *st = smem + (size_t)s * Cfg::STAGE_BYTES;
        const int64_t m = unit / Cfg::NQ;
        const int qt = (int)(unit % Cfg::NQ);
        const int row0 = (qt / Cfg::NQN) * Cfg::TILE, col0 = (qt % Cfg::NQN) * Cfg::TILE;
        if (lane == 0) {
#pragma unroll
          for (int sp = 0; sp < Cfg::TILE / 16; ++sp)
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;\n" ::"l"(
                    &maps.c),
                "r"(col0 + sp * 16), "r"((int)(m * BS + row0)), "r"(smem_u32(st + sp * Cfg::A_SP_BYTES)),
                "l"(c_policy)
                : "memory");
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
        if constexpr (Cfg::EW_NORM) {
        double ss0 = 0.0, ss1 = 0.0;
        bool nz = false;
#pragma unroll 1
        for (int sp = 0; sp < Cfg::TILE / 16; ++sp)
#pragma unroll
          for (int rr = 0; rr < Cfg::TILE / 32; ++rr) {
            const int r = rr * 32 + lane;
            const uint8_t *row = st + sp * Cfg::A_SP_BYTES + r * 128;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const double2 v = *(const double2 *)(row + ((c ^ (r & 7)) << 4));
              ss0 = fma(v.x, v.x, ss0);
              ss1 = fma(v.y, v.y, ss1);
              nz |= (v.x != 0.0) | (v.y != 0.0);
            }
          }
        double ss = ss0 + ss1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        const bool wnz = __any_sync(0xffffffffu, nz);
        if (lane == 0) {
          part_sq[unit] = ss;
          part_nz[unit] = wnz;
        }
        }
        if (lane == 0) {
          asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // the store has read the stage
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&empty[s])), "r"(Cfg::NCW)
                       : "memory");
        }
        __syncwarp();
      }
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
      return;
    }
  }

  if (warp == Cfg::NCW) {
    // ------------------------------ producer warp ------------------------------
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < NPOOL; ++i) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&maps.a[i]) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&maps.b[i]) : "memory");
      }
      // Dynamic work distribution: the first unit is blockIdx.x, later ones come from a global
      // counter in key order (so concurrently running CTAs still share A/B rows/columns in L2)
      // and no CTA is left with a long tail of heavy units.
      Cur L;
      cur_start<Cfg>(L, blockIdx.x, nU, tptr, order, tri_sm);
      int64_t next = claim_ahead && L.unit < nU ? (int64_t)gridDim.x + (int64_t)atomicAdd(counter, 1ull) : nU;
      int s = 0;
      uint32_t phase = 0;
      bool gated = gate_units < nU;  // claims >= gate_units read the staged halo
#if defined(QM_EXP_DEPHASE) && QM_EXP_DEPHASE > 0
      if (blockIdx.x >= gridDim.x / 2) __nanosleep(QM_EXP_DEPHASE);
#endif
      while (true) {
        mbar_wait(&empty[s], phase ^ 1u);
        if (L.unit >= nU) {
          meta[s] = -1;
          mbar_arrive(&full[s]);  // tx-free completion: tells the consumers to stop
          break;
        }
        if (gated && L.unit >= gate_units) {
          // the halo gather (the preceding grid, programmatic dependent launch) has completed and
          // its bulk stores are visible; then order this generic-proxy wait before the TMA reads
          asm volatile("griddepcontrol.wait;\n" ::: "memory");
          asm volatile("fence.proxy.async.global;\n" ::: "memory");
          gated = false;
        }
        const uint2 ab = tri[L.t];
        const uint32_t ao = NPOOL > 1 ? ab.x >> kOwnerShift : 0u;
        const uint32_t bo = NPOOL > 1 ? ab.y >> kOwnerShift : 0u;
        uint32_t al = NPOOL > 1 ? ab.x & kLocalMask : ab.x, bl = NPOOL > 1 ? ab.y & kLocalMask : ab.y;
        uint32_t ta = 0, tb = 0;
        if constexpr (TR) {
          ta = al >> 31;
          tb = bl >> 31;
          al &= ~kTransposed;
          bl &= ~kTransposed;
        }
        const int qt = (int)(L.mu % Cfg::NQ);
        const int row0 = (qt / Cfg::NQN) * Cfg::TILE, col0 = (qt % Cfg::NQN) * Cfg::TILE;
        uint8_t *st = smem + (size_t)s * Cfg::STAGE_BYTES;
        if constexpr (TR)
          meta[s] = ((L.mu * 2 + (cur_last(L) ? 1 : 0)) << 2) | (ta << 1) | tb;
        else
          meta[s] = L.mu * 2 + (cur_last(L) ? 1 : 0);
        mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
        if (TR && ta) {  // A(i,k) = S^T: S's rows k of the panel, columns = the tile's rows (B box)
          if constexpr (TR) {
#pragma unroll
            for (int q = 0; q < Cfg::TILE / 16; ++q)
              tma_load_2d(st + q * Cfg::B_SP_BYTES, &maps.at, row0 + q * 16, (int)(al * BS + L.p * Cfg::KP),
                          &full[s]);
          }
        } else {
#pragma unroll
          for (int q = 0; q < Cfg::KSP; ++q)
            tma_load_2d(st + q * Cfg::A_SP_BYTES, &maps.a[ao], L.p * Cfg::KP + q * 16, (int)(al * BS + row0),
                        &full[s]);
        }
        if (TR && tb) {  // B(k,j) = S^T: S's rows = the tile's columns, columns k of the panel (A box)
          if constexpr (TR) {
#pragma unroll
            for (int q = 0; q < Cfg::KSP; ++q)
              tma_load_2d(st + Cfg::A_BYTES + q * Cfg::A_SP_BYTES, &maps.bt, L.p * Cfg::KP + q * 16,
                          (int)(bl * BS + col0), &full[s]);
          }
        } else {
#pragma unroll
          for (int q = 0; q < Cfg::NSP; ++q)
            tma_load_2d(st + Cfg::A_BYTES + q * Cfg::B_SP_BYTES, &maps.b[bo], col0 + q * 16,
                        (int)(bl * BS + L.p * Cfg::KP), &full[s]);
        }
        cur_next<Cfg>(L, nU, tptr, order, tri_sm, counter, claim_ahead, &next);
        if (++s == STAGES) {
          s = 0;
          phase ^= 1u;
        }
      }
    }
    return;
  }

  // ------------------------------ consumer warps ------------------------------
  const int g = lane >> 2, tq = lane & 3;
  const uint64_t c_policy = l2_evict_first_policy();
  const int wm0 = (warp / Cfg::WARPS_N) * Cfg::TM;
  const int wn0 = (warp % Cfg::WARPS_N) * Cfg::TN;
  // Per-lane swizzled byte offsets of the fragment elements (see kperm).
  uint32_t aoff[4], boff[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int kk = kperm(tq, j);
    aoff[j] = g * 128 + (((kk >> 1) ^ g) << 4) + (kk & 1) * 8;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c0 = h * 4;  // (n % 16) / 2 of the fragment's first column: 0 or 4
      boff[j][h] = kk * 128 + (((c0 + (g >> 1)) ^ (kk & 7)) << 4) + (g & 1) * 8;
    }
  }

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  int s = 0;
  uint32_t phase = 0;
  int64_t jq = 0;  // EW: tiles queued so far
  while (true) {
    mbar_wait(&full[s], phase);
    int64_t mt = meta[s];
    if (mt < 0) {
      if constexpr (Cfg::EW) {  // tell the epilogue warp to finish
        __syncwarp();
        if (lane == 0) {
          if (warp == 0) cq[jq % STAGES] = -1;
          mbar_arrive(&cfull[jq % STAGES]);
        }
      }
      break;
    }
    bool ta = false, tb = false;
    if constexpr (TR) {
      ta = (mt >> 1) & 1;
      tb = mt & 1;
      mt >>= 2;
    }
    const uint8_t *sa = smem + (size_t)s * Cfg::STAGE_BYTES;
    const uint8_t *sb = sa + Cfg::A_BYTES;
    uint64_t dep = 0;
#pragma unroll
    for (int kb = 0; kb < Cfg::KSP; ++kb) {
      const uint8_t *pa = sa + kb * Cfg::A_SP_BYTES + wm0 * 128;
      const uint8_t *pb = sb + kb * 16 * 128;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double af[MT], bf[NT];
        // A transposed (TR): the stage holds S^T's panel in the B layout, so A's fragment is read
        // with B's addressing (same lane <-> (row, k) map: g indexes rows / columns, tq the k);
        // B transposed: the A layout, read with A's addressing.
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          if (TR && ta) {
            const int row = wm0 + i * 8;
            af[i] = *(const double *)(sa + (row >> 4) * Cfg::B_SP_BYTES + kb * 16 * 128 + boff[j][(row & 15) >> 3]);
          } else {
            af[i] = *(const double *)(pa + i * 8 * 128 + aoff[j]);
          }
        }
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const int col = wn0 + n * 8;
          if (TR && tb)
            bf[n] = *(const double *)(sb + kb * Cfg::A_SP_BYTES + col * 128 + aoff[j]);
          else
            bf[n] = *(const double *)(pb + (col >> 4) * Cfg::B_SP_BYTES + boff[j][(col & 15) >> 3]);
        }
        if (kb == Cfg::KSP - 1 && j == 3) {
          // The stage's last fragment loads: the release below depends on their values.
#pragma unroll
          for (int i = 0; i < MT; ++i) dep |= (uint64_t)__double_as_longlong(af[i]);
#pragma unroll
          for (int n = 0; n < NT; ++n) dep |= (uint64_t)__double_as_longlong(bf[n]);
        }
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int n = 0; n < NT; ++n) dmma(acc[i][n][0], acc[i][n][1], af[i], bf[n]);
      }
    }
    // Release the stage once every fragment of it is in registers: the arrive's address carries a
    // data dependency on the stage's last shared-memory loads (masked by zmask, a runtime zero), so
    // it cannot be hoisted above them; the DMMAs themselves read registers only, so the warp does
    // not drain its DMMA queue before releasing.
    dep &= zmask;
    __syncwarp();
    if constexpr (Cfg::EW) {
      if (mt & 1) {
        // the unit's last stage becomes its C tile: every consumer warp is past its operand reads
        // (named barrier), then writes its fragments in the TMA store layout and queues the tile;
        // the epilogue warp releases the stage to the producer after storing it
        asm volatile("bar.sync 1, %0;\n" ::"n"(Cfg::NCW * 32) : "memory");
        uint8_t *cs = smem + (size_t)s * Cfg::STAGE_BYTES;
        double ss0 = 0.0, ss1 = 0.0;
        bool nz = false;
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            const int r = wm0 + i * 8 + g, c = wn0 + n * 8 + 2 * tq;
            const uint32_t a = smem_u32(cs + (c >> 4) * Cfg::A_SP_BYTES + r * 128 + ((((c & 15) >> 1) ^ (r & 7)) << 4));
            const double v0 = acc[i][n][0], v1 = acc[i][n][1];
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(a), "d"(v0), "d"(v1) : "memory");
            if constexpr (!Cfg::EW_NORM) {
              ss0 = fma(v0, v0, ss0);
              ss1 = fma(v1, v1, ss1);
              nz |= (v0 != 0.0) | (v1 != 0.0);
            }
            acc[i][n][0] = acc[i][n][1] = 0.0;
          }
        if constexpr (!Cfg::EW_NORM) {
          double ss = ss0 + ss1;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
          const bool wnz = __any_sync(0xffffffffu, nz);
          if (lane == 0) {
            part_sq[(mt >> 1) * Cfg::NPART + warp] = ss;
            part_nz[(mt >> 1) * Cfg::NPART + warp] = wnz;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          if (warp == 0) cq[jq % STAGES] = ((mt >> 1) << 4) | s;
          mbar_arrive(&cfull[jq % STAGES]);
        }
        ++jq;
      } else if (lane == 0) {
        mbar_arrive(&empty[s] + (uint32_t)dep);
      }
    } else {
      if (lane == 0) mbar_arrive(&empty[s] + (uint32_t)dep);
    }
    if (++s == STAGES) {
      s = 0;
      phase ^= 1u;
    }

    if (!Cfg::EW && (mt & 1)) {
      const int64_t unit = mt >> 1;
      const int64_t m = unit / Cfg::NQ;
      const int qt = (int)(unit % Cfg::NQ);
      double *cb = C + (size_t)m * (BS * BS) + (size_t)(qt / Cfg::NQN) * Cfg::TILE * BS +
                   (qt % Cfg::NQN) * Cfg::TILE;
      // Barrier-free epilogue: each warp stores its tile fragment and writes its partial squared
      // norm / nonzero flag for the unit; k_combine_tiles sums the NQ*NCW partials of a block in a
      // fixed order afterwards (deterministic, no named barrier between the consumer warps).
      double ss0 = 0.0, ss1 = 0.0;
      bool nz = false;
      uint32_t nz_lo = 0u, nz_hi = 0u;
#if defined(QM_EXP_EPI) && QM_EXP_EPI == 3
      uint64_t xbits[4] = {0, 0, 0, 0};
#endif
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const double v0 = acc[i][n][0], v1 = acc[i][n][1];
#if !defined(QM_EXP_EPI) || (QM_EXP_EPI != 1 && QM_EXP_EPI != 3)
          st_evict_first(cb + (size_t)(wm0 + i * 8 + g) * BS + wn0 + n * 8 + 2 * tq, v0, v1, c_policy);
#endif
#if defined(QM_EXP_EPI) && QM_EXP_EPI == 3  // experiment: no epilogue work at all (upper bound)
          xbits[(i * NT + n) & 3] ^= (uint64_t)__double_as_longlong(v0) ^ (uint64_t)__double_as_longlong(v1);
#elif defined(QM_EXP_NZ_INT)  // measured slower (C3 1.078 -> 1.130 ms): integer exact-zero test
          ss0 = fma(v0, v0, ss0);
          ss1 = fma(v1, v1, ss1);
          const uint64_t b0 = (uint64_t)__double_as_longlong(v0), b1 = (uint64_t)__double_as_longlong(v1);
          nz_lo |= (uint32_t)b0 | (uint32_t)b1;
          nz_hi |= (uint32_t)(b0 >> 32) | (uint32_t)(b1 >> 32);
#elif defined(QM_EXP_NZ_SS)  // measured slower (C3 1.075 -> 1.18..1.21 ms): exact-zero test from ss
          ss0 = fma(v0, v0, ss0);
          ss1 = fma(v1, v1, ss1);
#else
          ss0 = fma(v0, v0, ss0);
          ss1 = fma(v1, v1, ss1);
          nz |= (v0 != 0.0) | (v1 != 0.0);
#endif
#if !defined(QM_EXP_NZ_SS)
          acc[i][n][0] = acc[i][n][1] = 0.0;
#endif
        }
      double ss = ss0 + ss1;
#if defined(QM_EXP_EPI) && QM_EXP_EPI == 3
      ss = __longlong_as_double((long long)((xbits[0] ^ xbits[1] ^ xbits[2] ^ xbits[3]) & 1ull));
#endif
#if defined(QM_EXP_EPI) && (QM_EXP_EPI == 2 || QM_EXP_EPI == 3)
      const bool wnz = true;
#else
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
#if !defined(QM_EXP_NZ_SS)
      nz |= (nz_lo | (nz_hi & 0x7fffffffu)) != 0u;
#else
      // Exact-zero test (_set_block's np.any) from the sum of squares: a nonzero, NaN or Inf square
      // means a nonzero value. Only a warp whose squares all vanish -- an exactly zero tile, or
      // values so small their squares underflow -- compares its values one by one.
      nz = ss != 0.0;
      if (!nz) {
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int n = 0; n < NT; ++n) nz |= (acc[i][n][0] != 0.0) | (acc[i][n][1] != 0.0);
      }
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int n = 0; n < NT; ++n) acc[i][n][0] = acc[i][n][1] = 0.0;
#endif
      const bool wnz = __any_sync(0xffffffffu, nz);
#endif
      if (lane == 0) {
        part_sq[unit * Cfg::NPART + warp] = ss;
        part_nz[unit * Cfg::NPART + warp] = wnz;
      }
    }
  }
}

// Fixed-order combination of the per-tile partial norms / nonzero flags of NQ-tile C blocks.
__global__ void k_combine_tiles(const double *part_sq, const uint8_t *part_nz, int nq, int64_t nC,
                                double *csq, uint8_t *cnz, int64_t *zero_count, int64_t *panel_count,
                                int64_t panel_fill) {
  if (panel_count && panel_fill >= 0 && blockIdx.x == 0 && threadIdx.x == 0) *panel_count = panel_fill;
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < nC;
       m += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    int any = 0;
    for (int q = 0; q < nq; ++q) {
      s += part_sq[m * nq + q];
      any |= part_nz[m * nq + q];
    }
    csq[m] = s;
    cnz[m] = (uint8_t)(any != 0);
    if (!any && zero_count) atomicAdd((unsigned long long *)zero_count, 1ull);
  }
}

// Claim-order key of each C block: lpt = 0: the k (block column of the A block) of its first
// triple; lpt = 1: the complement of its triple count (longest k list first).
__global__ void k_order_key(const uint2 *tri, const int64_t *tptr, const uint64_t *a_keys, int64_t nC, int nbl,
                            int lbits, int lpt, uint32_t *key, uint32_t *iota) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nC; c += (int64_t)gridDim.x * blockDim.x) {
    uint32_t bi, bj = 0;
    const int64_t t = tptr[c], n = tptr[c + 1] - t;
    if (lpt) bj = ~(uint32_t)(n < 0xffffffffll ? n : 0xffffffffll);
    else if (n > 0) qkey_decode(a_keys[tri[t].x], nbl, lbits, &bi, &bj);
    key[c] = bj;
    iota[c] = (uint32_t)c;
  }
}

// k panels of each triple that can contribute: panel p covers rows [p*KP, (p+1)*KP) of B and the
// same columns of A, i.e. mask bits [p*W, (p+1)*W) with W = 64*KP/max(BS, 64) (mask bit b = row b
// for BS <= 64, rows 2b, 2b+1 for BS = 128). A panel where A's columns and B's rows share no bit
// adds exactly zero -- unless either block holds a NaN or Inf (masks' flags row), where 0 * Inf = NaN
// must be formed as numpy's dgemm does. Disjoint supports overall (not filtered by the symbolic
// phase) keep one panel.
// Also counts the k rows to execute (KP per panel; warp partials, one atomic per warp).
template <class Cfg>
__global__ void k_triple_panels(const uint2 *tri, int64_t nT, const uint64_t *a_rows, const uint64_t *a_cols,
                                const uint64_t *a_flags, const uint64_t *b_rows, const uint64_t *b_cols,
                                const uint64_t *b_flags, uint8_t *sm, unsigned long long *panels) {
  constexpr int W = 64 * Cfg::KP / (Cfg::BS > 64 ? Cfg::BS : 64);
  constexpr uint64_t kW = W >= 64 ? ~0ull : ((1ull << W) - 1ull);
  uint32_t cnt = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nT; t += (int64_t)gridDim.x * blockDim.x) {
    const uint2 ab = tri[t];
    // A's columns are the stored block's rows when it is used transposed (bit 31), B's rows its columns
    const uint32_t a = ab.x & ~kTransposed, b = ab.y & ~kTransposed;
    const uint64_t ac = (ab.x & kTransposed) ? a_rows[a] : a_cols[a];
    const uint64_t br = (ab.y & kTransposed) ? b_cols[b] : b_rows[b];
    const uint64_t ov = ac & br;
    uint32_t m = 0;
#pragma unroll
    for (int p = 0; p < Cfg::NP; ++p)
      if ((ov >> (p * W)) & kW) m |= 1u << p;
    if (!m) m = 1u;
    // a block holding NaN/Inf (flags row, bit 0): every panel runs, so 0 * Inf still yields NaN
    if ((a_flags[a] | b_flags[b]) & 1ull) m = (1u << Cfg::NP) - 1u;
    sm[t] = (uint8_t)m;
    cnt += __popc(m) * Cfg::KP;  // k rows executed
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(panels, (unsigned long long)cnt);
}

int sm_count_tma() { return device_sm_count(); }

// Claim-ahead policy (cur_next): QM_CLAIM_AHEAD=1|0 forces it; by default it is used when C blocks
// have fewer than 2 triples on average (units of one or two stages).
bool claim_ahead(int64_t nC, int64_t nT) {
  const char *e = getenv("QM_CLAIM_AHEAD");
  if (e && e[0] == '1') return true;
  if (e && e[0] == '0') return false;
  return nT < 2 * nC;
}

// Claim order of the C blocks. Quadtree-key order is the default: neighbouring block rows and
// columns of A/B stay in L2 when C blocks have several triples (banded, decay). Two alternatives,
// measured and kept as options (QM_UNIT_ORDER=k|lpt):
//  * k: by the k of each C block's first triple, so the blocks sharing A(., k) and B(k, .) run
//    together -- for about one triple per C block and no locality (random patterns, C3). On C3
//    (ncu, r45) DRAM reads fall 2.39 -> 0.65 GB per launch at the same kernel time (1.082 ms, DMMA
//    pipe 88%): the kernel is not DRAM-bound there, and the ordering sort costs ~20 us.
//  * lpt: longest k list first, against a tail of CTAs that claimed long lists last. On C1 (1,016
//    C blocks, 296 CTAs, L2-resident) the numeric phase went 0.138 -> 0.141 ms (r48).
// Processing order never changes a C block's own summation order: results are bitwise the same.
enum { kOrderKey = 0, kOrderK = 1, kOrderLpt = 2 };
int claim_order() {
  const char *e = getenv("QM_UNIT_ORDER");
  if (e && strcmp(e, "k") == 0) return kOrderK;
  if (e && strcmp(e, "lpt") == 0) return kOrderLpt;
  return kOrderKey;
}

size_t order_cub_bytes(int64_t nC) {
  size_t b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b, (uint32_t *)nullptr, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                  (uint32_t *)nullptr, (int64_t)std::max<int64_t>(nC, 1), 0, 32);
  return b;
}

// Workspace: the work counter (256 B), per-warp partial norms / nonzero flags of every tile, the
// claim-order arrays (4 x nC uint32 + radix-sort scratch), then the per-triple panel masks (nT bytes).
template <class Cfg>
size_t tma_ws_base(int64_t nC) {
  return align_up(256 + (size_t)nC * Cfg::NQ * Cfg::NCW * (sizeof(double) + sizeof(uint8_t)) + 256);
}
template <class Cfg>
size_t tma_ws_panels_offset(int64_t nC) {
  return tma_ws_base<Cfg>(nC) + align_up(4 * sizeof(uint32_t) * (size_t)nC) + align_up(order_cub_bytes(nC));
}
template <class Cfg>
size_t tma_ws_bytes(int64_t nC, int64_t nT) {
  return tma_ws_panels_offset<Cfg>(nC) + align_up((size_t)std::max<int64_t>(nT, 1));
}

// Fills the claim order (k of each C block's first triple, stable radix sort) into the workspace
// tail; returns the order array.
template <class Cfg>
int make_order(int kind, const uint2 *tri, const int64_t *tptr, const uint64_t *a_keys, int nbl, int lbits,
               int64_t nbg, int64_t nC, void *ws, uint32_t **order_out, cudaStream_t st) {
  char *base = (char *)ws + tma_ws_base<Cfg>(nC);
  uint32_t *key = (uint32_t *)base, *iota = key + nC, *skey = iota + nC, *order = skey + nC;
  void *cub_tmp = base + align_up(4 * sizeof(uint32_t) * (size_t)nC);
  size_t tb = order_cub_bytes(nC);
  const int grid = (int)std::min<int64_t>((nC + 255) / 256, (int64_t)sm_count_tma() * 8);
  k_order_key<<<std::max(grid, 1), 256, 0, st>>>(tri, tptr, a_keys, nC, nbl, lbits, kind == kOrderLpt, key,
                                                  iota);
  QM_LAUNCHED("k_order_key");
  int bits = 32;
  if (kind == kOrderK)
    for (bits = 1; bits < 32 && ((uint64_t)(nbg - 1) >> bits) != 0;) ++bits;
  QM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(cub_tmp, tb, key, skey, iota, order, nC, 0, bits, st));
  *order_out = order;
  return QM_OK;
}

template <class Cfg, int NPOOL, bool TR>
int launch_tma_pools(const double *const *A, const int64_t *nA, int na, const double *const *B,
                     const int64_t *nB, int nb, const uint2 *tri, const int64_t *tptr, int64_t nC, int64_t nT,
                     const NumericAux &oi, double *C, double *csq, uint8_t *cnz, int64_t *zc, void *ws,
                     size_t ws_bytes, cudaStream_t st) {
  if (na < 1 || nb < 1 || na > NPOOL || nb > NPOOL) {
    set_error("qm_numeric: %d / %d operand pools (at most %d)", na, nb, NPOOL);
    return QM_ERR_INVALID;
  }
  if (!ws || ws_bytes < tma_ws_bytes<Cfg>(nC, nT)) {
    set_error("qm_numeric: workspace %zu < required %zu", ws_bytes, tma_ws_bytes<Cfg>(nC, nT));
    return QM_ERR_WORKSPACE;
  }
  unsigned long long *counter = (unsigned long long *)ws;
  double *part_sq = (double *)((char *)ws + 256);
  uint8_t *part_nz = (uint8_t *)(part_sq + nC * Cfg::NQ * Cfg::NPART);
  QM_CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st));
  for (int i = 0; i < na; ++i)
    if (nA[i] * (int64_t)Cfg::BS >= ((int64_t)1 << 31)) {
      set_error("qm_numeric: pool of %lld blocks exceeds TMA's int32 row coordinate", (long long)nA[i]);
      return QM_ERR_UNSUPPORTED;
    }
  for (int i = 0; i < nb; ++i)
    if (nB[i] * (int64_t)Cfg::BS >= ((int64_t)1 << 31)) {
      set_error("qm_numeric: pool of %lld blocks exceeds TMA's int32 row coordinate", (long long)nB[i]);
      return QM_ERR_UNSUPPORTED;
    }
  TmaMaps<NPOOL, TR> maps;
  memset(&maps, 0, sizeof(maps));
  for (int i = 0; i < NPOOL; ++i) {  // unused slots repeat pool 0 (never indexed)
    int rc = make_map(&maps.a[i], A[i < na ? i : 0], nA[i < na ? i : 0], Cfg::BS, Cfg::TILE);
    if (rc != QM_OK) return rc;
    rc = make_map(&maps.b[i], B[i < nb ? i : 0], nB[i < nb ? i : 0], Cfg::BS, Cfg::KP);
    if (rc != QM_OK) return rc;
  }
  if constexpr (Cfg::EW) {
    int rc = make_map(&maps.c, C, nC, Cfg::BS, Cfg::TILE);
    if (rc != QM_OK) return rc;
  }
  if constexpr (TR) {
    int rc = make_map(&maps.at, A[0], nA[0], Cfg::BS, Cfg::KP);
    if (rc != QM_OK) return rc;
    rc = make_map(&maps.bt, B[0], nB[0], Cfg::BS, Cfg::TILE);
    if (rc != QM_OK) return rc;
  }
  static PerDeviceOnce once;
  int rc = once.run([]() -> int {
    QM_CUDA_TRY(cudaFuncSetAttribute(k_numeric_tma<Cfg, NPOOL, TR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)Cfg::SMEM));
    return (int)QM_OK;
  });
  if (rc != QM_OK) return rc;
  int per_sm = 0;
  static PerDeviceInt occupancy;  // cudaOccupancy* costs microseconds of host time per call
  rc = occupancy.get(&per_sm, [](int *x) -> int {
    QM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(x, k_numeric_tma<Cfg, NPOOL, TR>, Cfg::NTHR,
                                                              Cfg::SMEM));
    return (int)QM_OK;
  });
  if (rc != QM_OK) return rc;
  if (per_sm < 1) per_sm = 1;
  const int64_t nU = nC * Cfg::NQ;
  int64_t grid = (int64_t)sm_count_tma() * per_sm;
  if (grid > nU) grid = nU;
  const uint32_t *order = oi.order;  // the caller's claim order (staged multi-GPU products)
  // (not with transposed references: their triple indices name stored blocks, not view entries)
  if (!order && oi.a_keys && na == 1 && nb == 1 && !TR) {
    const int kind = claim_order();
    if (kind != kOrderKey) {
      uint32_t *o = nullptr;
      rc = make_order<Cfg>(kind, tri, tptr, oi.a_keys, oi.nbl, oi.lbits, oi.nbg, nC, ws, &o, st);
      if (rc != QM_OK) return rc;
      order = o;
    }
  }
  uint8_t *tri_sm = nullptr;
  int64_t panel_fill = (int64_t)Cfg::BS * nT;  // every k row of every triple
  // panel masks: single pools index the masks with the triples themselves; several pools need the
  // triples' indices in the masks' index space (mask_tri, e.g. global block indices)
  const bool one_pool = na == 1 && nb == 1;
  if (oi.masked() && (one_pool || oi.mask_tri) && Cfg::NP > 1 && nT > 0) {
    tri_sm = (uint8_t *)ws + tma_ws_panels_offset<Cfg>(nC);
    if (oi.panel_count) QM_CUDA_TRY(cudaMemsetAsync(oi.panel_count, 0, sizeof(int64_t), st));
    const int g = (int)std::min<int64_t>((nT + 255) / 256, (int64_t)sm_count_tma() * 16);
    const uint2 *mt = oi.mask_tri ? (const uint2 *)oi.mask_tri : tri;
    k_triple_panels<Cfg><<<g, 256, 0, st>>>(mt, nT, oi.a_rows, oi.a_cols, oi.a_flags, oi.b_rows, oi.b_cols,
                                            oi.b_flags, tri_sm, (unsigned long long *)oi.panel_count);
    QM_LAUNCHED("k_triple_panels");
    panel_fill = -1;  // counted by k_triple_panels
  }
  if (oi.halo) {
    // staged halo: the gather runs on a few SMs' TMA engines while this kernel computes the
    // local-only C blocks; its claims >= gate_units wait for the gather grid (griddepcontrol.wait)
    GatherArgs ga;
    memset(&ga, 0, sizeof(ga));
    for (int o = 0; o < 2; ++o) {
      ga.index[o] = oi.halo->index[o];
      ga.count[o] = oi.halo->count[o];
      ga.pool[o] = oi.halo->pool[o];
      for (int r = 0; r < QM_MAX_RANKS; ++r) ga.base[o][r] = oi.halo->peer_base[o][r];
      for (int r = 0; r <= QM_MAX_RANKS; ++r) ga.off[o][r] = oi.halo->offset[o][r];
    }
    ga.world = oi.halo->world;
    ga.block_bytes = (int64_t)Cfg::BS * Cfg::BS * (int64_t)sizeof(double);
    ga.min_ns = oi.halo->min_ns;
    const int64_t jobs = (ga.count[0] + ga.count[1]) * ((ga.block_bytes + kGatherChunk - 1) / kGatherChunk);
    const int gg = (int)std::max<int64_t>(1, std::min<int64_t>((jobs + kGatherLanes - 1) / kGatherLanes, kGatherCtas));
    static PerDeviceOnce gonce;
    rc = gonce.run([]() -> int {
      QM_CUDA_TRY(cudaFuncSetAttribute(k_halo_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, kGatherSmem));
      return (int)QM_OK;
    });
    if (rc != QM_OK) return rc;
    k_halo_gather<<<gg, 32, kGatherSmem, st>>>(ga);
    QM_LAUNCHED("k_halo_gather");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(Cfg::NTHR);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int64_t gate_units = std::max<int64_t>(0, std::min<int64_t>(oi.gate_units, nU));
    QM_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_numeric_tma<Cfg, NPOOL, TR>, maps, tri, tptr, nC, C, csq, cnz, zc,
                                   part_sq, part_nz, counter, order, (const uint8_t *)tri_sm, (uint64_t)0ull,
                                   claim_ahead(nC, nT), gate_units));
  } else {
    k_numeric_tma<Cfg, NPOOL, TR><<<(int)grid, Cfg::NTHR, Cfg::SMEM, st>>>(
        maps, tri, tptr, nC, C, csq, cnz, zc, part_sq, part_nz, counter, order, tri_sm, /*zmask=*/0ull,
        claim_ahead(nC, nT), nU);
  }
  QM_LAUNCHED("k_numeric_tma");
  {
    int64_t g = std::min<int64_t>((nC + 255) / 256, (int64_t)sm_count_tma() * 8);
    k_combine_tiles<<<(int)std::max<int64_t>(g, 1), 256, 0, st>>>(part_sq, part_nz, Cfg::NQ * Cfg::NPART,
                                                                   nC, csq, cnz, zc, oi.panel_count, panel_fill);
    QM_LAUNCHED("k_combine_tiles");
  }
  return QM_OK;
}

template <class Cfg>
int launch_tma(const double *const *A, const int64_t *nA, int na, const double *const *B,
               const int64_t *nB, int nb, const uint2 *tri, const int64_t *tptr, int64_t nC, int64_t nT,
               const NumericAux &oi, double *C, double *csq, uint8_t *cnz, int64_t *zc, void *ws, size_t ws_bytes,
               cudaStream_t st) {
  if (na == 1 && nb == 1) {
    if (oi.transpose_bits)
      return launch_tma_pools<Cfg, 1, true>(A, nA, na, B, nB, nb, tri, tptr, nC, nT, oi, C, csq, cnz, zc, ws,
                                            ws_bytes, st);
    return launch_tma_pools<Cfg, 1, false>(A, nA, na, B, nB, nb, tri, tptr, nC, nT, oi, C, csq, cnz, zc, ws,
                                           ws_bytes, st);
  }
  if (oi.transpose_bits) {
    set_error("qm_numeric: transposed block references need a single pool per operand");
    return QM_ERR_INVALID;
  }
  return launch_tma_pools<Cfg, kMaxPools, false>(A, nA, na, B, nB, nb, tri, tptr, nC, nT, oi, C, csq, cnz, zc,
                                                 ws, ws_bytes, st);
}

//                     BS TILE WM WN KP STAGES MINB
// bs 32: a triple is one 16 KB stage; 4 warps of 16x16 and 6 CTAs/SM (6 consumer warps per SMSP
// hide the per-stage overheads better than 2 warps of 32x16 in 4 CTAs: C5-bs32 263.6 -> 259.1 ms).
using Tma32 = TmaCfg<32, 32, 2, 2, 32, 2, 6>;
using Tma64 = TmaCfg<64, 64, 2, 2, 32, 3, 2>;
// Many triples per C block: 3 CTAs/SM with 2 stages (more resident warps hide the per-stage
// overheads; C2-131072 -0.7%, C4 -0.9%); about one triple per block (random patterns, C3): 2 CTAs
// with 3 stages (deeper prefetch of DRAM-resident operands; C3 -1.4% against the 3-CTA variant).
using Tma64m = TmaCfg<64, 64, 2, 2, 32, 2, 3>;
// The epilogue warp variant of Tma64 (3 stages, 2 CTAs/SM), opt-in with QM_EPILOGUE_WARP=1.
// Measured and not adopted (C3, r2): numeric 1.077 -> 1.234 ms. Both CTAs' epilogue warps land on
// the same SM sub-partition, whose FP64 pipe then also runs every tile's sum-of-squares DFMAs
// (4096 per tile), and the consumers' per-unit named barrier couples all four math warps to that
// slowest sub-partition; C2-16384 1.104 -> 1.126 ms, banded / decay products unchanged.
using Tma64e = TmaCfg<64, 64, 2, 2, 32, 3, 2, 1>;
using Tma64s = TmaCfg<64, 64, 2, 2, 32, 3, 2, 2>;  // QM_EPILOGUE_WARP=2: the TMA store only
int use_ew() {
  const char *e = getenv("QM_EPILOGUE_WARP");
  return e ? atoi(e) : 0;
}
constexpr int64_t kManyTriplesPerBlock = 2;

// Variant choice for bs 64/128 (nU work units = C blocks x tiles per block): the 3-CTA variant needs
// >= 2 triples per C block and enough units that its shorter per-CTA queue does not lengthen the
// tail (>= 24 units per resident CTA: C2-16384 with 18 stays on 2 CTAs, C2-32768 with 37 moves).
// QM_TMA_VARIANT=deep|wide forces one (A/B measurements).
constexpr int64_t kWideUnitsPerCta = 24;
bool use_wide(int64_t nU, int64_t nC, int64_t nT) {
  const char *e = getenv("QM_TMA_VARIANT");
  if (e && strcmp(e, "deep") == 0) return false;
  if (e && strcmp(e, "wide") == 0) return true;
  return nT >= kManyTriplesPerBlock * nC && nU >= kWideUnitsPerCta * 3 * (int64_t)device_sm_count();
}

// Masked products (operands with partial block supports): 16-deep k panels, so the panel skip of
// k_triple_panels works at half the granularity; 4 stages of 16 KB, 3 CTAs/SM.
using Tma64k16 = TmaCfg<64, 64, 2, 2, 16, 4, 3>;
using Tma32k16 = TmaCfg<32, 32, 2, 2, 16, 4, 6>;  // same for bs 32: 4 stages of 8 KB, 6 CTAs/SM
bool use_k16(const NumericAux &oi) {
  const char *e = getenv("QM_PANEL16");
  return oi.masked() && !(e && strcmp(e, "0") == 0);
}

using Tma128 = TmaCfg<128, 64, 2, 2, 32, 3, 2>;
using Tma128m = TmaCfg<128, 64, 2, 2, 32, 2, 3>;

}  // namespace

size_t numeric_tma_ws_bytes(int bs, int64_t nC, int64_t nT) {
  switch (bs) {
    case 32: return std::max(tma_ws_bytes<Tma32>(nC, nT), tma_ws_bytes<Tma32k16>(nC, nT));
    case 64:
      return std::max(std::max(tma_ws_bytes<Tma64>(nC, nT), tma_ws_bytes<Tma64m>(nC, nT)),
                      std::max(tma_ws_bytes<Tma64k16>(nC, nT),
                               std::max(tma_ws_bytes<Tma64e>(nC, nT), tma_ws_bytes<Tma64s>(nC, nT))));
    case 128: return std::max(tma_ws_bytes<Tma128>(nC, nT), tma_ws_bytes<Tma128m>(nC, nT));
    default: return 0;
  }
}

// Returns QM_ERR_UNSUPPORTED when no TMA variant exists for bs. `na` / `nb` operand pools (1 =
// local; > 1 = every rank's pool, triple indices packed as owner << 28 | local).
int launch_numeric_tma(int bs, const double *const *A, const int64_t *nA, int na, const double *const *B,
                       const int64_t *nB, int nb, const uint32_t *tri, const int64_t *tptr, int64_t nC,
                       int64_t nT, const NumericAux &oi, double *C, double *csq, uint8_t *cnz, int64_t *zc,
                       void *ws, size_t ws_bytes, cudaStream_t st) {
  const uint2 *t2 = (const uint2 *)tri;
  switch (bs) {
    case 32:
      if (use_k16(oi))
        return launch_tma<Tma32k16>(A, nA, na, B, nB, nb, t2, tptr, nC, nT, oi, C, csq, cnz, zc, ws, ws_bytes, st);
      return launch_tma<Tma32>(A, nA, na, B, nB, nb, t2, tptr, nC, nT, oi, C, csq, cnz, zc, ws, ws_bytes, st);
    case 64:
      if (use_k16(oi))
        return launch_tma<Tma64k16>(A, nA, na, B, nB, nb, t2, tptr, nC, nT, oi, C, csq, cnz, zc, ws, ws_bytes, st);
      if (use_wide(nC, nC, nT))
        return launch_tma<Tma64m>(A, nA, na, B, nB, nb, t2, tptr, nC, nT, oi, C, csq, cnz, zc, ws, ws_bytes, st);
      if (use_ew() == 1)
        return launch_tma<Tma64e>(A, nA, na, B, nB, nb, t2, tptr, nC, nT, oi, C, csq, cnz, zc, ws, ws_bytes, st);
      if (use_ew() == 2)
        return launch_tma<Tma64s>(A, nA, na, B, nB, nb, t2, tptr, nC, nT, oi, C, csq, cnz, zc, ws, ws_bytes, st);
      return launch_tma<Tma64>(A, nA, na, B, nB, nb, t2, tptr, nC, nT, oi, C, csq, cnz, zc, ws, ws_bytes, st);
    case 128:
      if (use_wide(nC * Tma128::NQ, nC, nT))
        return launch_tma<Tma128m>(A, nA, na, B, nB, nb, t2, tptr, nC, nT, oi, C, csq, cnz, zc, ws, ws_bytes, st);
      return launch_tma<Tma128>(A, nA, na, B, nB, nb, t2, tptr, nC, nT, oi, C, csq, cnz, zc, ws, ws_bytes, st);
    default: return QM_ERR_UNSUPPORTED;
  }
}

}  // namespace qm

// Numeric phase: grouped FP64 block products accumulated per C block.
//
// Replaces BlockSparseLeaf.multiply (leaves/block_sparse.py:112-132: `prod = a @ b`,
// `acc = acc + prod`) and the cross-level sums of _add_body / BlockSparseLeaf.add
// (ops.py:147-159, block_sparse.py:134-152). Each C block is owned by one CTA for its whole k list,
// accumulated in registers, with no atomics and a fixed summation order; the epilogue fuses the
// exact-zero test and the Frobenius norm of _set_block (block_sparse.py:37-41).
//
// Tensor-core path (block sizes 16/32/64/128): sm_100a has no FP64 tcgen05 kind, so FP64 tensor
// math is the warp-level mma.sync.m8n8k4.f64 (SASS DMMA). Operands are staged into padded shared
// memory (row stride = cols + 4 doubles, which makes both fragment patterns bank-conflict free) by
// a multi-stage cp.async pipeline that streams k-panels continuously across triples and C blocks.
// CTAs are persistent and walk C blocks in quadtree-key order (grid-stride), so concurrently
// running CTAs touch neighbouring block rows/columns of A and B and reuse them from L2.
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include "qm_common.cuh"

namespace qm {
namespace {

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// D = A(8x4, row) * B(4x8, col) + D, fp64. Fragments: a = A[lane>>2][lane&3],
// b = B[lane&3][lane>>2], d = D[lane>>2][2*(lane&3) + {0,1}].
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int BS_, int WARPS_M_, int WARPS_N_, int KP_, int STAGES_, int MINB_>
struct DmmaCfg {
  static constexpr int BS = BS_, WARPS_M = WARPS_M_, WARPS_N = WARPS_N_, KP = KP_, STAGES = STAGES_;
  static constexpr int MINB = MINB_;
  static constexpr int NTHR = 32 * WARPS_M * WARPS_N;
  static constexpr int TM = BS / WARPS_M, TN = BS / WARPS_N;  // warp tile
  static constexpr int MT = TM / 8, NT = TN / 8;               // mma tiles per warp
  static constexpr int NP = BS / KP;                           // k panels per triple
  static constexpr int LDA = KP + 4, LDB = BS + 4;             // padded smem row strides (doubles)
  static constexpr int A_ELEMS = BS * LDA, B_ELEMS = KP * LDB;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_ELEMS * sizeof(double) + 64 * sizeof(double);
  static_assert(BS % (8 * WARPS_M) == 0 && BS % (8 * WARPS_N) == 0, "warp tiling");
  static_assert(BS % KP == 0 && KP % 4 == 0, "panel");
};

// Stage cursor: C block `item`, triple t of [t, tend), k panel p.
struct Cursor {
  int64_t item, t, tend;
  int p;
};

template <class Cfg>
__device__ __forceinline__ void cursor_start(Cursor &c, int64_t item, int64_t nC, const int64_t *tptr) {
  c.item = item;
  c.p = 0;
  if (item < nC) {
    c.t = tptr[item];
    c.tend = tptr[item + 1];
  } else {
    c.t = c.tend = 0;
  }
}

template <class Cfg>
__device__ __forceinline__ void cursor_next(Cursor &c, int64_t nC, const int64_t *tptr) {
  if (++c.p == Cfg::NP) {
    c.p = 0;
    if (++c.t == c.tend) cursor_start<Cfg>(c, c.item + gridDim.x, nC, tptr);
  }
}

template <class Cfg>
__device__ __forceinline__ void issue_stage(double *stage, const double *__restrict__ A,
                                            const double *__restrict__ B, const uint2 *__restrict__ tri,
                                            const Cursor &c) {
  constexpr int BS = Cfg::BS, KP = Cfg::KP;
  const uint2 ab = tri[c.t];
  const double *asrc = A + (size_t)ab.x * (BS * BS) + c.p * KP;
  const double *bsrc = B + (size_t)ab.y * (BS * BS) + (size_t)c.p * KP * BS;
  double *sA = stage;
  double *sB = stage + Cfg::A_ELEMS;
  constexpr int ACH = KP / 2;  // 16-byte chunks per A panel row
  for (int q = threadIdx.x; q < BS * ACH; q += Cfg::NTHR) {
    int r = q / ACH, cc = q % ACH;
    cp_async16(sA + r * Cfg::LDA + 2 * cc, asrc + (size_t)r * BS + 2 * cc);
  }
  constexpr int BCH = BS / 2;  // 16-byte chunks per B panel row
  for (int q = threadIdx.x; q < KP * BCH; q += Cfg::NTHR) {
    int r = q / BCH, cc = q % BCH;
    cp_async16(sB + r * Cfg::LDB + 2 * cc, bsrc + (size_t)r * BS + 2 * cc);
  }
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::NTHR, Cfg::MINB)
    k_numeric_dmma(const double *__restrict__ A, const double *__restrict__ B,
                   const uint2 *__restrict__ tri, const int64_t *__restrict__ tptr, int64_t nC,
                   double *__restrict__ C, double *__restrict__ csq, uint8_t *__restrict__ cnz,
                   int64_t *__restrict__ zero_count) {
  extern __shared__ __align__(16) double smem[];
  double *red = smem + (size_t)Cfg::STAGES * Cfg::STAGE_ELEMS;  // 64 doubles for the epilogue
  constexpr int BS = Cfg::BS, MT = Cfg::MT, NT = Cfg::NT, STAGES = Cfg::STAGES;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int wm0 = (warp / Cfg::WARPS_N) * Cfg::TM;
  const int wn0 = (warp % Cfg::WARPS_N) * Cfg::TN;

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  Cursor L, Cc;
  cursor_start<Cfg>(L, blockIdx.x, nC, tptr);
  Cc = L;

#pragma unroll 1
  for (int s = 0; s < STAGES - 1; ++s) {
    if (L.item < nC) {
      issue_stage<Cfg>(smem + (size_t)s * Cfg::STAGE_ELEMS, A, B, tri, L);
      cursor_next<Cfg>(L, nC, tptr);
    }
    cp_async_commit();
  }
  int cs = 0, ls = STAGES - 1;

#pragma unroll 1
  while (Cc.item < nC) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (L.item < nC) {
      issue_stage<Cfg>(smem + (size_t)ls * Cfg::STAGE_ELEMS, A, B, tri, L);
      cursor_next<Cfg>(L, nC, tptr);
    }
    cp_async_commit();
    ls = (ls + 1 == STAGES) ? 0 : ls + 1;

    const double *sA = smem + (size_t)cs * Cfg::STAGE_ELEMS;
    const double *sB = sA + Cfg::A_ELEMS;
    const double *pa = sA + (wm0 + g) * Cfg::LDA + tq;
    const double *pb = sB + tq * Cfg::LDB + wn0 + g;
#pragma unroll
    for (int ks = 0; ks < Cfg::KP / 4; ++ks) {
      double af[MT], bf[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) af[i] = pa[i * 8 * Cfg::LDA + ks * 4];
#pragma unroll
      for (int j = 0; j < NT; ++j) bf[j] = pb[ks * 4 * Cfg::LDB + j * 8];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    cs = (cs + 1 == STAGES) ? 0 : cs + 1;

    if (Cc.p == Cfg::NP - 1 && Cc.t + 1 == Cc.tend) {
      // Epilogue: store the C block, fused sum of squares + nonzero test (fixed order).
      const int64_t m = Cc.item;
      double *cb = C + (size_t)m * (BS * BS);
      double ss = 0.0;
      bool nz = false;
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const double v0 = acc[i][j][0], v1 = acc[i][j][1];
          *reinterpret_cast<double2 *>(cb + (size_t)(wm0 + i * 8 + g) * BS + wn0 + j * 8 + 2 * tq) =
              make_double2(v0, v1);
          ss = fma(v0, v0, ss);
          ss = fma(v1, v1, ss);
          nz |= (v0 != 0.0) | (v1 != 0.0);
          acc[i][j][0] = acc[i][j][1] = 0.0;
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      const bool wnz = __any_sync(0xffffffffu, nz);
      if (lane == 0) {
        red[warp] = ss;
        red[32 + warp] = wnz ? 1.0 : 0.0;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double tot = 0.0, anynz = 0.0;
        for (int w = 0; w < Cfg::NTHR / 32; ++w) {
          tot += red[w];
          anynz += red[32 + w];
        }
        csq[m] = tot;
        cnz[m] = anynz != 0.0;
        if (anynz == 0.0 && zero_count) atomicAdd((unsigned long long *)zero_count, 1ull);
      }
    }
    cursor_next<Cfg>(Cc, nC, tptr);
  }
  cp_async_wait<0>();
}

// Generic FP64 SIMT path for block sizes without a tensor-core variant: one CTA per
// (C block, 32x32 sub-tile), 4 outputs per thread.
__global__ void __launch_bounds__(256) k_numeric_generic(const double *__restrict__ A,
                                                         const double *__restrict__ B,
                                                         const uint2 *__restrict__ tri,
                                                         const int64_t *__restrict__ tptr, int64_t nC,
                                                         int bs, double *__restrict__ C) {
  __shared__ double As[32][33];
  __shared__ double Bs[32][33];
  const int nsub = (bs + 31) / 32;
  const int64_t nwork = nC * nsub * nsub;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int64_t m = w / (nsub * nsub);
    const int sub = (int)(w % (nsub * nsub));
    const int r0 = (sub / nsub) * 32, c0 = (sub % nsub) * 32;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t t = tptr[m]; t < tptr[m + 1]; ++t) {
      const uint2 ab = tri[t];
      const double *a = A + (size_t)ab.x * bs * bs;
      const double *b = B + (size_t)ab.y * bs * bs;
      for (int kc = 0; kc < bs; kc += 32) {
        for (int q = 0; q < 4; ++q) {
          const int r = ty + 8 * q;
          As[r][tx] = (r0 + r < bs && kc + tx < bs) ? a[(size_t)(r0 + r) * bs + kc + tx] : 0.0;
          Bs[r][tx] = (kc + r < bs && c0 + tx < bs) ? b[(size_t)(kc + r) * bs + c0 + tx] : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < 32; ++kk) {
          const double bv = Bs[kk][tx];
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[q] = fma(As[ty + 8 * q][kk], bv, acc[q]);
        }
        __syncthreads();
      }
    }
    double *cb = C + (size_t)m * bs * bs;
    for (int q = 0; q < 4; ++q) {
      const int r = r0 + ty + 8 * q, c = c0 + tx;
      if (r < bs && c < bs) cb[(size_t)r * bs + c] = acc[q];
    }
  }
}

// Per-block metadata in one read of the blocks (the reference stores a leaf's block norms with
// it, block_sparse.py:41; the support masks and non-finite flag are the same kind of input
// metadata): squared Frobenius norm, any-nonzero flag (_set_block's np.any, block_sparse.py:37-41),
// and optionally the support masks -- bit b of rmask / cmask is set when a row / column r with
// b = r (bs <= 64) or b = r*64/bs (bs > 64) holds a nonzero -- plus flags bit 0 = the block holds a
// NaN or Inf (its masks are then full: 0 * Inf is NaN, so none of its products is provably zero,
// and the numeric kernel must not skip any of its k panels). not_full[0] / [1] (OR-accumulated,
// one atomic per CTA) become nonzero when some block's row / column mask is not full.
// One CTA of 256 threads per block (grid-stride): thread t sums elements t, t+256, ... in an fma
// chain, warp xor tree, warps in order -- the order every fused statistics pass of the library
// (k_axpby, the numeric epilogues' tile partials aside) reproduces bit for bit.
template <int BS>
__global__ void __launch_bounds__(256) k_block_meta(const double *__restrict__ blocks, int64_t n, int bs_rt,
                                                    double *sumsq, uint8_t *nonzero, int64_t *zero_count,
                                                    uint64_t *rmask, uint64_t *cmask, uint64_t *flags,
                                                    unsigned long long *not_full) {
  __shared__ double red[8];
  __shared__ int rnz[8];
  __shared__ uint64_t rrm[8], rcm[8];
  __shared__ int rbad[8];
  const int bs = BS ? BS : bs_rt;
  const int64_t elems = (int64_t)bs * bs;
  const bool want_masks = rmask != nullptr;
  const uint64_t full = bs >= 64 ? ~0ull : ((1ull << bs) - 1ull);
  unsigned long long nf_rows = 0, nf_cols = 0;  // this CTA saw a block with a partial row / column mask
  for (int64_t m = blockIdx.x; m < n; m += gridDim.x) {
    const double *b = blocks + (size_t)m * elems;
    double ss = 0.0;
    bool nz = false, bad = false;
    uint64_t rb = 0, cb = 0;
    if (BS) {
#pragma unroll
      for (int j = 0; j < (BS * BS + 255) / 256; ++j) {
        const int e = threadIdx.x + 256 * j;
        if (BS * BS % 256 == 0 || e < BS * BS) {
          const double v = b[e];
          ss = fma(v, v, ss);
          nz |= v != 0.0;
          if (want_masks) {
            const int r = e / BS, c = e % BS;
            const uint64_t on = v != 0.0 ? 1ull : 0ull;
            rb |= on << (BS <= 64 ? r : r * 64 / BS);
            cb |= on << (BS <= 64 ? c : c * 64 / BS);
            bad |= !isfinite(v);
          }
        }
      }
    } else {
      for (int64_t e = threadIdx.x; e < elems; e += blockDim.x) {
        const double v = b[e];
        ss = fma(v, v, ss);
        nz |= v != 0.0;
        if (want_masks && v != 0.0) {
          const int r = (int)(e / bs), c = (int)(e % bs);
          rb |= 1ull << (bs <= 64 ? r : (r * 64) / bs);
          cb |= 1ull << (bs <= 64 ? c : (c * 64) / bs);
        }
        bad |= !isfinite(v);
      }
    }
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const bool wnz = __any_sync(0xffffffffu, nz);
    const int w = threadIdx.x >> 5;
    if (want_masks) {
      const uint32_t rl = __reduce_or_sync(0xffffffffu, (uint32_t)rb), rh = __reduce_or_sync(0xffffffffu, (uint32_t)(rb >> 32));
      const uint32_t cl = __reduce_or_sync(0xffffffffu, (uint32_t)cb), ch = __reduce_or_sync(0xffffffffu, (uint32_t)(cb >> 32));
      const bool wbad = __any_sync(0xffffffffu, bad);
      if ((threadIdx.x & 31) == 0) {
        rrm[w] = (uint64_t)rh << 32 | rl;
        rcm[w] = (uint64_t)ch << 32 | cl;
        rbad[w] = wbad;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      red[w] = ss;
      rnz[w] = wnz;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      int any = 0, nonfinite = 0;
      uint64_t r = 0, c = 0;
      for (int x = 0; x < (int)(blockDim.x >> 5); ++x) {
        tot += red[x];
        any |= rnz[x];
        if (want_masks) {
          r |= rrm[x];
          c |= rcm[x];
          nonfinite |= rbad[x];
        }
      }
      if (sumsq) sumsq[m] = tot;
      if (nonzero) nonzero[m] = (uint8_t)any;
      if (!any && zero_count) atomicAdd((unsigned long long *)zero_count, 1ull);
      if (want_masks) {
        if (nonfinite) r = c = full;
        rmask[m] = r;
        cmask[m] = c;
        if (flags) flags[m] = nonfinite ? 1ull : 0ull;
        nf_rows |= r != full;
        nf_cols |= c != full;
      }
    }
    __syncthreads();
  }
  if (not_full && threadIdx.x == 0) {
    if (nf_rows) atomicOr(&not_full[0], 1ull);
    if (nf_cols) atomicOr(&not_full[1], 1ull);
  }
}




int sm_count() { return device_sm_count(); }

template <class Cfg>
int launch_dmma(const double *A, const double *B, const uint2 *tri, const int64_t *tptr, int64_t nC,
                double *C, double *csq, uint8_t *cnz, int64_t *zc, cudaStream_t st) {
  static PerDeviceOnce once;
  int rc = once.run([]() -> int {
    QM_CUDA_TRY(cudaFuncSetAttribute(k_numeric_dmma<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)Cfg::SMEM));
    return (int)QM_OK;
  });
  if (rc != QM_OK) return rc;
  int per_sm = 0;
  QM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_numeric_dmma<Cfg>, Cfg::NTHR,
                                                            Cfg::SMEM));
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)sm_count() * per_sm;
  if (grid > nC) grid = nC;
  k_numeric_dmma<Cfg><<<(int)grid, Cfg::NTHR, Cfg::SMEM, st>>>(A, B, tri, tptr, nC, C, csq, cnz, zc);
  QM_LAUNCHED("k_numeric_dmma");
  return QM_OK;
}

//                       BS  WM WN  KP  STAGES MINB
using Cfg16 = DmmaCfg<16, 1, 2, 16, 4, 8>;
using Cfg32 = DmmaCfg<32, 2, 2, 32, 4, 3>;
using Cfg64 = DmmaCfg<64, 2, 2, 32, 3, 2>;
using Cfg128 = DmmaCfg<128, 2, 4, 16, 4, 1>;

}  // namespace

int launch_block_meta(int bs, int64_t n, const double *blocks, double *sumsq, uint8_t *nonzero,
                      int64_t *zero_count, uint64_t *rmask, uint64_t *cmask, uint64_t *flags,
                      int64_t *not_full, cudaStream_t st) {
  if (n <= 0) return QM_OK;
  // 8 CTAs of 256 threads per SM, several waves' worth of blocks in flight (each thread has all of
  // its bs*bs/256 loads of a block outstanding at once)
  const int64_t grid = std::min<int64_t>(n, (int64_t)sm_count() * 16);
  unsigned long long *nf = (unsigned long long *)not_full;
  switch (bs) {
#define QM_META_CASE(B)                                                                                   \
  case B:                                                                                                 \
    k_block_meta<B><<<(int)grid, 256, 0, st>>>(blocks, n, bs, sumsq, nonzero, zero_count, rmask, cmask, flags, nf); \
    break;
    QM_META_CASE(16)
    QM_META_CASE(32)
    QM_META_CASE(64)
    QM_META_CASE(128)
#undef QM_META_CASE
    default:
      k_block_meta<0><<<(int)grid, 256, 0, st>>>(blocks, n, bs, sumsq, nonzero, zero_count, rmask, cmask, flags, nf);
  }
  QM_LAUNCHED("k_block_meta");
  return QM_OK;
}

int launch_block_stats(int bs, int64_t n, const double *blocks, double *sumsq, uint8_t *nonzero,
                       int64_t *zero_count, cudaStream_t st) {
  return launch_block_meta(bs, n, blocks, sumsq, nonzero, zero_count, nullptr, nullptr, nullptr, nullptr, st);
}

int numeric_sm_count() { return sm_count(); }

int launch_numeric_tma(int bs, const double *const *A, const int64_t *nA, int na, const double *const *B,
                       const int64_t *nB, int nb, const uint32_t *tri, const int64_t *tptr, int64_t nC,
                       int64_t nT, const NumericAux &oi, double *C, double *csq, uint8_t *cnz, int64_t *zc,
                       void *ws, size_t ws_bytes, cudaStream_t st);
size_t numeric_tma_ws_bytes(int bs, int64_t nC, int64_t nT);
size_t numeric_group16_ws_bytes(int64_t nC, int64_t nT);
int launch_numeric_group16(const Geometry &g, const double *A, int64_t nA, const double *B, int64_t nB,
                           const uint64_t *a_keys, const uint32_t *tri, const int64_t *c_tptr,
                           const uint64_t *c_keys, int64_t nC, int64_t nT, double *C, double *csq,
                           uint8_t *cnz, int64_t *zc, void *ws, size_t ws_bytes, cudaStream_t st);

int launch_numeric_quad32(const Geometry &g, const double *A, int64_t nA, const double *B, int64_t nB,
                          const uint64_t *a_keys, const uint32_t *tri, const int64_t *c_tptr,
                          const uint64_t *c_keys, int64_t nC, int64_t nT, double *C, double *csq, uint8_t *cnz,
                          int64_t *zc, void *ws, size_t ws_bytes, cudaStream_t st);

// Numeric kernel selection: QM_NUMERIC=cpasync forces the v1 cp.async kernel (A/B comparisons).
static int numeric_impl() {
  const char *e = getenv("QM_NUMERIC");
  return (e && strcmp(e, "cpasync") == 0) ? 1 : 2;
}

}  // namespace qm

using namespace qm;

namespace qm {
bool quad32_selected(const Geometry &g, int64_t nC, int64_t nT);
bool group16_selected(const Geometry &g, int64_t nC, int64_t nT);
}  // namespace qm

extern "C" const char *qm_numeric_kernel(const qm_layout *layout, int64_t nC, int64_t nT, int32_t masked,
                                         int32_t flags) {
  Geometry g;
  if (make_geometry(layout, &g) != QM_OK) return "";
  const bool tbits = (flags & QM_NUMERIC_TRANSPOSED_REFS) != 0;
  if (numeric_impl() == 2) {
    if (g.bs == 16) return group16_selected(g, nC, nT) ? "k_numeric_group16" : "k_numeric_dmma";
    if (g.bs == 32 && !masked && !tbits && quad32_selected(g, nC, nT)) return "k_numeric_quad32";
    if (g.bs == 32 || g.bs == 64 || g.bs == 128) return "k_numeric_tma";
  }
  if (g.bs == 16 || g.bs == 32 || g.bs == 64 || g.bs == 128) return "k_numeric_dmma";
  return "k_numeric_generic";
}

extern "C" int qm_numeric_path(int32_t bs) {
  if ((bs == 16 || bs == 32 || bs == 64 || bs == 128) && numeric_impl() == 2) return 2;
  return (bs == 16 || bs == 32 || bs == 64 || bs == 128) ? 1 : 0;
}

extern "C" size_t qm_numeric_workspace_bytes(int32_t block_size, int64_t nC, int64_t nT) {
  if (numeric_impl() != 2) return 0;
  return block_size == 16 ? numeric_group16_ws_bytes(nC, nT) : numeric_tma_ws_bytes(block_size, nC, nT);
}

extern "C" int qm_numeric_masked(const qm_layout *layout, const uint64_t *a_keys, const double *a_blocks,
                                 const uint64_t *a_masks, int64_t nA, const double *b_blocks,
                                 const uint64_t *b_masks, int64_t nB, int32_t flags, const uint32_t *tri,
                                 const int64_t *c_tptr,
                                 const uint64_t *c_keys, int64_t nC, int64_t nT, double *c_blocks, double *c_sumsq,
                                 uint8_t *c_nonzero, int64_t *zero_count, int64_t *panel_count, void *ws,
                                 size_t ws_bytes, void *stream) {
  Geometry g;
  int rc = make_geometry(layout, &g);
  if (rc != QM_OK) return rc;
  if (nC < 0) {
    set_error("qm_numeric: negative nC");
    return QM_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (zero_count) QM_CUDA_TRY(cudaMemsetAsync(zero_count, 0, sizeof(int64_t), st));
  if (panel_count) QM_CUDA_TRY(cudaMemsetAsync(panel_count, nC == 0 ? 0 : 0xff, sizeof(int64_t), st));  // -1: not counted
  if (nC == 0) return QM_OK;
  const uint2 *t2 = (const uint2 *)tri;
  const bool tbits = (flags & QM_NUMERIC_TRANSPOSED_REFS) != 0;
  if (tbits && !(numeric_impl() == 2 && (g.bs == 32 || g.bs == 64 || g.bs == 128))) {
    set_error("qm_numeric: transposed block references need the bs 32/64/128 TMA kernel");
    return QM_ERR_UNSUPPORTED;
  }
  if (numeric_impl() == 2 && g.bs == 16) {
    rc = launch_numeric_group16(g, a_blocks, nA, b_blocks, nB, a_keys, tri, c_tptr, c_keys, nC, nT, c_blocks,
                                c_sumsq, c_nonzero, zero_count, ws, ws_bytes, st);
    if (rc != QM_ERR_UNSUPPORTED) return rc;
  }
  if (numeric_impl() == 2 && g.bs == 32 && !tbits && !(a_masks && b_masks)) {  // quads of C blocks
    rc = launch_numeric_quad32(g, a_blocks, nA, b_blocks, nB, a_keys, tri, c_tptr, c_keys, nC, nT, c_blocks,
                               c_sumsq, c_nonzero, zero_count, ws, ws_bytes, st);
    if (rc != QM_ERR_UNSUPPORTED) return rc;
  }
  if (numeric_impl() == 2) {
    NumericAux oi;
    oi.a_keys = a_keys;
    oi.nbl = g.nbl;
    oi.lbits = g.lbits;
    oi.nbg = g.nbg;
    if (a_masks && b_masks) {
      oi.a_rows = a_masks, oi.a_cols = a_masks + nA, oi.a_flags = a_masks + 2 * nA;
      oi.b_rows = b_masks, oi.b_cols = b_masks + nB, oi.b_flags = b_masks + 2 * nB;
    }
    oi.transpose_bits = tbits;
    oi.panel_count = panel_count;
    rc = launch_numeric_tma(g.bs, &a_blocks, &nA, 1, &b_blocks, &nB, 1, tri, c_tptr, nC, nT, oi, c_blocks,
                            c_sumsq, c_nonzero, zero_count, ws, ws_bytes, st);
    if (rc != QM_ERR_UNSUPPORTED) return rc;
  }
  switch (g.bs) {
    case 16: return launch_dmma<Cfg16>(a_blocks, b_blocks, t2, c_tptr, nC, c_blocks, c_sumsq, c_nonzero, zero_count, st);
    case 32: return launch_dmma<Cfg32>(a_blocks, b_blocks, t2, c_tptr, nC, c_blocks, c_sumsq, c_nonzero, zero_count, st);
    case 64: return launch_dmma<Cfg64>(a_blocks, b_blocks, t2, c_tptr, nC, c_blocks, c_sumsq, c_nonzero, zero_count, st);
    case 128: return launch_dmma<Cfg128>(a_blocks, b_blocks, t2, c_tptr, nC, c_blocks, c_sumsq, c_nonzero, zero_count, st);
    default: break;
  }
  const int nsub = (g.bs + 31) / 32;
  int64_t work = nC * nsub * nsub;
  int64_t grid = std::min<int64_t>(work, (int64_t)sm_count() * 8);
  k_numeric_generic<<<(int)grid, 256, 0, st>>>(a_blocks, b_blocks, t2, c_tptr, nC, g.bs, c_blocks);
  QM_LAUNCHED("k_numeric_generic");
  return launch_block_stats(g.bs, nC, c_blocks, c_sumsq, c_nonzero, zero_count, st);
}

extern "C" int qm_numeric(const qm_layout *layout, const uint64_t *a_keys, const double *a_blocks, int64_t nA,
                          const double *b_blocks, int64_t nB, const uint32_t *tri,
                          const int64_t *c_tptr, const uint64_t *c_keys, int64_t nC, int64_t nT, double *c_blocks,
                          double *c_sumsq, uint8_t *c_nonzero, int64_t *zero_count, void *ws,
                          size_t ws_bytes, void *stream) {
  return qm_numeric_masked(layout, a_keys, a_blocks, nullptr, nA, b_blocks, nullptr, nB, 0, tri, c_tptr, c_keys, nC,
                           nT, c_blocks, c_sumsq, c_nonzero, zero_count, nullptr, ws, ws_bytes, stream);
}

extern "C" int qm_block_stats(int32_t block_size, int64_t n, const double *blocks, double *sumsq,
                              uint8_t *nonzero, void *stream) {
  if (block_size < 1 || n < 0) {
    set_error("qm_block_stats: bad arguments");
    return QM_ERR_INVALID;
  }
  return launch_block_stats(block_size, n, blocks, sumsq, nonzero, nullptr, (cudaStream_t)stream);
}

extern "C" int qm_block_masks(int32_t block_size, int64_t n, const double *blocks, uint64_t *row_mask,
                              uint64_t *col_mask, void *stream) {
  if (block_size < 1 || n < 0 || (n > 0 && (!blocks || !row_mask || !col_mask))) {
    set_error("qm_block_masks: bad arguments");
    return QM_ERR_INVALID;
  }
  return launch_block_meta(block_size, n, blocks, nullptr, nullptr, nullptr, row_mask, col_mask, nullptr, nullptr,
                           (cudaStream_t)stream);
}

extern "C" int qm_block_meta(int32_t block_size, int64_t n, const double *blocks, double *sumsq, uint8_t *nonzero,
                             int64_t *zero_count, uint64_t *masks, int64_t *not_full, void *stream) {
  if (block_size < 1 || n < 0 || (n > 0 && !blocks)) {
    set_error("qm_block_meta: bad arguments");
    return QM_ERR_INVALID;
  }
  return launch_block_meta(block_size, n, blocks, sumsq, nonzero, zero_count, masks, masks ? masks + n : nullptr,
                           masks ? masks + 2 * n : nullptr, not_full, (cudaStream_t)stream);
}

extern "C" int qm_numeric_pools(const qm_layout *layout, const double *const *a_pools, const int64_t *a_counts,
                                int32_t n_a_pools, const double *const *b_pools, const int64_t *b_counts,
                                int32_t n_b_pools, const uint32_t *tri, const int64_t *c_tptr, int64_t nC,
                                int64_t nT, double *c_blocks, double *c_sumsq, uint8_t *c_nonzero,
                                int64_t *zero_count, void *ws, size_t ws_bytes, void *stream) {
  Geometry g;
  int rc = make_geometry(layout, &g);
  if (rc != QM_OK) return rc;
  if (zero_count) QM_CUDA_TRY(cudaMemsetAsync(zero_count, 0, sizeof(int64_t), (cudaStream_t)stream));
  if (nC <= 0) return nC < 0 ? QM_ERR_INVALID : QM_OK;
  if (!a_pools || !b_pools || !a_counts || !b_counts) {
    set_error("qm_numeric_pools: NULL pool arrays");
    return QM_ERR_INVALID;
  }
  return launch_numeric_tma(g.bs, a_pools, a_counts, n_a_pools, b_pools, b_counts, n_b_pools, tri, c_tptr,
                            nC, nT, NumericAux(), c_blocks, c_sumsq, c_nonzero, zero_count, ws, ws_bytes,
                            (cudaStream_t)stream);
}

extern "C" int qm_numeric_pools_ex(const qm_layout *layout, const double *const *a_pools, const int64_t *a_counts,
                                   int32_t n_a_pools, const double *const *b_pools, const int64_t *b_counts,
                                   int32_t n_b_pools, const uint32_t *tri, const uint32_t *mask_tri,
                                   const uint64_t *a_cmask, const uint64_t *a_flags, const uint64_t *b_rmask,
                                   const uint64_t *b_flags, const uint32_t *order, const qm_halo *halo,
                                   int64_t gate_units, const int64_t *c_tptr, int64_t nC, int64_t nT, double *c_blocks, double *c_sumsq,
                                   uint8_t *c_nonzero, int64_t *zero_count, int64_t *panel_count, void *ws,
                                   size_t ws_bytes, void *stream) {
  Geometry g;
  int rc = make_geometry(layout, &g);
  if (rc != QM_OK) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (zero_count) QM_CUDA_TRY(cudaMemsetAsync(zero_count, 0, sizeof(int64_t), st));
  if (panel_count) QM_CUDA_TRY(cudaMemsetAsync(panel_count, nC == 0 ? 0 : 0xff, sizeof(int64_t), st));
  if (nC <= 0) return nC < 0 ? QM_ERR_INVALID : QM_OK;
  if (!a_pools || !b_pools || !a_counts || !b_counts) {
    set_error("qm_numeric_pools_ex: NULL pool arrays");
    return QM_ERR_INVALID;
  }
  const bool any_mask = a_cmask || a_flags || b_rmask || b_flags;
  if (any_mask && (!a_cmask || !a_flags || !b_rmask || !b_flags || (!mask_tri && (n_a_pools > 1 || n_b_pools > 1)))) {
    set_error("qm_numeric_pools_ex: masks need A's column masks and flags, B's row masks and flags, and, for "
              "several pools, mask_tri");
    return QM_ERR_INVALID;
  }
  if (halo && (halo->world < 1 || halo->world > QM_MAX_RANKS || halo->count[0] < 0 || halo->count[1] < 0 ||
               (halo->count[0] && (!halo->index[0] || !halo->pool[0])) ||
               (halo->count[1] && (!halo->index[1] || !halo->pool[1])) || gate_units < 0)) {
    set_error("qm_numeric_pools_ex: bad halo arguments");
    return QM_ERR_INVALID;
  }
  NumericAux oi;
  oi.nbl = g.nbl;
  oi.lbits = g.lbits;
  oi.nbg = g.nbg;
  if (any_mask) {
    oi.a_cols = a_cmask, oi.a_flags = a_flags;
    oi.b_rows = b_rmask, oi.b_flags = b_flags;
  }
  oi.panel_count = panel_count;
  oi.order = order;
  oi.mask_tri = mask_tri;
  oi.halo = (halo && halo->count[0] + halo->count[1] > 0) ? halo : nullptr;
  oi.gate_units = gate_units;
  return launch_numeric_tma(g.bs, a_pools, a_counts, n_a_pools, b_pools, b_counts, n_b_pools, tri, c_tptr, nC, nT,
                            oi, c_blocks, c_sumsq, c_nonzero, zero_count, ws, ws_bytes, st);
}

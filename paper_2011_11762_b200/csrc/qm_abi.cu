// C-ABI plumbing of libqmb200: error state, launch counter, key encode/decode, exact-zero
// compaction and block gather (halo packing).
#include <cub/cub.cuh>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "qm_common.cuh"

namespace qm {

static thread_local char t_err[1024] = "";
static std::atomic<uint64_t> g_launches{0};

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(t_err, sizeof(t_err), fmt, ap);
  va_end(ap);
}

void note_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

__global__ void k_read_i64(const int64_t *src, int n, const int64_t *src2, volatile int64_t *dst) {
  if (threadIdx.x < n) dst[threadIdx.x] = src[threadIdx.x];
  if (src2 && threadIdx.x == 0) dst[n] = *src2;
}

int mapped_i64(int64_t **host, int64_t **dev) {
  // One mapped buffer per (thread, device): a thread that alternates GPUs reuses each device's
  // buffer instead of allocating (and leaking) a new one on every switch. (Not freed at thread
  // exit: the CUDA runtime may already be unloading then; it is 64 bytes per thread and device.)
  struct Mapped {
    int64_t *host[64] = {};
    int64_t *dev[64] = {};
  };
  static thread_local Mapped m;
  int device = 0;
  QM_CUDA_TRY(cudaGetDevice(&device));
  const int d = device & 63;
  if (m.host[d] == nullptr) {
    QM_CUDA_TRY(cudaHostAlloc((void **)&m.host[d], 8 * sizeof(int64_t), cudaHostAllocMapped | cudaHostAllocPortable));
    QM_CUDA_TRY(cudaHostGetDevicePointer((void **)&m.dev[d], m.host[d], 0));
  }
  *host = m.host[d];
  *dev = m.dev[d];
  return QM_OK;
}

int read_device_i64(const void *dev_src, int n, int64_t *host_out, cudaStream_t stream,
                    const void *dev_src2) {
  struct {
    int64_t *host = nullptr, *dev = nullptr;
  } m;
  int rc = mapped_i64(&m.host, &m.dev);
  if (rc != QM_OK) return rc;
  if (n < 1 || n > 8) {
    set_error("read_device_i64: n=%d out of range", n);
    return QM_ERR_INVALID;
  }
  if (dev_src2 && n > 7) {
    set_error("read_device_i64: n=%d too large with a second source", n);
    return QM_ERR_INVALID;
  }
  k_read_i64<<<1, 32, 0, stream>>>((const int64_t *)dev_src, n, (const int64_t *)dev_src2, m.dev);
  QM_LAUNCHED("k_read_i64");
  QM_CUDA_TRY(cudaStreamSynchronize(stream));
  const int total = n + (dev_src2 ? 1 : 0);
  for (int i = 0; i < total; ++i) host_out[i] = ((volatile int64_t *)m.host)[i];
  return QM_OK;
}

int launch_block_stats(int bs, int64_t n, const double *blocks, double *sumsq, uint8_t *nonzero,
                       int64_t *zero_count, cudaStream_t st);

namespace {

inline int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (int)g;
}

__global__ void k_encode(const int32_t *bi, const int32_t *bj, int64_t n, int nbl, int lbits,
                         uint64_t *keys) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x)
    keys[x] = qkey((uint32_t)bi[x], (uint32_t)bj[x], nbl, lbits);
}

__global__ void k_decode(const uint64_t *keys, int64_t n, int nbl, int lbits, int32_t *bi,
                         int32_t *bj) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    uint32_t r, c;
    qkey_decode(keys[x], nbl, lbits, &r, &c);
    bi[x] = (int32_t)r;
    bj[x] = (int32_t)c;
  }
}

__global__ void k_flags_to_i64(const uint8_t *f, int64_t n, int64_t *out) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x)
    out[x] = f[x] ? 1 : 0;
}

// One CTA copies one block: 16-byte vectors, four loads in flight per thread (streaming loads --
// the source is read once).
__device__ __forceinline__ void copy_block(const double *__restrict__ s, double *__restrict__ o,
                                           int64_t elems) {
  if ((elems & 1) == 0) {
    const double2 *s2 = reinterpret_cast<const double2 *>(s);
    double2 *o2 = reinterpret_cast<double2 *>(o);
    const int64_t n2 = elems / 2, st = blockDim.x;
    int64_t e = threadIdx.x;
    for (; e + 3 * st < n2; e += 4 * st) {
      const double2 v0 = __ldcs(s2 + e), v1 = __ldcs(s2 + e + st), v2 = __ldcs(s2 + e + 2 * st),
                    v3 = __ldcs(s2 + e + 3 * st);
      o2[e] = v0;
      o2[e + st] = v1;
      o2[e + 2 * st] = v2;
      o2[e + 3 * st] = v3;
    }
    for (; e < n2; e += st) o2[e] = __ldcs(s2 + e);
  } else {
    for (int64_t e = threadIdx.x; e < elems; e += blockDim.x) o[e] = s[e];
  }
}

// One CTA per block: copies the kept blocks to their compacted slot.
__global__ void __launch_bounds__(256) k_compact(int bs, int64_t n, const uint8_t *flags,
                                                 const int64_t *pos, const uint64_t *keys_in,
                                                 const double *blocks_in, const double *sumsq_in,
                                                 uint64_t *keys_out, double *blocks_out,
                                                 double *sumsq_out) {
  const int64_t elems = (int64_t)bs * bs;
  for (int64_t m = blockIdx.x; m < n; m += gridDim.x) {
    if (!flags[m]) continue;
    const int64_t d = pos[m];
    if (threadIdx.x == 0) {
      keys_out[d] = keys_in[m];
      if (sumsq_out) sumsq_out[d] = sumsq_in[m];
    }
    copy_block(blocks_in + (size_t)m * elems, blocks_out + (size_t)d * elems, elems);
  }
}

__global__ void __launch_bounds__(256) k_gather_blocks(int bs, const double *src, const int64_t *idx,
                                                       int64_t n, double *dst) {
  const int64_t elems = (int64_t)bs * bs;
  for (int64_t m = blockIdx.x; m < n; m += gridDim.x) {
    copy_block(src + (size_t)idx[m] * elems, dst + (size_t)m * elems, elems);
  }
}

// dst[i] = transpose(src[i]) for bs x bs blocks (32x33 smem tiles).
__global__ void __launch_bounds__(256) k_transpose_blocks(int bs, const double *src, int64_t n, double *dst) {
  __shared__ double tile[32][33];
  const int nt = (bs + 31) / 32;
  const int64_t work = n * nt * nt;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int64_t w = blockIdx.x; w < work; w += gridDim.x) {
    const int64_t m = w / (nt * nt);
    const int t = (int)(w % (nt * nt));
    const int r0 = (t / nt) * 32, c0 = (t % nt) * 32;
    const double *s = src + (size_t)m * bs * bs;
    double *d = dst + (size_t)m * bs * bs;
    for (int q = ty; q < 32; q += 8)
      if (r0 + q < bs && c0 + tx < bs) tile[q][tx] = s[(size_t)(r0 + q) * bs + c0 + tx];
    __syncthreads();
    for (int q = ty; q < 32; q += 8)
      if (c0 + q < bs && r0 + tx < bs) d[(size_t)(c0 + q) * bs + r0 + tx] = tile[tx][q];
    __syncthreads();
  }
}

// dst[m] = src[idx[m]], transposed when tflag[m] != 0 (32x33 smem tiles): the expansion of a
// symmetric operand's stored upper triangle in one pass (variants.expand_symmetric).
__global__ void __launch_bounds__(256) k_gather_blocks_t(int bs, const double *src, const int64_t *idx,
                                                         const uint8_t *tflag, int64_t n, double *dst) {
  __shared__ double tile[32][33];
  const int nt = (bs + 31) / 32;
  const int64_t work = n * nt * nt;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int64_t w = blockIdx.x; w < work; w += gridDim.x) {
    const int64_t m = w / (nt * nt);
    const int t = (int)(w % (nt * nt));
    const int r0 = (t / nt) * 32, c0 = (t % nt) * 32;
    const double *sb = src + (size_t)idx[m] * bs * bs;
    double *d = dst + (size_t)m * bs * bs;
    const bool tr = tflag && tflag[m];
    for (int q = ty; q < 32; q += 8)
      if (r0 + q < bs && c0 + tx < bs) tile[q][tx] = __ldcs(sb + (size_t)(r0 + q) * bs + c0 + tx);
    __syncthreads();
    for (int q = ty; q < 32; q += 8) {
      if (tr) {
        if (c0 + q < bs && r0 + tx < bs) d[(size_t)(c0 + q) * bs + r0 + tx] = tile[tx][q];
      } else if (r0 + q < bs && c0 + tx < bs) {
        d[(size_t)(r0 + q) * bs + c0 + tx] = tile[q][tx];
      }
    }
    __syncthreads();
  }
}

// out[m] = alpha*A[ia[m]] + beta*B[ib[m]] with an operand absent when its index is -1 (then
// alpha*A or beta*B alone). Exact IEEE products and sum (no FMA contraction), like numpy's
// `alpha * a + beta * b` in BlockSparseLeaf.add / scale (block_sparse.py:134-160).
__device__ __forceinline__ double axpby1(bool ha, bool hb, double alpha, double beta, double a, double b) {
  if (ha && hb) return __dadd_rn(__dmul_rn(alpha, a), __dmul_rn(beta, b));
  return ha ? __dmul_rn(alpha, a) : __dmul_rn(beta, b);
}

// One CTA (256 threads) per output block; thread t handles elements t, t+256, ... with four
// loads per operand in flight (no FMA contraction: alpha*a + beta*b rounds like numpy's two
// products and one sum). Optionally fuses the output block's statistics in exactly
// k_block_stats's order (per-thread fma chain over its elements, warp xor tree, warps in order),
// so the sum of squares is bit-identical to a separate qm_block_stats pass over the output.
__global__ void __launch_bounds__(256) k_axpby(int64_t elems, int64_t n, const int64_t *ia,
                                               const int64_t *ib, double alpha, double beta,
                                               const double *A, const double *B, double *out,
                                               double *sumsq, uint8_t *nonzero, int64_t *zero_count) {
  __shared__ double red[8];
  __shared__ int rnz[8];
  const bool stats = sumsq || nonzero || zero_count;
  for (int64_t m = blockIdx.x; m < n; m += gridDim.x) {
    const int64_t x = ia[m], y = ib[m];
    const bool ha = x >= 0, hb = y >= 0;
    const double *a = ha ? A + (size_t)x * elems : nullptr;
    const double *b = hb ? B + (size_t)y * elems : nullptr;
    double *o = out + (size_t)m * elems;
    const int64_t st = blockDim.x;
    double ss = 0.0;
    bool nz = false;
    int64_t e = threadIdx.x;
    for (; e + 3 * st < elems; e += 4 * st) {
      double va[4], vb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        va[u] = ha ? a[e + u * st] : 0.0;
        vb[u] = hb ? b[e + u * st] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double v = axpby1(ha, hb, alpha, beta, va[u], vb[u]);
        o[e + u * st] = v;
        ss = fma(v, v, ss);
        nz |= v != 0.0;
      }
    }
    for (; e < elems; e += st) {
      const double v = axpby1(ha, hb, alpha, beta, ha ? a[e] : 0.0, hb ? b[e] : 0.0);
      o[e] = v;
      ss = fma(v, v, ss);
      nz |= v != 0.0;
    }
    if (!stats) continue;
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    const bool wnz = __any_sync(0xffffffffu, nz);
    if ((threadIdx.x & 31) == 0) {
      red[threadIdx.x >> 5] = ss;
      rnz[threadIdx.x >> 5] = wnz;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      int any = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        tot += red[w];
        any |= rnz[w];
      }
      if (sumsq) sumsq[m] = tot;
      if (nonzero) nonzero[m] = (uint8_t)any;
      if (!any && zero_count) atomicAdd((unsigned long long *)zero_count, 1ull);
    }
    __syncthreads();
  }
}

// Diagonal blocks of A + c*I (ops.py:253-345, block_sparse.py:162-175). mode[m]:
//   0  leaf of A present and inside n_logical: A_blk + c*eye (c*eye alone when A_blk absent)
//   1  partial / absent leaf: identity block from triplets (c on the logical diagonal, +0.0
//      elsewhere), added as 1.0*A + 1.0*I when A_blk is present.
__global__ void __launch_bounds__(256) k_add_identity(int bs, int64_t n, const int64_t *ia,
                                                      const int64_t *bi, const int8_t *mode, double c,
                                                      int64_t n_logical, const double *A, double *out) {
  const int64_t elems = (int64_t)bs * bs;
  for (int64_t m = blockIdx.x; m < n; m += gridDim.x) {
    const double *a = ia[m] >= 0 ? A + (size_t)ia[m] * elems : nullptr;
    double *o = out + (size_t)m * elems;
    const int64_t row0 = bi[m] * bs;
    for (int64_t e = threadIdx.x; e < elems; e += blockDim.x) {
      const int r = (int)(e / bs), col = (int)(e % bs);
      double v;
      if (mode[m] == 0) {
        const double ce = __dmul_rn(c, r == col ? 1.0 : 0.0);
        v = a ? __dadd_rn(a[e], ce) : ce;
      } else {
        const double id = (r == col && row0 + r < n_logical) ? c : 0.0;
        v = a ? __dadd_rn(__dmul_rn(1.0, a[e]), __dmul_rn(1.0, id)) : id;
      }
      o[e] = v;
    }
  }
}

size_t compact_cub_bytes(int64_t n) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t *)nullptr, (int64_t *)nullptr, n);
  return b;
}

}  // namespace
}  // namespace qm

using namespace qm;

extern "C" int qm_abi_version(void) { return QM_ABI_VERSION; }

extern "C" const char *qm_last_error(void) { return qm::t_err; }

extern "C" uint64_t qm_launch_count(void) { return qm::g_launches.load(std::memory_order_relaxed); }

extern "C" int qm_encode_keys(const qm_layout *layout, const int32_t *bi, const int32_t *bj, int64_t n,
                              uint64_t *keys, void *stream) {
  Geometry g;
  int rc = make_geometry(layout, &g);
  if (rc != QM_OK) return rc;
  if (n <= 0) return QM_OK;
  k_encode<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(bi, bj, n, g.nbl, g.lbits, keys);
  QM_LAUNCHED("k_encode");
  return QM_OK;
}

extern "C" int qm_decode_keys(const qm_layout *layout, const uint64_t *keys, int64_t n, int32_t *bi,
                              int32_t *bj, void *stream) {
  Geometry g;
  int rc = make_geometry(layout, &g);
  if (rc != QM_OK) return rc;
  if (n <= 0) return QM_OK;
  k_decode<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(keys, n, g.nbl, g.lbits, bi, bj);
  QM_LAUNCHED("k_decode");
  return QM_OK;
}

extern "C" size_t qm_compact_workspace_bytes(int64_t nC) {
  Carver cv(nullptr, 0);
  cv.take<int64_t>(nC);
  cv.take<int64_t>(nC);
  cv.take<char>(compact_cub_bytes(nC));
  return cv.off;
}

extern "C" int qm_compact(int32_t block_size, int64_t nC, const uint8_t *c_nonzero,
                          const uint64_t *keys_in, const double *blocks_in, const double *sumsq_in,
                          uint64_t *keys_out, double *blocks_out, double *sumsq_out, void *ws,
                          size_t ws_bytes, void *stream) {
  if (block_size < 1 || nC < 0) {
    set_error("qm_compact: bad arguments");
    return QM_ERR_INVALID;
  }
  if (nC == 0) return QM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Carver cv(ws, ws_bytes);
  int64_t *f64 = cv.take<int64_t>(nC);
  int64_t *pos = cv.take<int64_t>(nC);
  size_t cb = compact_cub_bytes(nC);
  void *cub = cv.take<char>(cb);
  if (!cv.ok() || !ws) {
    set_error("qm_compact: workspace %zu < required %zu", ws_bytes, cv.off);
    return QM_ERR_WORKSPACE;
  }
  k_flags_to_i64<<<grid_for(nC), 256, 0, st>>>(c_nonzero, nC, f64);
  QM_LAUNCHED("k_flags_to_i64");
  QM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(cub, cb, f64, pos, nC, st));
  int64_t grid = std::min<int64_t>(nC, 148 * 16);
  k_compact<<<(int)grid, 256, 0, st>>>(block_size, nC, c_nonzero, pos, keys_in, blocks_in, sumsq_in,
                                       keys_out, blocks_out, sumsq_out);
  QM_LAUNCHED("k_compact");
  return QM_OK;
}

extern "C" int qm_gather_blocks(int32_t block_size, const double *src, const int64_t *idx, int64_t n,
                                double *dst, void *stream) {
  if (block_size < 1 || n < 0) {
    set_error("qm_gather_blocks: bad arguments");
    return QM_ERR_INVALID;
  }
  if (n == 0) return QM_OK;
  int64_t grid = std::min<int64_t>(n, 148 * 16);
  k_gather_blocks<<<(int)grid, 256, 0, (cudaStream_t)stream>>>(block_size, src, idx, n, dst);
  QM_LAUNCHED("k_gather_blocks");
  return QM_OK;
}

extern "C" int qm_transpose_blocks(int32_t block_size, const double *src, int64_t n, double *dst,
                                   void *stream) {
  if (block_size < 1 || n < 0 || src == dst) {
    set_error("qm_transpose_blocks: bad arguments (in-place is not supported)");
    return QM_ERR_INVALID;
  }
  if (n == 0) return QM_OK;
  const int nt = (block_size + 31) / 32;
  int64_t grid = std::min<int64_t>(n * nt * nt, 148 * 16);
  k_transpose_blocks<<<(int)grid, 256, 0, (cudaStream_t)stream>>>(block_size, src, n, dst);
  QM_LAUNCHED("k_transpose_blocks");
  return QM_OK;
}

extern "C" int qm_gather_blocks_t(int32_t block_size, const double *src, const int64_t *idx,
                                  const uint8_t *transpose, int64_t n, double *dst, void *stream) {
  if (block_size < 1 || n < 0 || (n > 0 && (!src || !idx || !dst))) {
    set_error("qm_gather_blocks_t: bad arguments");
    return QM_ERR_INVALID;
  }
  if (n == 0) return QM_OK;
  const int nt = (block_size + 31) / 32;
  int64_t grid = std::min<int64_t>(n * nt * nt, 148 * 32);
  k_gather_blocks_t<<<(int)grid, 256, 0, (cudaStream_t)stream>>>(block_size, src, idx, transpose, n, dst);
  QM_LAUNCHED("k_gather_blocks_t");
  return QM_OK;
}

extern "C" int qm_axpby_blocks(int32_t block_size, int64_t n, const int64_t *ia, const int64_t *ib,
                               double alpha, double beta, const double *a_blocks,
                               const double *b_blocks, double *out, double *out_sumsq,
                               uint8_t *out_nonzero, int64_t *zero_count, void *stream) {
  if (block_size < 1 || n < 0) {
    set_error("qm_axpby_blocks: bad arguments");
    return QM_ERR_INVALID;
  }
  if (n == 0) return QM_OK;
  int64_t grid = std::min<int64_t>(n, 148 * 16);
  k_axpby<<<(int)grid, 256, 0, (cudaStream_t)stream>>>((int64_t)block_size * block_size, n, ia, ib, alpha,
                                                       beta, a_blocks, b_blocks, out, out_sumsq,
                                                       out_nonzero, zero_count);
  QM_LAUNCHED("k_axpby");
  return QM_OK;
}

extern "C" int qm_add_identity_blocks(int32_t block_size, int64_t n, const int64_t *ia,
                                      const int64_t *bi, const int8_t *mode, double c, int64_t n_logical,
                                      const double *a_blocks, double *out, void *stream) {
  if (block_size < 1 || n < 0) {
    set_error("qm_add_identity_blocks: bad arguments");
    return QM_ERR_INVALID;
  }
  if (n == 0) return QM_OK;
  int64_t grid = std::min<int64_t>(n, 148 * 16);
  k_add_identity<<<(int)grid, 256, 0, (cudaStream_t)stream>>>(block_size, n, ia, bi, mode, c, n_logical,
                                                              a_blocks, out);
  QM_LAUNCHED("k_add_identity");
  return QM_OK;
}

extern "C" int qm_read_i64(const int64_t *dev_src, int32_t n, int64_t *host_out, void *stream) {
  return read_device_i64(dev_src, n, host_out, (cudaStream_t)stream);
}

// ---- CUDA IPC for the fused multi-GPU product: a block pool is exported as the IPC handle of its
// ---- allocation plus the pool's byte offset inside it (torch's caching allocator sub-allocates).
extern "C" int qm_ipc_export(const void *ptr, void *handle_out /*64 bytes*/, int64_t *offset_out) {
  static const PFN_cuMemGetAddressRange_v3020 get_range = [] {  // thread-safe one-time lookup
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return (PFN_cuMemGetAddressRange_v3020)fn;
  }();
  if (!get_range) {
    set_error("qm_ipc_export: cuMemGetAddressRange unavailable");
    return QM_ERR_CUDA;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) {
    set_error("qm_ipc_export: pointer %p is not a device allocation", ptr);
    return QM_ERR_INVALID;
  }
  cudaIpcMemHandle_t h;
  QM_CUDA_TRY(cudaIpcGetMemHandle(&h, (void *)base));
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = (int64_t)((CUdeviceptr)ptr - base);
  return QM_OK;
}

extern "C" int qm_ipc_open(const void *handle /*64 bytes*/, void **base_out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  QM_CUDA_TRY(cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess));
  return QM_OK;
}

extern "C" int qm_ipc_close(void *base) {
  QM_CUDA_TRY(cudaIpcCloseMemHandle(base));
  return QM_OK;
}

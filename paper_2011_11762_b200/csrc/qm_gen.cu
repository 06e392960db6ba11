// Device-side synthetic inputs and the FP64 peak microbenchmarks.
//
// The block-keyed generator gives block (bi, bj) of matrix m the values of
// numpy's np.random.default_rng([seed, m, bi, bj]).uniform(-1, 1, (bs, bs)). This file restates
// numpy's SeedSequence (pool size 4, hashmix/mix constants) and PCG64 (128-bit LCG, XSL-RR output,
// double = (next >> 11) * 2^-53) so any block is produced on the device bit-identically to the
// host oracle; the CPU oracle can therefore regenerate and check any sampled block of a product too
// large for the CPU (C5). One thread per block row: the stream is advanced by row * bs draws with
// the O(log n) LCG jump-ahead.
#include <cuda_runtime.h>

#include "qm_common.cuh"

namespace qm {
int launch_block_stats(int bs, int64_t n, const double *blocks, double *sumsq, uint8_t *nonzero,
                       int64_t *zero_count, cudaStream_t st);
int numeric_sm_count();

namespace {

typedef unsigned __int128 u128;

constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u, kInitB = 0x8b51f9ddu,
                   kMultB = 0x58f38dedu, kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

__device__ __forceinline__ uint32_t hashmix(uint32_t v, uint32_t &hc) {
  v ^= hc;
  hc *= kMultA;
  v *= hc;
  v ^= v >> 16;
  return v;
}

__device__ __forceinline__ uint32_t mixw(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  r ^= r >> 16;
  return r;
}

// numpy SeedSequence(entropy).generate_state(4, uint64) for an entropy of up to 8 uint32 words.
__device__ void seed_sequence_state(const uint32_t *ent, int n, uint64_t out[4]) {
  uint32_t pool[4];
  uint32_t hc = kInitA;
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n ? ent[i] : 0u, hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mixw(pool[d], hashmix(pool[s], hc));
  for (int s = 4; s < n; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mixw(pool[d], hashmix(ent[s], hc));
  uint32_t w[8];
  uint32_t hb = kInitB;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  for (int i = 0; i < 4; ++i) out[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
}

__device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

struct Pcg64 {
  u128 state, inc;
  __device__ void seed(const uint64_t v[4]) {
    const u128 s = ((u128)v[0] << 64) | v[1];
    const u128 i = ((u128)v[2] << 64) | v[3];
    inc = (i << 1) | 1u;
    state = 0;
    state = state * pcg_mult() + inc;
    state += s;
    state = state * pcg_mult() + inc;
  }
  __device__ void advance(uint64_t delta) {
    u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
    while (delta > 0) {
      if (delta & 1) {
        acc_mult *= cur_mult;
        acc_plus = acc_plus * cur_mult + cur_plus;
      }
      cur_plus = (cur_mult + 1) * cur_plus;
      cur_mult *= cur_mult;
      delta >>= 1;
    }
    state = acc_mult * state + acc_plus;
  }
  __device__ __forceinline__ uint64_t next() {
    state = state * pcg_mult() + inc;
    const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
    const unsigned r = (unsigned)(state >> 122);
    return (x >> r) | (x << ((64 - r) & 63));
  }
};

__device__ __forceinline__ int push_words(uint32_t *ent, int n, uint64_t v) {
  if (v == 0) {
    ent[n++] = 0;
    return n;
  }
  while (v) {
    ent[n++] = (uint32_t)v;
    v >>= 32;
  }
  return n;
}

__global__ void __launch_bounds__(128) k_generate(const uint64_t *keys, int64_t nblk, int bs, int nbl,
                                                  int lbits, int64_t n_logical, uint64_t seed,
                                                  uint32_t mid, int pattern, int64_t hb,
                                                  double *blocks) {
  const int64_t rows = nblk * bs;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < rows;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = w / bs;
    const int r = (int)(w % bs);
    uint32_t bi, bj;
    qkey_decode(keys[m], nbl, lbits, &bi, &bj);
    const int64_t gi = (int64_t)bi * bs + r;
    double *out = blocks + (size_t)m * bs * bs + (size_t)r * bs;
    if (pattern == 2) {
      for (int c = 0; c < bs; ++c) {
        const int64_t gj = (int64_t)bj * bs + c;
        const int64_t d = gi - gj;
        out[c] = (gi < n_logical && gj < n_logical && d <= hb && -d <= hb) ? 1.0 : 0.0;
      }
      continue;
    }
    uint32_t ent[8];
    int ne = 0;
    ne = push_words(ent, ne, seed);
    ne = push_words(ent, ne, mid);
    ne = push_words(ent, ne, bi);
    ne = push_words(ent, ne, bj);
    uint64_t st[4];
    seed_sequence_state(ent, ne, st);
    Pcg64 g;
    g.seed(st);
    if (r) g.advance((uint64_t)r * bs);
    for (int c = 0; c < bs; ++c) {
      const double u = (double)(g.next() >> 11) * (1.0 / 9007199254740992.0);
      const double v = -1.0 + 2.0 * u;
      const int64_t gj = (int64_t)bj * bs + c;
      bool keep = gi < n_logical && gj < n_logical;
      if (pattern == 1) {
        const int64_t d = gi - gj;
        keep = keep && d <= hb && -d <= hb;
      }
      out[c] = keep ? v : 0.0;
    }
  }
}

// FP64 peak probes: 8 independent accumulator chains per thread (DMMA: per warp).
__global__ void k_peak_dmma(int64_t iters, double *sink) {
  double d[8][2];
  const double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
#pragma unroll
  for (int u = 0; u < 8; ++u) d[u][0] = d[u][1] = 0.0;
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[u][0]), "+d"(d[u][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += d[u][0] + d[u][1];
  if (s == 12345.678) sink[0] = s;
}

__global__ void k_peak_dfma(int64_t iters, double *sink) {
  double d[8];
  const double a = 1.0 + 1e-9 * threadIdx.x, b = 1e-9;
#pragma unroll
  for (int u = 0; u < 8; ++u) d[u] = u;
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) asm volatile("fma.rn.f64 %0, %0, %1, %2;\n" : "+d"(d[u]) : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += d[u];
  if (s == 12345.678) sink[0] = s;
}

}  // namespace
}  // namespace qm

using namespace qm;

extern "C" int qm_generate_blocks(const qm_layout *layout, const uint64_t *keys, int64_t n,
                                  uint64_t seed, uint32_t matrix_id, int32_t pattern, int64_t half_bw,
                                  double *blocks, double *sumsq, void *stream) {
  Geometry g;
  int rc = make_geometry(layout, &g);
  if (rc != QM_OK) return rc;
  if (pattern < 0 || pattern > 2 || n < 0) {
    set_error("qm_generate_blocks: bad pattern %d or count", pattern);
    return QM_ERR_INVALID;
  }
  if (n == 0) return QM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rows = n * g.bs;
  int64_t grid = std::min<int64_t>((rows + 127) / 128, (int64_t)numeric_sm_count() * 16);
  k_generate<<<(int)grid, 128, 0, st>>>(keys, n, g.bs, g.nbl, g.lbits, layout->n_logical, seed,
                                        matrix_id, pattern, half_bw, blocks);
  QM_LAUNCHED("k_generate");
  if (sumsq) return launch_block_stats(g.bs, n, blocks, sumsq, nullptr, nullptr, st);
  return QM_OK;
}

extern "C" int qm_fp64_peak_kernel(int kind, int ctas, int threads, int64_t iters, double *sink,
                                   double *flops, void *stream) {
  if (ctas < 1 || threads < 32 || threads % 32 || iters < 1 || (kind != 0 && kind != 1)) {
    set_error("qm_fp64_peak_kernel: bad arguments");
    return QM_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (kind == 0) {
    k_peak_dmma<<<ctas, threads, 0, st>>>(iters, sink);
    if (flops) *flops = (double)ctas * (threads / 32) * (double)iters * 8.0 * 512.0;
  } else {
    k_peak_dfma<<<ctas, threads, 0, st>>>(iters, sink);
    if (flops) *flops = (double)ctas * threads * (double)iters * 8.0 * 2.0;
  }
  QM_LAUNCHED("k_peak");
  return QM_OK;
}

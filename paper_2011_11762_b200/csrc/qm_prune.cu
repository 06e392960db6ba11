// Approximate (norm-pruned) multiply: the reference's prune decisions, level by level, on device.
//
// Reference: every multiply task at quadtree level l whose operand nodes X (rows I, cols K) and
// Y (rows K, cols J) are both non-nil first tests norm(X) * norm(Y) < tau_l (ops.py:199-204) with
// tau_0 = tau and tau_{l+1} = tau_l / 8 (ops.py:232); a pruned task logs its bound
// (ctx.log_prune, engine.py:273-275) and returns nil, otherwise it spawns its 8 child products.
// Node norms are the store's id-carried Frobenius norms: a leaf's is sqrt(fsum(block_norm^2))
// (block_sparse.py:91-92), a branch's sqrt(fsum(child_norm^2)) (quadtree.py:138-140).
//
// B200 form:
//   qm_node_norms  -- every level's node table of one operand (Morton node code, norm), built
//                     bottom-up from the block sums of squares: runs of equal codes in quadtree-key
//                     order are the nodes, summed with compensated (Neumaier) summation in order,
//                     which rounds like fsum for these short runs of positive terms;
//   qm_prune_level -- one level of the task recursion: the 8 children of every surviving pair of
//                     the previous level (or the root pair), node lookups by binary search in the
//                     tables (stored-chunk norms: a symmetric operand's lower nodes read their
//                     upper mirror, a transposed operand swaps the coordinates), classification
//                     dead / pruned / alive, and stream compaction of the alive pairs (packed
//                     I<<42 | K<<21 | J) and of the pruned bounds (the prune log).
#include <math.h>
#include <string.h>

#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "qm_common.cuh"

namespace qm {
namespace {

constexpr int kPairBits = 21;  // node coordinates of up to 2^21 per side per level
constexpr uint64_t kPairMask = (1ull << kPairBits) - 1ull;

inline int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (int)g;
}

__device__ __forceinline__ void neumaier_add(double &s, double &c, double x) {
  const double t = s + x;
  if (fabs(s) >= fabs(x)) c += (s - t) + x;
  else c += (x - t) + s;
  s = t;
}

// head[i] = 1 when code(i) = in[i] >> shift starts a run; head[n] = 0 (exclusive-scan tail).
__global__ void k_run_heads(const uint64_t *in, int64_t n, int shift, int64_t *head) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
    head[i] = (i < n && (i == 0 || (in[i] >> shift) != (in[i - 1] >> shift))) ? 1 : 0;
}

__global__ void k_run_starts(const uint64_t *in, int64_t n, int shift, const int64_t *head,
                             const int64_t *pos, uint64_t *out_code, int64_t *start) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (head[i]) {
      out_code[pos[i]] = in[i] >> shift;
      start[pos[i]] = i;
    }
}

// norm of run j = sqrt(sum over its members of v^2), v = sqrt(sumsq) for blocks (from_sumsq)
// or the member's norm for nodes; members summed in key order.
__global__ void k_run_norms(const double *vals, int from_sumsq, int64_t n_in, const int64_t *start,
                            int64_t n_runs, double *out_norm) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_runs;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = j + 1 < n_runs ? start[j + 1] : n_in;
    double s = 0.0, c = 0.0;
    for (int64_t i = start[j]; i < e; ++i) {
      const double v = from_sumsq ? sqrt(vals[i]) : vals[i];
      neumaier_add(s, c, v * v);
    }
    out_norm[j] = sqrt(s + c);
  }
}

struct Table {
  const uint64_t *code;
  const double *norm;
  int64_t n;
};

// Norm of node (r, c) (0 when absent). sym: a lower node reads its stored upper mirror.
__device__ __forceinline__ bool lookup(const Table &t, uint32_t r, uint32_t c, bool sym, double *norm) {
  if (sym && r > c) {
    const uint32_t x = r;
    r = c;
    c = x;
  }
  const uint64_t q = (spread_bits(r) << 1) | spread_bits(c);
  int64_t lo = 0, hi = t.n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (t.code[mid] < q) lo = mid + 1; else hi = mid;
  }
  if (lo < t.n && t.code[lo] == q) {
    *norm = t.norm[lo];
    return true;
  }
  return false;
}

// Candidate x: child (x % 8) of parent x / 8 (or the root pair). status: 0 dead, 1 pruned, 2 alive.
__global__ void k_prune_expand(const uint64_t *parents, int64_t n_cand, int root, Table ta, int a_sym,
                               Table tb, int b_sym, int b_transposed, int upper, double tau_l,
                               uint64_t *cand, double *bound, uint8_t *alive, uint8_t *pruned) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n_cand;
       x += (int64_t)gridDim.x * blockDim.x) {
    uint32_t I = 0, K = 0, J = 0;
    if (!root) {
      const uint64_t p = parents[x >> 3];
      const uint32_t d = (uint32_t)(x & 7);
      I = 2 * (uint32_t)(p >> (2 * kPairBits)) + (d >> 2);
      K = 2 * (uint32_t)((p >> kPairBits) & kPairMask) + ((d >> 1) & 1u);
      J = 2 * (uint32_t)(p & kPairMask) + (d & 1u);
    }
    double na = 0.0, nb = 0.0;
    bool live = lookup(ta, I, K, a_sym, &na);
    if (live) live = b_transposed ? lookup(tb, J, K, b_sym, &nb) : lookup(tb, K, J, b_sym, &nb);
    if (upper && I > J) live = false;
    const double bd = na * nb;
    const bool pr = live && bd < tau_l;
    cand[x] = ((uint64_t)I << (2 * kPairBits)) | ((uint64_t)K << kPairBits) | J;
    bound[x] = bd;
    alive[x] = (uint8_t)(live && !pr);
    pruned[x] = (uint8_t)pr;
  }
}

// Classification of candidate x (shared by the two level kernels).
__device__ __forceinline__ void prune_classify(const uint64_t *parents, int64_t x, int root, const Table &ta,
                                               int a_sym, const Table &tb, int b_sym, int b_transposed, int upper,
                                               double tau_l, uint64_t *code, double *bd, bool *live, bool *pr) {
  uint32_t I = 0, K = 0, J = 0;
  if (!root) {
    const uint64_t p = parents[x >> 3];
    const uint32_t d = (uint32_t)(x & 7);
    I = 2 * (uint32_t)(p >> (2 * kPairBits)) + (d >> 2);
    K = 2 * (uint32_t)((p >> kPairBits) & kPairMask) + ((d >> 1) & 1u);
    J = 2 * (uint32_t)(p & kPairMask) + (d & 1u);
  }
  double na = 0.0, nb = 0.0;
  bool lv = lookup(ta, I, K, a_sym, &na);
  if (lv) lv = b_transposed ? lookup(tb, J, K, b_sym, &nb) : lookup(tb, K, J, b_sym, &nb);
  if (upper && I > J) lv = false;
  *bd = na * nb;
  *pr = lv && *bd < tau_l;
  *live = lv && !*pr;
  *code = ((uint64_t)I << (2 * kPairBits)) | ((uint64_t)K << kPairBits) | J;
}

// Small levels in one CTA (one launch instead of expand + two stream compactions): each thread
// classifies up to kSmallPer consecutive candidates (kept in registers), a block-wide exclusive scan
// orders the survivors exactly as the stable compaction of the multi-kernel path does, and the two
// counts go straight to the caller's mapped host buffer.
constexpr int kSmallThreads = 1024;
constexpr int kSmallPer = 4;
constexpr int64_t kSmallLevelMax = (int64_t)kSmallThreads * kSmallPer;
__global__ void __launch_bounds__(kSmallThreads) k_prune_small(const uint64_t *parents, int64_t n_cand, int root,
                                                             Table ta, int a_sym, Table tb, int b_sym,
                                                             int b_transposed, int upper, double tau_l,
                                                             uint64_t *alive_out, double *pruned_out,
                                                             volatile int64_t *host_cnt) {
  __shared__ uint32_t wsa[32], wsp[32];
  const int t = threadIdx.x;
  uint64_t code[kSmallPer];
  double bd[kSmallPer];
  uint32_t live = 0, pr = 0, na = 0, np = 0;
#pragma unroll
  for (int q = 0; q < kSmallPer; ++q) {
    const int64_t x = (int64_t)t * kSmallPer + q;
    if (x < n_cand) {
      bool lv, p;
      prune_classify(parents, x, root, ta, a_sym, tb, b_sym, b_transposed, upper, tau_l, &code[q], &bd[q], &lv, &p);
      live |= (uint32_t)lv << q;
      pr |= (uint32_t)p << q;
    }
  }
  na = __popc(live);
  np = __popc(pr);
  const int lane = t & 31, warp = t >> 5;
  uint32_t ia = na, ip = np;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t xa = __shfl_up_sync(0xffffffffu, ia, o), xp = __shfl_up_sync(0xffffffffu, ip, o);
    if (lane >= o) {
      ia += xa;
      ip += xp;
    }
  }
  if (lane == 31) {
    wsa[warp] = ia;
    wsp[warp] = ip;
  }
  __syncthreads();
  uint32_t ba = 0, bp = 0, tot_a = 0, tot_p = 0;
  for (int w = 0; w < kSmallThreads / 32; ++w) {
    if (w < warp) {
      ba += wsa[w];
      bp += wsp[w];
    }
    tot_a += wsa[w];
    tot_p += wsp[w];
  }
  uint32_t oa = ba + ia - na, op = bp + ip - np;
#pragma unroll
  for (int q = 0; q < kSmallPer; ++q) {
    if (live & (1u << q)) alive_out[oa++] = code[q];
    if (pr & (1u << q)) pruned_out[op++] = bd[q];
  }
  __syncthreads();
  if (t == 0) {
    __threadfence();
    host_cnt[0] = tot_a;
    host_cnt[1] = tot_p;
    __threadfence_system();
  }
}

// ---- every level in one launch ----------------------------------------------------------------
// The whole pruned recursion as one cooperative (grid-synchronised) kernel: level l's candidates are
// the 8 children of level l-1's survivors; survivors and prune bounds are appended with
// warp-aggregated atomics (the order of both lists is immaterial: the leaf pairs are sorted
// afterwards and the prune log is a multiset, engine.py:273-275), then one grid-wide barrier
// separates the levels. No host round trip between levels.
constexpr int kMaxLevels = 22;
struct PruneTables {
  Table a[kMaxLevels], b[kMaxLevels];
  double tau[kMaxLevels];  // tau_l = tau / 8^l, computed on the host exactly as the reference does
};

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__global__ void __launch_bounds__(256) k_prune_all(const __grid_constant__ PruneTables t, int depth, int a_sym,
                                                   int b_sym, int b_transposed, int upper, uint64_t *ping,
                                                   uint64_t *pong, uint64_t *leaf_out, int64_t cap,
                                                   double *log_out, int64_t cap_log,
                                                   unsigned long long *cnt /* [2*(depth+1)] */,
                                                   unsigned long long *log_cnt, unsigned int *overflow) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const uint64_t *par = nullptr;
  int64_t n_par = 0;
  for (int lev = 0; lev <= depth; ++lev) {
    const int root = lev == 0;
    const int64_t n_cand = root ? 1 : 8 * n_par;
    uint64_t *out = lev == depth ? leaf_out : ((lev & 1) ? pong : ping);
    // grid-stride with whole warps active (warp-aggregated appends)
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n_cand; base += nthreads) {
      const int64_t x = base + lane;
      uint64_t code = 0;
      double bd = 0.0;
      bool live = false, pr = false;
      if (x < n_cand)
        prune_classify(par, x, root, t.a[lev], a_sym, t.b[lev], b_sym, b_transposed, upper, t.tau[lev], &code, &bd,
                       &live, &pr);
      const uint32_t ml = __ballot_sync(0xffffffffu, live), mp = __ballot_sync(0xffffffffu, pr);
      unsigned long long bl = 0, bp = 0, bg = 0;
      if (lane == 0) {
        if (ml) bl = atomicAdd(&cnt[2 * lev], (unsigned long long)__popc(ml));
        if (mp) {
          bp = atomicAdd(&cnt[2 * lev + 1], (unsigned long long)__popc(mp));
          bg = atomicAdd(log_cnt, (unsigned long long)__popc(mp));
        }
      }
      bl = __shfl_sync(0xffffffffu, bl, 0);
      bg = __shfl_sync(0xffffffffu, bg, 0);
      (void)bp;
      if (live) {
        const unsigned long long pos = bl + __popc(ml & lanemask_lt());
        if ((int64_t)pos < cap) out[pos] = code; else atomicOr(overflow, 1u);
      }
      if (pr) {
        const unsigned long long pos = bg + __popc(mp & lanemask_lt());
        if ((int64_t)pos < cap_log) log_out[pos] = bd; else atomicOr(overflow, 2u);
      }
    }
    grid.sync();
    const int64_t alive = (int64_t)((volatile unsigned long long *)cnt)[2 * lev];
    n_par = alive < cap ? alive : cap;
    par = out;
    if (n_par == 0) break;  // every thread reads the same count: a uniform exit
  }
}

size_t select_bytes(int64_t n) {
  size_t a = 0, b = 0;
  cub::DeviceSelect::Flagged(nullptr, a, (uint64_t *)nullptr, (uint8_t *)nullptr, (uint64_t *)nullptr,
                             (int64_t *)nullptr, n);
  cub::DeviceSelect::Flagged(nullptr, b, (double *)nullptr, (uint8_t *)nullptr, (double *)nullptr,
                             (int64_t *)nullptr, n);
  return std::max(a, b);
}

size_t scan_bytes(int64_t n) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t *)nullptr, (int64_t *)nullptr, n);
  return b;
}

}  // namespace
}  // namespace qm

using namespace qm;

extern "C" size_t qm_node_norms_workspace_bytes(int64_t n) {
  Carver cv(nullptr, 0);
  cv.take<int64_t>(n + 1);  // head
  cv.take<int64_t>(n + 1);  // pos
  cv.take<int64_t>(n + 1);  // start
  cv.take<char>(scan_bytes(n + 1));
  return cv.off;
}

extern "C" int qm_node_norms(const qm_layout *layout, const uint64_t *keys, const double *sumsq, int64_t n,
                             uint64_t *codes, double *norms, int64_t *counts, void *ws, size_t ws_bytes,
                             void *stream) {
  Geometry g;
  int rc = make_geometry(layout, &g);
  if (rc != QM_OK) return rc;
  if (n < 0 || !counts || (n > 0 && (!keys || !sumsq || !codes || !norms))) {
    set_error("qm_node_norms: bad arguments");
    return QM_ERR_INVALID;
  }
  if (g.depth >= kPairBits) {
    set_error("qm_node_norms: depth %d exceeds %d", g.depth, kPairBits - 1);
    return QM_ERR_UNSUPPORTED;
  }
  Carver cv(ws, ws_bytes);
  int64_t *head = cv.take<int64_t>(n + 1), *pos = cv.take<int64_t>(n + 1), *start = cv.take<int64_t>(n + 1);
  const size_t sb = scan_bytes(n + 1);
  void *cub = cv.take<char>(sb);
  if (!cv.ok() || !ws) {
    set_error("qm_node_norms: workspace %zu < required %zu", ws_bytes, cv.off);
    return QM_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  // Level L (root 0 .. depth) occupies codes/norms [L*n, L*n + counts[L]); built bottom-up: the
  // leaves from the blocks (code = key >> 2*lbits), every level above from the one below (>> 2).
  const uint64_t *in = keys;
  const double *vals = sumsq;
  int64_t n_in = n;
  int shift = 2 * g.lbits, from_sumsq = 1;
  for (int L = g.depth; L >= 0; --L) {
    if (n_in == 0) {
      counts[L] = 0;
      continue;
    }
    uint64_t *oc = codes + (size_t)L * n;
    double *on = norms + (size_t)L * n;
    k_run_heads<<<grid_for(n_in + 1), 256, 0, st>>>(in, n_in, shift, head);
    QM_LAUNCHED("k_run_heads");
    size_t tb = sb;
    QM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(cub, tb, head, pos, n_in + 1, st));
    k_run_starts<<<grid_for(n_in), 256, 0, st>>>(in, n_in, shift, head, pos, oc, start);
    QM_LAUNCHED("k_run_starts");
    int64_t runs = 0;
    rc = read_device_i64(pos + n_in, 1, &runs, st);
    if (rc != QM_OK) return rc;
    k_run_norms<<<grid_for(runs), 256, 0, st>>>(vals, from_sumsq, n_in, start, runs, on);
    QM_LAUNCHED("k_run_norms");
    counts[L] = runs;
    in = oc;
    vals = on;
    n_in = runs;
    shift = 2;
    from_sumsq = 0;
  }
  return QM_OK;
}

extern "C" size_t qm_prune_level_workspace_bytes(int64_t n_parents) {
  const int64_t n = std::max<int64_t>(n_parents * 8, 1);
  Carver cv(nullptr, 0);
  cv.take<uint64_t>(n);  // candidates
  cv.take<double>(n);    // bounds
  cv.take<uint8_t>(n);   // alive
  cv.take<uint8_t>(n);   // pruned
  cv.take<int64_t>(2);   // selected counts
  cv.take<char>(select_bytes(n));
  return cv.off;
}

extern "C" int qm_prune_level(const qm_layout *layout, int32_t level, double tau_l, const uint64_t *parents,
                              int64_t n_parents, const uint64_t *a_codes, const double *a_norms,
                              int64_t a_count, int32_t a_sym, const uint64_t *b_codes, const double *b_norms,
                              int64_t b_count, int32_t b_sym, int32_t b_transposed, int32_t upper,
                              uint64_t *alive_out, double *pruned_out, int64_t *n_alive, int64_t *n_pruned,
                              void *ws, size_t ws_bytes, void *stream) {
  Geometry g;
  int rc = make_geometry(layout, &g);
  if (rc != QM_OK) return rc;
  if (level < 0 || level > g.depth || n_parents < 0 || !n_alive || !n_pruned || (level > 0 && n_parents == 0)) {
    set_error("qm_prune_level: bad arguments");
    return QM_ERR_INVALID;
  }
  const int root = level == 0;
  const int64_t n_cand = root ? 1 : n_parents * 8;
  if (n_cand <= kSmallLevelMax) {  // one launch, counts through mapped memory
    int64_t *host_cnt = nullptr, *dev_cnt = nullptr;
    rc = mapped_i64(&host_cnt, &dev_cnt);
    if (rc != QM_OK) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    Table ta{a_codes, a_norms, a_count}, tb{b_codes, b_norms, b_count};
    k_prune_small<<<1, kSmallThreads, 0, st>>>(parents, n_cand, root, ta, a_sym, tb, b_sym, b_transposed, upper,
                                                tau_l, alive_out, pruned_out, dev_cnt);
    QM_LAUNCHED("k_prune_small");
    QM_CUDA_TRY(cudaStreamSynchronize(st));
    *n_alive = ((volatile int64_t *)host_cnt)[0];
    *n_pruned = ((volatile int64_t *)host_cnt)[1];
    return QM_OK;
  }
  Carver cv(ws, ws_bytes);
  const int64_t cap = std::max<int64_t>(n_cand, 1);
  uint64_t *cand = cv.take<uint64_t>(cap);
  double *bound = cv.take<double>(cap);
  uint8_t *alive = cv.take<uint8_t>(cap), *pruned = cv.take<uint8_t>(cap);
  int64_t *sel = cv.take<int64_t>(2);
  const size_t sb = select_bytes(cap);
  void *cub = cv.take<char>(sb);
  if (!cv.ok() || !ws) {
    set_error("qm_prune_level: workspace %zu < required %zu", ws_bytes, cv.off);
    return QM_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  Table ta{a_codes, a_norms, a_count}, tb{b_codes, b_norms, b_count};
  k_prune_expand<<<grid_for(n_cand), 256, 0, st>>>(parents, n_cand, root, ta, a_sym, tb, b_sym, b_transposed,
                                                   upper, tau_l, cand, bound, alive, pruned);
  QM_LAUNCHED("k_prune_expand");
  size_t t1 = sb;
  QM_CUDA_TRY(cub::DeviceSelect::Flagged(cub, t1, cand, alive, alive_out, sel, n_cand, st));
  size_t t2 = sb;
  QM_CUDA_TRY(cub::DeviceSelect::Flagged(cub, t2, bound, pruned, pruned_out, sel + 1, n_cand, st));
  int64_t cnt[2];
  rc = read_device_i64(sel, 2, cnt, st);
  if (rc != QM_OK) return rc;
  *n_alive = cnt[0];
  *n_pruned = cnt[1];
  return QM_OK;
}

// ---- filter of the symbolic plan by the surviving leaf pairs -----------------------------------

namespace qm {
namespace {

// keep[t] = leaf pair (li, lk, lj) of triple t survived; code = (li*w + lk)*w + lj.
__global__ void k_filter_keep(const uint2 *tri, int64_t nT, const uint64_t *a_keys, const uint64_t *b_keys,
                              int b_transposed, int nbl, int lbits, int depth, const uint64_t *pairs,
                              int64_t n_pairs, int64_t *keep) {
  const uint64_t w = 1ull << depth;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= nT; t += (int64_t)gridDim.x * blockDim.x) {
    if (t == nT) {
      keep[t] = 0;  // exclusive-scan tail
      continue;
    }
    uint32_t ai, ak, bk, bj;
    qkey_decode(a_keys[tri[t].x], nbl, lbits, &ai, &ak);
    qkey_decode(b_keys[tri[t].y], nbl, lbits, &bk, &bj);
    if (b_transposed) bj = bk;
    const uint64_t code = ((uint64_t)(ai / nbl) * w + ak / nbl) * w + bj / nbl;
    int64_t lo = 0, hi = n_pairs;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (pairs[mid] < code) lo = mid + 1; else hi = mid;
    }
    keep[t] = (lo < n_pairs && pairs[lo] == code) ? 1 : 0;
  }
}

// cnt[c] = kept triples of C block c; alive[c] = cnt[c] > 0; tails 0.
__global__ void k_filter_count(const int64_t *tptr, int64_t nC, const int64_t *keep, int64_t *cnt,
                               int64_t *alive) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= nC; c += (int64_t)gridDim.x * blockDim.x) {
    if (c == nC) {
      cnt[c] = 0;
      alive[c] = 0;
      continue;
    }
    int64_t s = 0;
    for (int64_t t = tptr[c]; t < tptr[c + 1]; ++t) s += keep[t];
    cnt[c] = s;
    alive[c] = s > 0 ? 1 : 0;
  }
}

__global__ void k_filter_scatter_tri(const uint2 *tri, int64_t nT, const int64_t *keep, const int64_t *kpos,
                                     uint2 *tri_out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nT; t += (int64_t)gridDim.x * blockDim.x)
    if (keep[t]) tri_out[kpos[t]] = tri[t];
}

__global__ void k_filter_scatter_c(const uint64_t *c_keys, int64_t nC, const int64_t *alive, const int64_t *apos,
                                   const int64_t *cpos, uint64_t *keys_out, int64_t *tptr_out) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= nC; c += (int64_t)gridDim.x * blockDim.x) {
    if (c == nC) {
      tptr_out[apos[nC]] = cpos[nC];
    } else if (alive[c]) {
      keys_out[apos[c]] = c_keys[c];
      tptr_out[apos[c]] = cpos[c];
    }
  }
}

}  // namespace
}  // namespace qm

extern "C" size_t qm_filter_triples_workspace_bytes(int64_t nC, int64_t nT) {
  Carver cv(nullptr, 0);
  cv.take<int64_t>(nT + 1);  // keep
  cv.take<int64_t>(nT + 1);  // kpos
  cv.take<int64_t>(nC + 1);  // cnt
  cv.take<int64_t>(nC + 1);  // alive
  cv.take<int64_t>(nC + 1);  // cpos
  cv.take<int64_t>(nC + 1);  // apos
  cv.take<char>(std::max(scan_bytes(nT + 1), scan_bytes(nC + 1)));
  return cv.off;
}

namespace qm {
namespace {
// Compaction of a symbolic plan by per-triple keep flags (keep[nT] = 0 tail set by the caller's
// keep kernel): C blocks left without triples vanish, order preserved; counts to the host.
int filter_compact(const uint2 *t2, const int64_t *c_tptr, const uint64_t *c_keys, int64_t nC, int64_t nT,
                   int64_t *keep, int64_t *kpos, int64_t *cnt, int64_t *alive, int64_t *cpos, int64_t *apos,
                   void *cub, size_t sb, uint32_t *tri_out, int64_t *c_tptr_out, uint64_t *c_keys_out,
                   int64_t *nC_out, int64_t *nT_out, cudaStream_t st) {
  k_filter_count<<<grid_for(nC + 1), 256, 0, st>>>(c_tptr, nC, keep, cnt, alive);
  QM_LAUNCHED("k_filter_count");
  size_t tb = sb;
  QM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(cub, tb, keep, kpos, nT + 1, st));
  tb = sb;
  QM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(cub, tb, cnt, cpos, nC + 1, st));
  tb = sb;
  QM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(cub, tb, alive, apos, nC + 1, st));
  k_filter_scatter_tri<<<grid_for(nT), 256, 0, st>>>(t2, nT, keep, kpos, (uint2 *)tri_out);
  QM_LAUNCHED("k_filter_scatter_tri");
  k_filter_scatter_c<<<grid_for(nC + 1), 256, 0, st>>>(c_keys, nC, alive, apos, cpos, c_keys_out, c_tptr_out);
  QM_LAUNCHED("k_filter_scatter_c");
  int64_t counts[2];
  int rc = read_device_i64(apos + nC, 1, counts, st, kpos + nT);
  if (rc != QM_OK) return rc;
  *nC_out = counts[0];
  *nT_out = counts[1];
  return QM_OK;
}

// out[l*n + m] = norm of the level-l ancestor node of entry m (key -> leaf coordinates >> (depth-l);
// sym: a lower node reads its stored upper mirror), looked up in that level's node table.
__global__ void k_ancestor_norms(const uint64_t *keys, int64_t n, int nbl, int lbits, int depth,
                                 const __grid_constant__ PruneTables t, int sym, double *out) {
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n; m += (int64_t)gridDim.x * blockDim.x) {
    uint32_t bi, bj;
    qkey_decode(keys[m], nbl, lbits, &bi, &bj);
    const uint32_t li = bi / (uint32_t)nbl, lj = bj / (uint32_t)nbl;
    for (int l = 0; l <= depth; ++l) {
      double v = 0.0;
      lookup(t.a[l], li >> (depth - l), lj >> (depth - l), sym != 0, &v);
      out[(size_t)l * n + m] = v;
    }
  }
}

// keep[t]: no ancestor pair of triple t was pruned -- norm(A anc_l) * norm(B anc_l) >= tau_l at every
// level l (the reference prunes a task when the product is < tau_l, ops.py:199-204, 232; a leaf
// product survives iff none of its ancestor tasks was pruned, and its ancestors' nodes all exist).
__global__ void k_keep_by_norms(const uint2 *tri, int64_t nT, const double *anc_a, int64_t nA, const double *anc_b,
                                int64_t nB, int depth, const __grid_constant__ PruneTables t, int64_t *keep) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x <= nT; x += (int64_t)gridDim.x * blockDim.x) {
    if (x == nT) {
      keep[x] = 0;  // exclusive-scan tail
      continue;
    }
    const uint32_t a = tri[x].x & 0x7FFFFFFFu, b = tri[x].y & 0x7FFFFFFFu;
    int64_t k = 1;
    for (int l = 0; l <= depth; ++l)
      if (anc_a[(size_t)l * nA + a] * anc_b[(size_t)l * nB + b] < t.tau[l]) {
        k = 0;
        break;
      }
    keep[x] = k;
  }
}
}  // namespace
}  // namespace qm

extern "C" int qm_filter_triples(const qm_layout *layout, const uint64_t *a_keys, const uint64_t *b_keys,
                                 int32_t b_transposed, const uint32_t *tri, const int64_t *c_tptr,
                                 const uint64_t *c_keys, int64_t nC, int64_t nT, const uint64_t *leaf_pairs,
                                 int64_t n_pairs, uint32_t *tri_out, int64_t *c_tptr_out, uint64_t *c_keys_out,
                                 int64_t *nC_out, int64_t *nT_out, void *ws, size_t ws_bytes, void *stream) {
  Geometry g;
  int rc = make_geometry(layout, &g);
  if (rc != QM_OK) return rc;
  if (nC < 0 || nT < 0 || n_pairs < 0 || !nC_out || !nT_out) {
    set_error("qm_filter_triples: bad arguments");
    return QM_ERR_INVALID;
  }
  Carver cv(ws, ws_bytes);
  int64_t *keep = cv.take<int64_t>(nT + 1), *kpos = cv.take<int64_t>(nT + 1);
  int64_t *cnt = cv.take<int64_t>(nC + 1), *alive = cv.take<int64_t>(nC + 1);
  int64_t *cpos = cv.take<int64_t>(nC + 1), *apos = cv.take<int64_t>(nC + 1);
  const size_t sb = std::max(scan_bytes(nT + 1), scan_bytes(nC + 1));
  void *cub = cv.take<char>(sb);
  if (!cv.ok() || !ws) {
    set_error("qm_filter_triples: workspace %zu < required %zu", ws_bytes, cv.off);
    return QM_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const uint2 *t2 = (const uint2 *)tri;
  k_filter_keep<<<grid_for(nT + 1), 256, 0, st>>>(t2, nT, a_keys, b_keys, b_transposed, g.nbl, g.lbits, g.depth,
                                                  leaf_pairs, n_pairs, keep);
  QM_LAUNCHED("k_filter_keep");
  return filter_compact(t2, c_tptr, c_keys, nC, nT, keep, kpos, cnt, alive, cpos, apos, cub, sb, tri_out,
                        c_tptr_out, c_keys_out, nC_out, nT_out, st);
}

extern "C" int qm_ancestor_norms(const qm_layout *layout, const uint64_t *keys, int64_t n, const uint64_t *codes,
                                 const double *norms, int64_t stride, const int64_t *counts, int32_t sym,
                                 double *out, void *stream) {
  Geometry g;
  int rc = make_geometry(layout, &g);
  if (rc != QM_OK) return rc;
  if (n < 0 || !counts || (n > 0 && (!keys || !codes || !norms || !out))) {
    set_error("qm_ancestor_norms: bad arguments");
    return QM_ERR_INVALID;
  }
  if (g.depth + 1 > kMaxLevels) {
    set_error("qm_ancestor_norms: depth %d exceeds %d", g.depth, kMaxLevels - 1);
    return QM_ERR_UNSUPPORTED;
  }
  if (n == 0) return QM_OK;
  PruneTables t;
  memset(&t, 0, sizeof(t));
  for (int l = 0; l <= g.depth; ++l) t.a[l] = Table{codes + (size_t)l * stride, norms + (size_t)l * stride, counts[l]};
  cudaStream_t st = (cudaStream_t)stream;
  k_ancestor_norms<<<grid_for(n), 256, 0, st>>>(keys, n, g.nbl, g.lbits, g.depth, t, sym, out);
  QM_LAUNCHED("k_ancestor_norms");
  return QM_OK;
}

extern "C" int qm_filter_triples_norms(const qm_layout *layout, double tau, const uint32_t *tri, const int64_t *c_tptr,
                                       const uint64_t *c_keys, int64_t nC, int64_t nT, const double *anc_a,
                                       int64_t nA, const double *anc_b, int64_t nB, uint32_t *tri_out,
                                       int64_t *c_tptr_out, uint64_t *c_keys_out, int64_t *nC_out, int64_t *nT_out,
                                       void *ws, size_t ws_bytes, void *stream) {
  Geometry g;
  int rc = make_geometry(layout, &g);
  if (rc != QM_OK) return rc;
  if (nC < 0 || nT < 0 || !nC_out || !nT_out || (nT > 0 && (!anc_a || !anc_b))) {
    set_error("qm_filter_triples_norms: bad arguments");
    return QM_ERR_INVALID;
  }
  if (g.depth + 1 > kMaxLevels) {
    set_error("qm_filter_triples_norms: depth %d exceeds %d", g.depth, kMaxLevels - 1);
    return QM_ERR_UNSUPPORTED;
  }
  Carver cv(ws, ws_bytes);
  int64_t *keep = cv.take<int64_t>(nT + 1), *kpos = cv.take<int64_t>(nT + 1);
  int64_t *cnt = cv.take<int64_t>(nC + 1), *alive = cv.take<int64_t>(nC + 1);
  int64_t *cpos = cv.take<int64_t>(nC + 1), *apos = cv.take<int64_t>(nC + 1);
  const size_t sb = std::max(scan_bytes(nT + 1), scan_bytes(nC + 1));
  void *cub = cv.take<char>(sb);
  if (!cv.ok() || !ws) {
    set_error("qm_filter_triples_norms: workspace %zu < required %zu", ws_bytes, cv.off);
    return QM_ERR_WORKSPACE;
  }
  PruneTables t;
  memset(&t, 0, sizeof(t));
  for (int l = 0; l <= g.depth; ++l) t.tau[l] = tau / ldexp(1.0, 3 * l);  // tau / 8.0**l (ops.py:232)
  cudaStream_t st = (cudaStream_t)stream;
  const uint2 *t2 = (const uint2 *)tri;
  k_keep_by_norms<<<grid_for(nT + 1), 256, 0, st>>>(t2, nT, anc_a, nA, anc_b, nB, g.depth, t, keep);
  QM_LAUNCHED("k_keep_by_norms");
  return filter_compact(t2, c_tptr, c_keys, nC, nT, keep, kpos, cnt, alive, cpos, apos, cub, sb, tri_out,
                        c_tptr_out, c_keys_out, nC_out, nT_out, st);
}

extern "C" size_t qm_prune_all_workspace_bytes(int64_t cap_pairs) {
  Carver cv(nullptr, 0);
  cv.take<uint64_t>(std::max<int64_t>(cap_pairs, 1));  // ping
  cv.take<uint64_t>(std::max<int64_t>(cap_pairs, 1));  // pong
  cv.take<unsigned long long>(2 * kMaxLevels + 2);      // counters, log count, overflow
  return cv.off;
}

extern "C" int qm_prune_all(const qm_layout *layout, double tau, const uint64_t *a_codes, const double *a_norms,
                            int64_t a_stride, const int64_t *a_counts, int32_t a_sym, const uint64_t *b_codes,
                            const double *b_norms, int64_t b_stride, const int64_t *b_counts, int32_t b_sym,
                            int32_t b_transposed, int32_t upper, int64_t cap_pairs, uint64_t *leaf_pairs_out,
                            double *log_out, int64_t cap_log, int64_t *counts_out, void *ws, size_t ws_bytes,
                            void *stream) {
  Geometry g;
  int rc = make_geometry(layout, &g);
  if (rc != QM_OK) return rc;
  if (!a_codes || !a_norms || !a_counts || !b_codes || !b_norms || !b_counts || !counts_out || cap_pairs < 1 ||
      cap_log < 1 || !leaf_pairs_out || !log_out) {
    set_error("qm_prune_all: bad arguments");
    return QM_ERR_INVALID;
  }
  if (g.depth + 1 > kMaxLevels || g.depth >= kPairBits) {
    set_error("qm_prune_all: depth %d exceeds %d", g.depth, kMaxLevels - 1);
    return QM_ERR_UNSUPPORTED;
  }
  Carver cv(ws, ws_bytes);
  uint64_t *ping = cv.take<uint64_t>(cap_pairs), *pong = cv.take<uint64_t>(cap_pairs);
  unsigned long long *ctr = cv.take<unsigned long long>(2 * kMaxLevels + 2);
  if (!cv.ok() || !ws) {
    set_error("qm_prune_all: workspace %zu < required %zu", ws_bytes, cv.off);
    return QM_ERR_WORKSPACE;
  }
  PruneTables t;
  memset(&t, 0, sizeof(t));
  for (int l = 0; l <= g.depth; ++l) {
    t.a[l] = Table{a_codes + (size_t)l * a_stride, a_norms + (size_t)l * a_stride, a_counts[l]};
    t.b[l] = Table{b_codes + (size_t)l * b_stride, b_norms + (size_t)l * b_stride, b_counts[l]};
    t.tau[l] = tau / ldexp(1.0, 3 * l);  // tau / 8.0**l (ops.py:232), exact power-of-two scaling
  }
  cudaStream_t st = (cudaStream_t)stream;
  QM_CUDA_TRY(cudaMemsetAsync(ctr, 0, (2 * kMaxLevels + 2) * sizeof(unsigned long long), st));
  static PerDeviceInt occupancy;
  int per_sm = 0;
  rc = occupancy.get(&per_sm, [](int *x) -> int {
    QM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(x, k_prune_all, 256, 0));
    return (int)QM_OK;
  });
  if (rc != QM_OK) return rc;
  const int grid = device_sm_count() * std::max(1, std::min(per_sm, 4));
  int depth = g.depth;
  unsigned long long *cnt = ctr, *log_cnt = ctr + 2 * kMaxLevels;
  unsigned int *overflow = (unsigned int *)(ctr + 2 * kMaxLevels + 1);
  void *args[] = {(void *)&t,   (void *)&depth,   (void *)&a_sym,          (void *)&b_sym,  (void *)&b_transposed,
                  (void *)&upper, (void *)&ping, (void *)&pong,          (void *)&leaf_pairs_out, (void *)&cap_pairs,
                  (void *)&log_out, (void *)&cap_log, (void *)&cnt, (void *)&log_cnt, (void *)&overflow};
  QM_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)k_prune_all, grid, 256, args, 0, st));
  QM_LAUNCHED("k_prune_all");
  // counts_out (host): [alive_0, pruned_0, ..., alive_depth, pruned_depth, log total, overflow]
  unsigned long long host[2 * kMaxLevels + 2];
  QM_CUDA_TRY(cudaMemcpyAsync(host, ctr, sizeof(host), cudaMemcpyDeviceToHost, st));
  QM_CUDA_TRY(cudaStreamSynchronize(st));
  for (int l = 0; l <= g.depth; ++l) {
    counts_out[2 * l] = (int64_t)host[2 * l];
    counts_out[2 * l + 1] = (int64_t)host[2 * l + 1];
  }
  counts_out[2 * (g.depth + 1)] = (int64_t)host[2 * kMaxLevels];
  counts_out[2 * (g.depth + 1) + 1] = (int64_t)(unsigned int)host[2 * kMaxLevels + 1];
  return QM_OK;
}

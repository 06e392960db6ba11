// Staging plan of one rank of a multi-GPU product (qm_stage_plan): which of the rank's operand
// references are owned by a peer, the distinct peer blocks it must gather (its halo), its triples
// re-indexed into [local pool | halo pool], and the claim order that puts the C blocks needing no
// halo first -- all on the device, so the host reads three counts and launches the staged numeric
// phase (qm_numeric_pools_ex). The reference's analogue is the transfer layer's per-worker fetch
// of remote chunks (TransferSim.fetch, chunkstore.py:188-210), here done once per distinct block.
#include <cub/cub.cuh>

#include "qm_common.cuh"

namespace qm {
namespace {

constexpr uint32_t kHaloBit = 1u << 28;  // qm_numeric_pools_ex pool 1 (the halo)

inline int stage_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

// Marks every peer-owned block a triple references (flags are idempotent byte-wide writes).
__global__ void k_stage_mark(const uint2 *tri, int64_t nT, int64_t a_lo, int64_t a_hi, int64_t b_lo, int64_t b_hi,
                             uint32_t *flag_a, uint32_t *flag_b) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nT; t += (int64_t)gridDim.x * blockDim.x) {
    const uint2 ab = tri[t];
    if ((int64_t)ab.x < a_lo || (int64_t)ab.x >= a_hi) flag_a[ab.x] = 1u;
    if ((int64_t)ab.y < b_lo || (int64_t)ab.y >= b_hi) flag_b[ab.y] = 1u;
  }
}

// Halo lists: index g is the pos[g]-th distinct peer block (ascending g).
__global__ void k_stage_halo(const uint32_t *flag, const uint32_t *pos, int64_t n, uint32_t *halo) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x)
    if (flag[g]) halo[pos[g]] = (uint32_t)g;
}

// Per C block: its triples re-indexed (local index, or halo bit | halo position) and whether any
// of them needs the halo.
__global__ void k_stage_pack(const uint2 *tri, const int64_t *tptr, int64_t nC, int64_t a_lo, int64_t a_hi,
                             int64_t b_lo, int64_t b_hi, const uint32_t *pos_a, const uint32_t *pos_b, uint2 *packed,
                             uint32_t *need) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nC; c += (int64_t)gridDim.x * blockDim.x) {
    uint32_t any = 0;
    for (int64_t t = tptr[c]; t < tptr[c + 1]; ++t) {
      const uint2 ab = tri[t];
      const bool ra = (int64_t)ab.x < a_lo || (int64_t)ab.x >= a_hi;
      const bool rb = (int64_t)ab.y < b_lo || (int64_t)ab.y >= b_hi;
      packed[t] = make_uint2(ra ? (kHaloBit | pos_a[ab.x]) : (uint32_t)((int64_t)ab.x - a_lo),
                             rb ? (kHaloBit | pos_b[ab.y]) : (uint32_t)((int64_t)ab.y - b_lo));
      any |= (uint32_t)(ra || rb);
    }
    need[c] = any;
  }
}

// Stable partition of the C blocks: local-only ones (in key order) then the others.
__global__ void k_stage_order(const uint32_t *need, const uint32_t *npos, int64_t nC, uint32_t *order,
                              int64_t *counts) {
  const int64_t n_need = (int64_t)npos[nC];
  const int64_t n_local = nC - n_need;
  if (blockIdx.x == 0 && threadIdx.x == 0) counts[0] = n_local;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nC; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = need[c] ? n_local + npos[c] : c - npos[c];
    order[p] = (uint32_t)c;
  }
}

// Halo counts next to n_local (the totals of the exclusive scans).
__global__ void k_stage_counts(const uint32_t *pos_a, const uint32_t *flag_a, int64_t nA, const uint32_t *pos_b,
                               const uint32_t *flag_b, int64_t nB, int b_is_a, int64_t *counts) {
  if (threadIdx.x != 0) return;
  counts[1] = nA ? (int64_t)pos_a[nA - 1] + flag_a[nA - 1] : 0;
  counts[2] = b_is_a ? 0 : (nB ? (int64_t)pos_b[nB - 1] + flag_b[nB - 1] : 0);
}

struct StageWs {
  uint32_t *flag_a, *pos_a, *flag_b, *pos_b, *need, *npos;
  int64_t *counts;
  void *cub;
  size_t cub_bytes;
};

size_t stage_cub_bytes(int64_t n) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (uint32_t *)nullptr, (uint32_t *)nullptr, std::max<int64_t>(n, 1));
  return b;
}

StageWs carve_stage(Carver &cv, int64_t nA, int64_t nB, int64_t nC, int b_is_a) {
  StageWs w;
  w.flag_a = cv.take<uint32_t>(std::max<int64_t>(nA, 1));
  w.pos_a = cv.take<uint32_t>(std::max<int64_t>(nA, 1));
  w.flag_b = b_is_a ? w.flag_a : cv.take<uint32_t>(std::max<int64_t>(nB, 1));
  w.pos_b = b_is_a ? w.pos_a : cv.take<uint32_t>(std::max<int64_t>(nB, 1));
  w.need = cv.take<uint32_t>(nC + 1);
  w.npos = cv.take<uint32_t>(nC + 1);
  w.counts = cv.take<int64_t>(4);
  w.cub_bytes = std::max(stage_cub_bytes(std::max(nA, nB)), stage_cub_bytes(nC + 1));
  w.cub = cv.take<char>(w.cub_bytes);
  return w;
}

}  // namespace
}  // namespace qm

using namespace qm;

extern "C" size_t qm_stage_plan_workspace_bytes(int64_t nA, int64_t nB, int64_t nC, int32_t b_is_a) {
  Carver cv(nullptr, 0);
  carve_stage(cv, nA, nB, nC, b_is_a);
  return cv.off;
}

extern "C" int qm_stage_plan(const uint32_t *tri, int64_t nT, const int64_t *c_tptr, int64_t nC, int64_t a_lo,
                             int64_t a_hi, int64_t nA, int64_t b_lo, int64_t b_hi, int64_t nB, int32_t b_is_a,
                             void *ws, size_t ws_bytes, uint32_t *tri_packed, uint32_t *order, uint32_t *halo_a,
                             uint32_t *halo_b, int64_t *counts_out, void *stream) {
  if (nT < 0 || nC < 0 || nA < 0 || nB < 0 || !counts_out || (nC > 0 && (!tri || !c_tptr || !tri_packed || !order)) ||
      a_lo < 0 || a_hi < a_lo || a_hi > nA || b_lo < 0 || b_hi < b_lo || b_hi > nB || (b_is_a && nA != nB) ||
      nA >= ((int64_t)1 << 28) || nB >= ((int64_t)1 << 28)) {
    set_error("qm_stage_plan: bad arguments");
    return QM_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  Carver cv(ws, ws_bytes);
  StageWs w = carve_stage(cv, nA, nB, nC, b_is_a);
  if (!cv.ok() || !ws) {
    set_error("qm_stage_plan: workspace %zu bytes < required %zu", ws_bytes, cv.off);
    return QM_ERR_WORKSPACE;
  }
  QM_CUDA_TRY(cudaMemsetAsync(w.flag_a, 0, sizeof(uint32_t) * std::max<int64_t>(nA, 1), st));
  if (!b_is_a) QM_CUDA_TRY(cudaMemsetAsync(w.flag_b, 0, sizeof(uint32_t) * std::max<int64_t>(nB, 1), st));
  if (nT > 0) {
    k_stage_mark<<<stage_grid(nT), 256, 0, st>>>((const uint2 *)tri, nT, a_lo, a_hi, b_lo, b_hi, w.flag_a,
                                                 w.flag_b);
    QM_LAUNCHED("k_stage_mark");
  }
  size_t tb = w.cub_bytes;
  if (nA > 0) QM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(w.cub, tb, w.flag_a, w.pos_a, nA, st));
  if (!b_is_a && nB > 0) {
    tb = w.cub_bytes;
    QM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(w.cub, tb, w.flag_b, w.pos_b, nB, st));
  }
  if (nA > 0 && halo_a) {
    k_stage_halo<<<stage_grid(nA), 256, 0, st>>>(w.flag_a, w.pos_a, nA, halo_a);
    QM_LAUNCHED("k_stage_halo");
  }
  if (!b_is_a && nB > 0 && halo_b) {
    k_stage_halo<<<stage_grid(nB), 256, 0, st>>>(w.flag_b, w.pos_b, nB, halo_b);
    QM_LAUNCHED("k_stage_halo");
  }
  k_stage_counts<<<1, 32, 0, st>>>(w.pos_a, w.flag_a, nA, w.pos_b, w.flag_b, nB, b_is_a, w.counts);
  QM_LAUNCHED("k_stage_counts");
  if (nC > 0) {
    k_stage_pack<<<stage_grid(nC), 256, 0, st>>>((const uint2 *)tri, c_tptr, nC, a_lo, a_hi, b_lo, b_hi, w.pos_a,
                                                 w.pos_b, (uint2 *)tri_packed, w.need);
    QM_LAUNCHED("k_stage_pack");
    QM_CUDA_TRY(cudaMemsetAsync(w.need + nC, 0, sizeof(uint32_t), st));
    tb = w.cub_bytes;
    QM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(w.cub, tb, w.need, w.npos, nC + 1, st));
    k_stage_order<<<stage_grid(nC), 256, 0, st>>>(w.need, w.npos, nC, order, w.counts);
    QM_LAUNCHED("k_stage_order");
  } else {
    QM_CUDA_TRY(cudaMemsetAsync(w.counts, 0, sizeof(int64_t), st));
  }
  return read_device_i64(w.counts, 3, counts_out, st);
}

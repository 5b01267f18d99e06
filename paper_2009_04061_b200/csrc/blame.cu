// blame.cu -- rows a2-a6: candidate pruning (rules 1-3), Eq. 1 shares for all and latency
// samples, self-attribution, Fig. 6 classification and the def-side reduction.
//
//   k_blame_tiles a warp per 32 use rows (a3, a4): rules 1-3 per in-edge, weights
//                 max(A_d,1)/max_len (Q1-Q4) with A_d summed from the def's count row,
//                 W summed in CSR order, shares w/W (Eq. 1), self flags when no
//                 candidate survives (Q5)
//   k_def_tiles   a warp per 32 defs over the create-time def-major transpose (a5, a6):
//                 S_j[r]*share and SL_j[r]*share summed into i's category
//                 (k_def_rows: a thread per def, for programs of 2^20 instructions and more)
// A_i and L_i themselves (a2): k_summaries for programs of 2^20 instructions and more (p.al_pre),
// else summed by the rollup tiles, which read every count row anyway.
// fp64 adds/multiplies use __dadd_rn/__dmul_rn (no FMA contraction), and every sum runs in
// CSR/edge order, so results match a sequential evaluation of the definitions exactly.
#include <algorithm>

#include "gpa_internal.cuh"

namespace gpa {
namespace {

// A_d = sum over reasons of the def's active samples ("issued samples", Q3), from
// its count row: the row is 2R u64 = R 16-byte units, the active half its first R u64.  Computed
// where the weight needs it (the gather of one def row per candidate edge) instead of in a separate
// pass over the whole table; an integer sum, exact in any order.
__device__ __forceinline__ uint64_t def_issue(const DevProgram &p, uint32_t d) {
  const uint4 *r4 = reinterpret_cast<const uint4 *>(p.C + (uint64_t)d * 2 * p.R);
  uint4 v[kReasonsMax / 2];
#pragma unroll
  for (uint32_t k = 0; k < kReasonsMax / 2; ++k)
    if (2 * k < p.R) v[k] = r4[k];
  uint64_t a = 0;
#pragma unroll
  for (uint32_t k = 0; k < kReasonsMax / 2; ++k) {
    if (2 * k < p.R) a += (uint64_t)v[k].y << 32 | v[k].x;
    if (2 * k + 1 < p.R) a += (uint64_t)v[k].w << 32 | v[k].z;
  }
  return a;
}

// A_i, L_i for every instruction (a2), one thread per row: a pass over the whole table that pays
// off only for large programs (p.al_pre, below)
__device__ __forceinline__ void body_summaries(const uint64_t *__restrict__ C, uint32_t n, uint32_t R,
                                               uint64_t *__restrict__ AL, uint32_t bx, uint32_t gx) {
  pdl_wait();
  for (uint32_t i = bx * blockDim.x + threadIdx.x; i < n; i += gx * blockDim.x) {
    const uint64_t *row = C + (uint64_t)i * 2 * R;
    uint64_t a = 0, l = 0;
    for (uint32_t r = 0; r < R; ++r) {
      a += row[r];
      l += row[R + r];
    }
    AL[2 * (uint64_t)i] = a;
    AL[2 * (uint64_t)i + 1] = l;
  }
}

__global__ void k_summaries(const uint64_t *__restrict__ C, uint32_t n, uint32_t R, uint64_t *__restrict__ AL) {
  body_summaries(C, n, R, AL, blockIdx.x, gridDim.x);
}

// A_d for the weight of an edge: from AL when k_summaries ran (large programs: the gather of one
// 8-byte word per edge), else summed from the def's count row (small programs: one dependent
// kernel fewer; on config 4 the 72-byte row gathers cost more than the pass, 2.21 -> 2.44 ms)
// (a template parameter, so that each instantiation issues only its own loads)
template <bool kPre>
__device__ __forceinline__ uint64_t def_A(const DevProgram &p, uint32_t d) {
  if (kPre) return p.AL[2 * (uint64_t)d];
  return def_issue(p, d);
}

// rule 1 (Q6): bit r-1 set when def class c may cause a stall of reason r
__device__ __forceinline__ uint32_t rule1_mask(uint32_t c) {
  const bool mem = c == OC_GLOBAL || c == OC_LOCAL || c == OC_CONSTANT || c == OC_TEXTURE;
  return (mem ? 1u : 0u) | 2u | (c == OC_SYNC ? 4u : 0u);
}

// Blame rows, warp-cooperative (north_star: "CSR edge-parallel ... warp-level ... pruning
// and normalisation"): a warp takes a tile of 32 use rows.  (1) lane = row: the live test from the
// row's dependency-reason counts; (2) lanes over the tile's edges (coalesced edge fields, the defs'
// latency / class / A_i gathered by 32 lanes at once): rules 1-3 and the weight of every edge, staged
// in shared memory; (3) lane = row: W per dependency reason summed over the row's edges in CSR order
// from shared memory (the sequential order of the definition, so shares stay bit-identical to a
// sequential evaluation), self flags; (4) lanes over edges again: shares w / W written coalesced.
// Tiles with more than kTileEdges edges fall back to a row-per-lane loop.
constexpr uint32_t kTileEdges = 256;
constexpr uint32_t kBlameWarps = 4;
struct BlameSmem {
  double sw[kBlameWarps][kTileEdges];
  double sW[kBlameWarps][3][32];
  uint8_t sm[kBlameWarps][kTileEdges];
  uint8_t slive[kBlameWarps][32];
};
template <bool kPre>
__device__ __forceinline__ void body_blame_tiles(DevProgram p, uint32_t bx, uint32_t gx) {
  pdl_wait();
  BlameSmem &S = dyn_smem<BlameSmem>();
  auto &sw = S.sw;
  auto &sm = S.sm;
  auto &sW = S.sW;
  auto &slive = S.slive;
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t n_tiles = (p.n + 31) / 32, warps = gx * kBlameWarps;
  double *w_ = sw[wib];
  uint8_t *m_ = sm[wib];
  for (uint32_t tile = bx * kBlameWarps + wib; tile < n_tiles; tile += warps) {
    const uint32_t j0 = tile * 32, j = j0 + lane;
    const bool in = j < p.n;
    const uint32_t E0 = p.row_ptr[j0], E1 = p.row_ptr[min(j0 + 32, p.n)];
    bool live = false;
    if (in) {
      const uint64_t *row = p.C + (uint64_t)j * 2 * p.R;
      live = (row[R_MEM] + row[p.R + R_MEM] + row[R_EXEC] + row[p.R + R_EXEC] + row[R_SYNC] + row[p.R + R_SYNC]) != 0;
    }
    if (E1 - E0 > kTileEdges) {   // rare: a long row -- lane-per-row, CSR order
      if (in) {
        const uint32_t e0 = p.row_ptr[j], e1 = p.row_ptr[j + 1];
        double W0 = 0.0, W1 = 0.0, W2 = 0.0;
        if (live)
          for (uint32_t e = e0; e < e1; ++e) {
            const uint32_t d = p.edge_def[e];
            const DefInfo di = p.dinfo[d];
            if (!(p.edge_dom[e] < 0 && p.edge_min[e] <= di.latency)) continue;
            const uint32_t m = rule1_mask(di.cls_flags & 0xffu);
            const uint64_t a = def_A<kPre>(p, d);
            const double w = __ddiv_rn((double)(a ? a : 1ull), (double)p.edge_max[e]);
            if (m & 1u) W0 = __dadd_rn(W0, w);
            W1 = __dadd_rn(W1, w);
            if (m & 4u) W2 = __dadd_rn(W2, w);
          }
        for (uint32_t e = e0; e < e1; ++e) {
          uint32_t m = 0;
          double w = 0.0;
          if (live) {
            const uint32_t d = p.edge_def[e];
            const DefInfo di = p.dinfo[d];
            if (p.edge_dom[e] < 0 && p.edge_min[e] <= di.latency) {
              m = rule1_mask(di.cls_flags & 0xffu);
              const uint64_t a = def_A<kPre>(p, d);
              w = __ddiv_rn((double)(a ? a : 1ull), (double)p.edge_max[e]);
            }
          }
          p.cand[e] = (uint8_t)m;
          p.share[3 * (uint64_t)e] = (m & 1u) ? __ddiv_rn(w, W0) : 0.0;
          p.share[3 * (uint64_t)e + 1] = m ? __ddiv_rn(w, W1) : 0.0;
          p.share[3 * (uint64_t)e + 2] = (m & 4u) ? __ddiv_rn(w, W2) : 0.0;
        }
        p.selfm[j] = live ? (uint8_t)((W0 > 0.0 ? 0u : 1u) | (W1 > 0.0 ? 0u : 2u) | (W2 > 0.0 ? 0u : 4u)) : 0;
      }
      continue;
    }
    slive[wib][lane] = live;
    __syncwarp();
    // (2) per edge: rules 1-3 and the weight, lanes over the tile's edges
    for (uint32_t e = E0 + lane; e < E1; e += 32) {
      const uint32_t u = p.edge_use[e];
      uint32_t m = 0;
      double w = 0.0;
      if (slive[wib][u - j0]) {
        const uint32_t d = p.edge_def[e], mn = p.edge_min[e], mx = p.edge_max[e];
        const int32_t dom = p.edge_dom[e];
        const DefInfo di = p.dinfo[d];
        const uint32_t lat = di.latency, cls = di.cls_flags & 0xffu;
        const uint64_t a = def_A<kPre>(p, d);
        if (dom < 0 && mn <= lat) {   // rules 2, 3
          m = rule1_mask(cls);
          w = __ddiv_rn((double)(a ? a : 1ull), (double)mx);
        }
      }
      w_[e - E0] = w;
      m_[e - E0] = (uint8_t)m;
    }
    __syncwarp();
    // (3) lane = row: W per reason in CSR order, self flags
    if (in) {
      double W0 = 0.0, W1 = 0.0, W2 = 0.0;
      if (live) {
        const uint32_t e0 = p.row_ptr[j] - E0, e1 = p.row_ptr[j + 1] - E0;
        for (uint32_t k = e0; k < e1; ++k) {
          const uint32_t m = m_[k];
          if (!m) continue;
          const double w = w_[k];
          if (m & 1u) W0 = __dadd_rn(W0, w);
          W1 = __dadd_rn(W1, w);
          if (m & 4u) W2 = __dadd_rn(W2, w);
        }
        p.selfm[j] = (uint8_t)((W0 > 0.0 ? 0u : 1u) | (W1 > 0.0 ? 0u : 2u) | (W2 > 0.0 ? 0u : 4u));
      } else {
        p.selfm[j] = 0;
      }
      sW[wib][0][lane] = W0;
      sW[wib][1][lane] = W1;
      sW[wib][2][lane] = W2;
    }
    __syncwarp();
    // (4) lanes over edges: candidate masks and shares
    for (uint32_t e = E0 + lane; e < E1; e += 32) {
      const uint32_t m = m_[e - E0], r = p.edge_use[e] - j0;
      const double w = w_[e - E0];
      p.cand[e] = (uint8_t)m;
      p.share[3 * (uint64_t)e] = (m & 1u) ? __ddiv_rn(w, sW[wib][0][r]) : 0.0;
      p.share[3 * (uint64_t)e + 1] = m ? __ddiv_rn(w, sW[wib][1][r]) : 0.0;
      p.share[3 * (uint64_t)e + 2] = (m & 4u) ? __ddiv_rn(w, sW[wib][2][r]) : 0.0;
    }
    __syncwarp();
  }
}

template <bool kPre>
__global__ void __launch_bounds__(32 * kBlameWarps) k_blame_tiles(DevProgram p) {
  body_blame_tiles<kPre>(p, blockIdx.x, gridDim.x);
}

// one lane per def (def_acc_one, gpa_internal.cuh), B stored
__device__ __forceinline__ void def_reduce_one(const DevProgram &p, uint32_t i) {
  double acc[4][2];
  def_acc_one(p, i, acc);
  store_B(p, i, acc);
}

// Warp-cooperative def reduction: a warp per tile of 32 consecutive defs (def_tile_acc,
// gpa_internal.cuh)
constexpr uint32_t kDefWarps = 4;
struct DefSmem {
  DefWarpSmem w[kDefWarps];
};
__device__ __forceinline__ void body_def_tiles(DevProgram p, uint32_t bx, uint32_t gx) {
  pdl_wait();
  DefSmem &S = dyn_smem<DefSmem>();
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t n_tiles = (p.n + 31) / 32, warps = gx * kDefWarps;
  for (uint32_t tile = bx * kDefWarps + wib; tile < n_tiles; tile += warps) {
    double acc[4][2];
    def_tile_acc(p, tile, lane, S.w[wib], acc);
  }
}

__global__ void __launch_bounds__(32 * kDefWarps) k_def_tiles(DevProgram p) {
  body_def_tiles(p, blockIdx.x, gridDim.x);
}

// the thread-per-def form, for large programs (launch_def_reduce)
__global__ void k_def_rows(DevProgram p) {
  pdl_wait();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += gridDim.x * blockDim.x) def_reduce_one(p, i);
}

inline uint32_t grid_for(uint64_t items, uint32_t threads, int n_sms) {
  return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((items + threads - 1) / threads, (uint64_t)n_sms * 16));
}

}  // namespace

#ifndef GPA_FUSED_TU
// candidates / shares / self flags (rows a3-a4): everything the estimate step reads
cudaError_t launch_blame_rows(const DevProgram &p, int n_sms, cudaStream_t s, uint64_t *launches) {
  if (p.al_pre) {
    k_summaries<<<grid_for(p.n, 256, n_sms), 256, 0, s>>>(p.C, p.n, p.R, p.AL);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    *launches += 1;
  }
  const uint32_t tiles = (p.n + 31) / 32;
  const uint32_t g = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((tiles + kBlameWarps - 1) / kBlameWarps,
                                                                        (uint64_t)n_sms * 16));
  const cudaError_t e = p.al_pre ? launch_pdl(p.n, k_blame_tiles<true>, g, 32 * kBlameWarps, sizeof(BlameSmem), s, p)
                                  : launch_pdl(p.n, k_blame_tiles<false>, g, 32 * kBlameWarps, sizeof(BlameSmem), s, p);
  *launches += 1;
  return e;
}

// def-side reduction (rows a5-a6): B, read by the rollup only
cudaError_t launch_def_reduce(const DevProgram &p, int n_sms, cudaStream_t s, uint64_t *launches) {
  // the warp-cooperative tiles for programs below kPdlMaxInstr instructions (config 3's analysis
  // 78 -> 74 us); on config 4 their 25 KB of staging per CTA slowed the estimate branch running
  // beside them (analysis 2.21 -> 2.37 ms), so large programs keep a thread per def
  if (p.n < kPdlMaxInstr) {
    const uint32_t tiles = (p.n + 31) / 32;
    const uint32_t g = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((tiles + kDefWarps - 1) / kDefWarps,
                                                                          (uint64_t)n_sms * 16));
    const cudaError_t e = launch_pdl(p.n, k_def_tiles, g, 32 * kDefWarps, sizeof(DefSmem), s, p);
    *launches += 1;
    return e;
  }
  const cudaError_t e = launch_pdl(p.n, k_def_rows, grid_for(p.n, 128, n_sms), 128, 0, s, p);
  *launches += 1;
  return e;
}

cudaError_t launch_blame(const DevProgram &p, int n_sms, cudaStream_t s, uint64_t *launches) {
  cudaError_t e = launch_blame_rows(p, n_sms, s, launches);
  return e != cudaSuccess ? e : launch_def_reduce(p, n_sms, s, launches);
}

#endif  // GPA_FUSED_TU

}  // namespace gpa

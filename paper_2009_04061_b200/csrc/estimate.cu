// estimate.cu -- row a8: optimizer matching (Table 2; Loop Unrolling workflow
// P:457-460) and the estimators of §5.2: Eq. 2, Eq. 3, Eq. 4
// (P:496-503), Eq. 5 (Q16), Eqs. 6-10 (Q18), per kernel.
//
//   k_est_rows    one thread per (use row j, pattern group): the matched samples of each
//                 in-edge (blamed at the def, scope loop = lca(def, use)) and of j itself
//                 (self / pass-through columns, scope loop = loop of j); row totals mrow[q][j]
//                 and the loop-scoped patterns' per-instruction item values.
//   k_est_edges   per-edge item values of the loop-scoped patterns (edge-parallel).
//   k_segsum      one warp per (segment, pattern): fixed-order strided sums + xor-shuffle tree
//                 (deterministic).  Stage 1: loop-exclusive (by scope-loop item lists) and
//                 function sums; stage 2: loop-inclusive (preorder subtree ranges) and kernel sums.
//   k_est_final   one warp per (kernel, pattern): T, A, R_I, M, Eqs. 2-5 / 10, best scope.
#include <algorithm>
#include <math.h>

#include "gpa_internal.cuh"

namespace gpa {
namespace {

// one thread per (use row j, group of kEstGroup patterns): the row's counts and in-edges are read
// once per group and every pattern of the group is evaluated from registers; consecutive threads
// take consecutive rows (coalesced).  Per (j, pattern) the sum runs over the row's edges in CSR
// order, then adds j's own part -- the oracle's order.
#ifndef GPA_EST_GROUP
#define GPA_EST_GROUP 4
#endif
constexpr int kEstGroup = GPA_EST_GROUP;

// A CTA = one warp per pattern group over the same 32 rows (a tile): the pattern fields are uniform
// in a warp, and a row's C entries and edges are fetched from DRAM once and served from L1 to the
// other groups' warps.  Measured and dropped: a warp-cooperative edge-parallel form
// (the blame tiles' pattern; config 4: 1.17 ms against 0.86 ms for this kernel plus k_est_edges --
// its shared-memory staging cut the resident warps of this latency-bound loop) and summing the row
// totals per function run of the tile with a shuffle scan instead of storing them per row (config
// 4's analysis 2.37 -> 2.49 ms, config 3's 74 -> 76 us).
__device__ __forceinline__ void body_est_rows(DevProgram p, EstimatePlan ep, uint32_t bx, uint32_t gx) {
  pdl_wait();
  __shared__ gpa_pattern sp[kPatternsMax];
  __shared__ int8_t sslot[kPatternsMax];
  for (uint32_t q = threadIdx.x; q < ep.n_pat; q += blockDim.x) {
    sp[q] = ep.pats[q];
    sslot[q] = ep.loop_slot[q];
  }
  __syncthreads();
  const uint64_t stride_items = (uint64_t)p.E + p.n;
  // a CTA = one warp per pattern group over the same 32 rows: the pattern fields are uniform in a
  // warp (no divergence on them), and a row's C entries and edges are fetched from DRAM once and
  // served from L1 to the other groups' warps
  const uint32_t grp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (grp * kEstGroup >= ep.n_pat) return;   // spare warps of a wider CTA (the fused analysis kernel)
  for (uint32_t j = bx * 32 + lane; j - lane < p.n; j += gx * 32) {
    if (j >= p.n) continue;
    const uint32_t q0 = grp * kEstGroup;
    const uint32_t nq = min((uint32_t)kEstGroup, ep.n_pat - q0);
    const uint64_t *row = p.C + (uint64_t)j * 2 * p.R;
    double XA[4], XL[4];   // all / latency samples of the dependency reasons at j
#pragma unroll
    for (int r = 1; r <= 3; ++r) {
      const uint64_t lat = row[p.R + r];
      XL[r] = (double)lat;
      XA[r] = (double)(lat + row[r]);
    }
    const uint32_t e0 = p.row_ptr[j], e1 = p.row_ptr[j + 1];
    const int32_t loop_j = p.loop_id[j];
    double sum[kEstGroup];
#pragma unroll
    for (int k = 0; k < kEstGroup; ++k) sum[k] = 0.0;
    // a row without dependency-reason samples gets 0 from every edge (X = 0 and, the row not being a
    // node of the graph, no candidates): skip the walk (no +0.0 adds, so the sums are unchanged)
    const bool dep = (XA[1] != 0.0) | (XA[2] != 0.0) | (XA[3] != 0.0);
    for (uint32_t e = e0; dep && e < e1; ++e) {   // loads only: per-edge values go to k_est_edges
      const EdgeInfo x = edge_info(p, e, loop_j);
      if (!x.m) continue;                  // no candidate reason: adds 0 to every pattern
#pragma unroll
      for (int k = 0; k < kEstGroup; ++k) {
        if ((uint32_t)k >= nq) break;
        const gpa_pattern &q = sp[q0 + k];
        if (q.model == 5) continue;
        sum[k] = __dadd_rn(sum[k], edge_match(q, x, q.sample_class ? XL : XA));
      }
    }
    const uint32_t cls_j = p.opclass[j], flags_j = p.iflags[j], self_j = p.selfm[j];
#pragma unroll
    for (int k = 0; k < kEstGroup; ++k) {
      if ((uint32_t)k >= nq) break;
      const uint32_t qi = q0 + k;
      const gpa_pattern &q = sp[qi];
      if (q.model == 5) {
        ep.mrow[(uint64_t)qi * p.n + j] = 0.0;
        continue;
      }
      const double mi = instr_match(q, p.R, row, q.sample_class ? XL : XA, cls_j, flags_j, self_j, loop_j);
      const int slot = sslot[qi];
      if (slot >= 0) ep.mval[(uint64_t)slot * stride_items + p.E + j] = mi;
      ep.mrow[(uint64_t)qi * p.n + j] = __dadd_rn(sum[k], mi);
    }
  }
}

__global__ void k_est_rows(DevProgram p, EstimatePlan ep) {
  body_est_rows(p, ep, blockIdx.x, gridDim.x);
}

// per-edge matched samples of the loop-scoped patterns (mval[slot][e]), edge-parallel and
// coalesced; the same arithmetic as k_est_rows, so the item values and the row sums agree
__device__ __forceinline__ void body_est_edges(DevProgram p, EstimatePlan ep, uint32_t bx, uint32_t gx) {
  pdl_wait();
  __shared__ gpa_pattern sp[kPatternsMax];
  __shared__ int8_t sslot[kPatternsMax];
  __shared__ uint32_t slot_q[kPatternsMax], n_slot_q;
  if (threadIdx.x == 0) {
    uint32_t c = 0;
    for (uint32_t q = 0; q < ep.n_pat; ++q)
      if (ep.loop_slot[q] >= 0 && ep.pats[q].model != 5) slot_q[c++] = q;
    n_slot_q = c;
  }
  for (uint32_t q = threadIdx.x; q < ep.n_pat; q += blockDim.x) {
    sp[q] = ep.pats[q];
    sslot[q] = ep.loop_slot[q];
  }
  __syncthreads();
  const uint64_t stride_items = (uint64_t)p.E + p.n;
  for (uint32_t e = bx * blockDim.x + threadIdx.x; e < p.E; e += gx * blockDim.x) {
    const uint32_t j = p.edge_use[e];
    const uint64_t *row = p.C + (uint64_t)j * 2 * p.R;
    double XA[4], XL[4];
#pragma unroll
    for (int r = 1; r <= 3; ++r) {
      const uint64_t lat = row[p.R + r];
      XL[r] = (double)lat;
      XA[r] = (double)(lat + row[r]);
    }
    const EdgeInfo x = edge_info(p, e, p.loop_id[j]);
    for (uint32_t k = 0; k < n_slot_q; ++k) {
      const gpa_pattern &q = sp[slot_q[k]];
      ep.mval[(uint64_t)sslot[slot_q[k]] * stride_items + e] = edge_match(q, x, q.sample_class ? XL : XA);
    }
  }
}

__global__ void k_est_edges(DevProgram p, EstimatePlan ep) {
  body_est_edges(p, ep, blockIdx.x, gridDim.x);
}

// the two independent item passes in one launch: CTAs [0, g_rows) are k_est_rows', the rest
// k_est_edges' (both read only the blame outputs and C) -- one dependent level fewer in the graph
__global__ void k_est_items(DevProgram p, EstimatePlan ep, uint32_t g_rows) {
  if (blockIdx.x < g_rows) body_est_rows(p, ep, blockIdx.x, g_rows);
  else body_est_edges(p, ep, blockIdx.x - g_rows, gridDim.x - g_rows);
}


struct SegFamily {
  const double *values;     // value row v starts at values + v * row_stride
  uint64_t row_stride;
  const uint32_t *perm;     // position -> item (nullable)
  const uint32_t *begin;    // [n_seg] (or ptr array of n_seg+1 when end == nullptr)
  const uint32_t *end;
  uint32_t n_seg;
  double *out;              // out[q * n_seg + s]
  int32_t vrow[kPatternsMax]; // pattern -> value row, -1 = not applicable (output 0)
};

struct SegLaunch {
  SegFamily fam[2];
  uint32_t n_fam, n_pat;
};

__device__ __forceinline__ void body_segsum(SegLaunch L, uint32_t fam, uint32_t bx, uint32_t gx) {
  pdl_wait();
  const uint32_t lane = threadIdx.x & 31;
  const SegFamily &F = L.fam[fam];
  const uint64_t items = (uint64_t)F.n_seg * L.n_pat;
  const uint32_t warps = (gx * blockDim.x) >> 5;
  for (uint64_t w = (bx * blockDim.x + threadIdx.x) >> 5; w < items; w += warps) {
    const uint32_t q = (uint32_t)(w / F.n_seg), s = (uint32_t)(w % F.n_seg);
    const int32_t vr = F.vrow[q];
    double acc = 0.0;
    if (vr >= 0) {
      const double *vals = F.values + (uint64_t)vr * F.row_stride;
      const uint32_t b = F.begin[s], e = F.end ? F.end[s] : F.begin[s + 1];
      double a1 = 0.0, a2 = 0.0, a3 = 0.0;   // four interleaved accumulators: loads in flight
      uint32_t pos = b + lane;
      for (; pos + 96 < e; pos += 128) {
        const double x0 = vals[F.perm ? F.perm[pos] : pos], x1 = vals[F.perm ? F.perm[pos + 32] : pos + 32];
        const double x2 = vals[F.perm ? F.perm[pos + 64] : pos + 64], x3 = vals[F.perm ? F.perm[pos + 96] : pos + 96];
        acc = __dadd_rn(acc, x0);
        a1 = __dadd_rn(a1, x1);
        a2 = __dadd_rn(a2, x2);
        a3 = __dadd_rn(a3, x3);
      }
      for (; pos < e; pos += 32) acc = __dadd_rn(acc, vals[F.perm ? F.perm[pos] : pos]);
      acc = __dadd_rn(__dadd_rn(acc, a1), __dadd_rn(a2, a3));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    }
    if (lane == 0) F.out[(uint64_t)q * F.n_seg + s] = acc;
  }
}

__global__ void k_segsum(SegLaunch L) {
  body_segsum(L, blockIdx.y, blockIdx.x, gridDim.x);
}

__device__ __forceinline__ double eq2(double T, double M) {
  if (T <= 0.0) return 1.0;
  if (M >= T) return INFINITY;
  return T / (T - M);
}

// one warp per (kernel, pattern); lanes stride over the kernel's scopes for Eq. 5 and the warp
// takes the max with ties to the lowest scope id (loops before functions), as a sequential scan
// in scope order would.
__device__ __forceinline__ void body_est_final(DevProgram p, EstimatePlan ep, uint32_t bx, uint32_t gx) {
  pdl_wait();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t total = p.n_kernels * ep.n_pat;
  const uint32_t warps = (gx * blockDim.x) >> 5;
  for (uint32_t t = (bx * blockDim.x + threadIdx.x) >> 5; t < total; t += warps) {
    const uint32_t k = t / ep.n_pat, qi = t % ep.n_pat;
    const gpa_pattern q = ep.pats[qi];
    const uint64_t A = ep.kern_al[2 * (uint64_t)k], T = A + ep.kern_al[2 * (uint64_t)k + 1];
    const double Td = (double)T, Ad = (double)A;
    gpa_estimate_out o;
    o.T = T;
    o.A = A;
    o.model = q.model;
    o.pad = 0;
    o.best_scope = -1;
    if (q.model == 5) {
      const double R_I = T ? Ad / Td : 0.0;
      const uint32_t gb = p.kernel_grid_blocks[k];
      bool matched = q.parallel_rule == 1 || (q.parallel_rule == 2 && gb != 0xffffffffu && gb < q.sm_count);
      double W = q.W, W_new = q.W_new;
      if (q.parallel_rule == 3 || q.parallel_rule == 4) {   // occupancy model (gpa_set_launches)
        const KernOcc &oc = ep.occ[k];
        matched = q.parallel_rule == 3 ? oc.match_block != 0 : oc.match_thread != 0;
        if (matched) {
          W = oc.W;
          W_new = q.parallel_rule == 3 ? oc.W_new_block : oc.W_new_thread;
        }
      }
      double s = 1.0;
      if (matched) {
        const double C_W = W_new / W;
        const double I = 1.0 - pow(1.0 - R_I, W);
        const double In = 1.0 - pow(1.0 - R_I, W_new);
        const double C_I = (I == 0.0) ? 1.0 : In / I;
        s = (1.0 / C_W) * C_I * q.f;
      }
      o.speedup = s;
      o.M = 0.0;
      o.eq3 = o.eq4 = 1.0;
      o.matched = matched;
    } else {
      const double M = ep.kM[(uint64_t)qi * p.n_kernels + k];
      o.M = M;
      o.matched = M > 0.0;
      o.eq3 = eq2(Td, M);
      o.eq4 = eq2(Td, fmin(Ad, M));
      if (q.model == 0) {
        o.speedup = eq2(Td, q.ratio * M);
      } else if (q.model == 1) {
        o.speedup = o.eq4;
      } else {
        double best = -1.0;
        int32_t bs = -1;
        if (q.model == 2 || q.model == 4) {
          // four loop scopes per lane in flight (ids first, then their A and M^L), evaluated in the
          // same per-lane order as one at a time
          const uint32_t x0 = ep.kloop_ptr[k], x1 = ep.kloop_ptr[k + 1];
          for (uint32_t xb = x0 + lane; xb < x1; xb += 4 * 32) {
            uint32_t l[4];
            double Al[4], Ml[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) l[u] = xb + 32u * u < x1 ? ep.kloops[xb + 32u * u] : 0xffffffffu;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              Al[u] = l[u] != 0xffffffffu ? (double)ep.loop_incl_al[2 * (uint64_t)l[u]] : 0.0;
              Ml[u] = l[u] != 0xffffffffu ? ep.lM_incl[(uint64_t)qi * p.n_loops + l[u]] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (l[u] == 0xffffffffu) break;
              const double sv = eq2(Td, fmin(Al[u], Ml[u]));
              if (bs < 0 || sv > best) { best = sv; bs = (int32_t)l[u]; }
            }
          }
        }
        if (q.model == 3 || q.model == 4) {
          for (uint32_t f = p.kernel_func_begin[k] + lane; f < p.kernel_func_begin[k + 1]; f += 32) {
            const double Af = (double)ep.func_al[2 * (uint64_t)f];
            const double sv = eq2(Td, fmin(Af, ep.fM[(uint64_t)qi * p.n_funcs + f]));
            if (bs < 0 || sv > best) { best = sv; bs = (int32_t)(p.n_loops + f); }
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, off);
          const int32_t os = __shfl_xor_sync(0xffffffffu, bs, off);
          const bool take = os >= 0 && (bs < 0 || ob > best || (ob == best && os < bs));
          if (take) { best = ob; bs = os; }
        }
        o.speedup = bs < 0 ? 1.0 : best;
        o.best_scope = bs;
      }
    }
    o.unbounded = isinf(o.speedup) ? 1 : 0;
    if (lane == 0) ep.out[t] = o;
  }
}

__global__ void k_est_final(DevProgram p, EstimatePlan ep) {
  body_est_final(p, ep, blockIdx.x, gridDim.x);
}

// the two k_segsum stages: (1) loops exclusive (by scope-loop items) and functions, (2) loops
// inclusive (preorder subtree ranges over the exclusive sums) and kernels
inline void make_seg_launches(const DevProgram &p, const EstimatePlan &ep, SegLaunch &a, SegLaunch &b) {
  a = SegLaunch{};
  a.n_pat = ep.n_pat;
  a.n_fam = 2;
  a.fam[0] = SegFamily{ep.mval, (uint64_t)p.E + p.n, ep.loop_items, ep.loop_item_ptr, nullptr, p.n_loops, ep.lM_excl, {}};
  a.fam[1] = SegFamily{ep.mrow, p.n, nullptr, p.func_begin, nullptr, p.n_funcs, ep.fM, {}};
  for (int q = 0; q < kPatternsMax; ++q) {
    a.fam[0].vrow[q] = ep.loop_slot[q];
    a.fam[1].vrow[q] = q < (int)ep.n_pat ? q : -1;
  }
  b = SegLaunch{};
  b.n_pat = ep.n_pat;
  b.n_fam = 2;
  b.fam[0] = SegFamily{ep.lM_excl, p.n_loops, ep.pre_perm, ep.pre_begin, ep.pre_end, p.n_loops, ep.lM_incl, {}};
  b.fam[1] = SegFamily{ep.fM, p.n_funcs, nullptr, p.kernel_func_begin, nullptr, p.n_kernels, ep.kM, {}};
  for (int q = 0; q < kPatternsMax; ++q) {
    b.fam[0].vrow[q] = ep.loop_slot[q] >= 0 ? q : -1;
    b.fam[1].vrow[q] = q < (int)ep.n_pat ? q : -1;
  }
}

}  // namespace

#ifndef GPA_FUSED_TU
static cudaError_t launch_segsums(const DevProgram &p, const EstimatePlan &ep, int n_sms, cudaStream_t s,
                                  uint64_t *launches);

// matched samples per item, loop / function / kernel sums: reads only the blame rows' outputs
// (cand, share, selfm) and C, so it can run beside the def reduction and the rollup
cudaError_t launch_estimate_sums(const DevProgram &p, const EstimatePlan &ep, int n_sms, cudaStream_t s,
                                 uint64_t *launches) {
  const uint32_t n_groups = (ep.n_pat + kEstGroup - 1) / kEstGroup;   // <= 8: a warp per group
  const uint32_t g = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(((uint64_t)p.n + 31) / 32, (uint64_t)n_sms * 64));
  bool any_slot = false;
  for (uint32_t q = 0; q < ep.n_pat; ++q) any_slot |= ep.loop_slot[q] >= 0;
#ifndef GPA_EST_MERGE
#define GPA_EST_MERGE 1
#endif
#ifndef GPA_EST_MERGE_MAX_N
#define GPA_EST_MERGE_MAX_N kPdlMaxInstr
#endif
  if (GPA_EST_MERGE && any_slot && p.E && p.n < (uint32_t)(GPA_EST_MERGE_MAX_N)) {   // config 4: separate kernels measured faster
    const uint32_t bt = 32 * n_groups;
    const uint32_t ge = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(((uint64_t)p.E + bt - 1) / bt, (uint64_t)n_sms * 32));
    k_est_items<<<g + ge, bt, 0, s>>>(p, ep, g);
    *launches += 1;
    return launch_segsums(p, ep, n_sms, s, launches);
  }
  k_est_rows<<<g, 32 * n_groups, 0, s>>>(p, ep);
  if (any_slot && p.E) {
    const uint32_t ge = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(((uint64_t)p.E + 255) / 256, (uint64_t)n_sms * 16));
    const cudaError_t e = launch_pdl(p.n, k_est_edges, ge, 256, 0, s, p, ep);
    if (e != cudaSuccess) return e;
    *launches += 1;
  }
  *launches += 1;
  return launch_segsums(p, ep, n_sms, s, launches);
}

// the two segment-sum stages over the item values
static cudaError_t launch_segsums(const DevProgram &p, const EstimatePlan &ep, int n_sms, cudaStream_t s,
                                  uint64_t *launches) {
  SegLaunch a, b;
  make_seg_launches(p, ep, a, b);
  const uint64_t w1 = std::max<uint64_t>((uint64_t)p.n_loops, p.n_funcs) * ep.n_pat;
  dim3 g1((uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((w1 + 3) / 4, (uint64_t)n_sms * 32)), 2);
  cudaError_t e = launch_pdl(p.n, k_segsum, g1, 128, 0, s, a);
  if (e != cudaSuccess) return e;
  const uint64_t w2 = std::max<uint64_t>((uint64_t)p.n_loops, p.n_kernels) * ep.n_pat;
  dim3 g2((uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((w2 + 3) / 4, (uint64_t)n_sms * 32)), 2);
  e = launch_pdl(p.n, k_segsum, g2, 128, 0, s, b);
  *launches += 2;
  return e;
}

// Eqs. 2-5 / 10 per (kernel, pattern): needs the sums above and the rollup's A sums
cudaError_t launch_estimate_final(const DevProgram &p, const EstimatePlan &ep, int n_sms, cudaStream_t s,
                                  uint64_t *launches) {
  const uint32_t total = p.n_kernels * ep.n_pat;
  k_est_final<<<std::max<uint32_t>(1, std::min<uint32_t>((total + 3) / 4, n_sms * 32)), 128, 0, s>>>(p, ep);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_estimate(const DevProgram &p, const EstimatePlan &ep, int n_sms, cudaStream_t s,
                            uint64_t *launches) {
  cudaError_t e = launch_estimate_sums(p, ep, n_sms, s, launches);
  return e != cudaSuccess ? e : launch_estimate_final(p, ep, n_sms, s, launches);
}

#endif  // GPA_FUSED_TU

}  // namespace gpa

// advice.cu -- after the path: the data of GPA's advice report
// (readings DESIGN.md §3.2 Q30-Q32).
//
//   k_hotspots   one CTA per (kernel, pattern): every thread scans a strided share of the kernel's
//                items -- its in-edges (def, use, max_len, matched samples) and its instructions'
//                own samples -- evaluating the pattern with the estimate kernels' arithmetic
//                (edge_match / instr_match, bit-identical values), keeps a register top-k, and
//                the CTA merges the 256 lists by k rounds of a block argmax.  Order: samples
//                descending, ties by item id (edge index, then E + instruction).
//   k_rank       one thread per kernel: patterns by estimated speedup descending, stable.
//   k_coverage   one CTA per kernel: single-dependency nodes before / after pruning, integer
//                block reduction (exact, order-free).
#include <algorithm>
#include <math.h>

#include "gpa_internal.cuh"

namespace gpa {
namespace {

constexpr uint32_t kAdvThreads = 256;

__device__ __forceinline__ bool hot_before(double sa, uint32_t ia, double sb, uint32_t ib) {
  return sa > sb || (sa == sb && ia < ib);
}

__global__ void __launch_bounds__(kAdvThreads) k_hotspots(DevProgram p, EstimatePlan ep, AdvicePlan ap) {
  const uint32_t k = blockIdx.x / ep.n_pat, qi = blockIdx.x % ep.n_pat;
  const gpa_pattern q = ep.pats[qi];
  const uint32_t top_k = ap.top_k;
  __shared__ double s_val[kAdvThreads * kTopKMax];
  __shared__ uint32_t s_item[kAdvThreads * kTopKMax];
  __shared__ double w_val[kAdvThreads / 32];
  __shared__ uint32_t w_item[kAdvThreads / 32], w_tid[kAdvThreads / 32];
  __shared__ uint32_t s_win;
  // register top list of this thread (sorted, samples > 0 only)
  double val[kTopKMax];
  uint32_t item[kTopKMax];
#pragma unroll
  for (int t = 0; t < kTopKMax; ++t) { val[t] = 0.0; item[t] = 0xffffffffu; }
  auto offer = [&](double v, uint32_t id) {
    if (!(v > 0.0)) return;
#pragma unroll
    for (int t = 0; t < kTopKMax; ++t) {   // insertion by compare-and-swap down the list
      if ((uint32_t)t < top_k && hot_before(v, id, val[t], item[t])) {
        const double tv = val[t];
        const uint32_t ti = item[t];
        val[t] = v; item[t] = id;
        v = tv; id = ti;
      }
    }
  };
  if (q.model != 5) {
    const uint32_t i0 = p.func_begin[p.kernel_func_begin[k]], i1 = p.func_begin[p.kernel_func_begin[k + 1]];
    for (uint32_t j = i0 + threadIdx.x; j < i1; j += blockDim.x) {
      const uint64_t *row = p.C + (uint64_t)j * 2 * p.R;
      double X[4];
#pragma unroll
      for (int r = 1; r <= 3; ++r) {
        const uint64_t lat = row[p.R + r];
        X[r] = q.sample_class ? (double)lat : (double)(lat + row[r]);
      }
      const int32_t loop_j = p.loop_id[j];
      for (uint32_t e = p.row_ptr[j]; e < p.row_ptr[j + 1]; ++e) offer(edge_match(q, edge_info(p, e, loop_j), X), e);
      offer(instr_match(q, p.R, row, X, p.opclass[j], p.iflags[j], p.selfm[j], loop_j), p.E + j);
    }
  }
#pragma unroll
  for (int t = 0; t < kTopKMax; ++t) {
    s_val[threadIdx.x * kTopKMax + t] = val[t];
    s_item[threadIdx.x * kTopKMax + t] = item[t];
  }
  __syncthreads();
  // merge: top_k rounds of a block argmax over the heads of the per-thread lists
  uint32_t head = 0;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  gpa_hotspot *out = ap.hot + ((uint64_t)k * ep.n_pat + qi) * kTopKMax;
  uint32_t n_out = 0;
  for (uint32_t round = 0; round < top_k; ++round) {
    double v = head < top_k ? s_val[threadIdx.x * kTopKMax + head] : 0.0;
    uint32_t id = head < top_k ? s_item[threadIdx.x * kTopKMax + head] : 0xffffffffu;
    uint32_t who = threadIdx.x;
    if (!(v > 0.0)) { v = 0.0; id = 0xffffffffu; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const uint32_t oi = __shfl_xor_sync(0xffffffffu, id, o), ow = __shfl_xor_sync(0xffffffffu, who, o);
      if (hot_before(ov, oi, v, id)) { v = ov; id = oi; who = ow; }
    }
    if (lane == 0) { w_val[warp] = v; w_item[warp] = id; w_tid[warp] = who; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double bv = w_val[0];
      uint32_t bi = w_item[0], bw = w_tid[0];
      for (uint32_t w = 1; w < kAdvThreads / 32; ++w)
        if (hot_before(w_val[w], w_item[w], bv, bi)) { bv = w_val[w]; bi = w_item[w]; bw = w_tid[w]; }
      if (bv > 0.0) {
        gpa_hotspot h;
        if (bi < p.E) {
          h.def_pc = p.edge_def[bi]; h.use_pc = p.edge_use[bi]; h.distance = p.edge_max[bi];
        } else {
          h.def_pc = h.use_pc = bi - p.E; h.distance = 0;
        }
        h.item = bi;
        h.samples = bv;
        out[n_out++] = h;
        s_win = bw;
      } else {
        s_win = 0xffffffffu;
      }
    }
    __syncthreads();
    const uint32_t win = s_win;
    if (win == 0xffffffffu) break;   // uniform: every thread read the same s_win
    if (threadIdx.x == win) ++head;
    __syncthreads();
  }
  if (threadIdx.x == 0) ap.n_hot[(uint64_t)k * ep.n_pat + qi] = n_out;
}

__global__ void k_rank(EstimatePlan ep, uint32_t n_kernels, uint32_t *rank) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n_kernels; k += gridDim.x * blockDim.x) {
    const gpa_estimate_out *x = ep.out + (uint64_t)k * ep.n_pat;
    uint32_t o[kPatternsMax];
    for (uint32_t a = 0; a < ep.n_pat; ++a) {   // stable insertion sort, descending speedup
      uint32_t b = a;
      while (b > 0 && x[o[b - 1]].speedup < x[a].speedup) {
        o[b] = o[b - 1];
        --b;
      }
      o[b] = a;
    }
    for (uint32_t a = 0; a < ep.n_pat; ++a) rank[(uint64_t)k * ep.n_pat + a] = o[a];
  }
}

__global__ void __launch_bounds__(kAdvThreads) k_coverage(DevProgram p, gpa_coverage *cov) {
  const uint32_t k = blockIdx.x;
  const uint32_t i0 = p.func_begin[p.kernel_func_begin[k]], i1 = p.func_begin[p.kernel_func_begin[k + 1]];
  unsigned long long nodes = 0, before = 0, after = 0;
  for (uint32_t j = i0 + threadIdx.x; j < i1; j += blockDim.x) {
    const uint64_t *row = p.C + (uint64_t)j * 2 * p.R;
    const uint32_t e0 = p.row_ptr[j], e1 = p.row_ptr[j + 1];
    bool live = false, single_b = true, single_a = true;
    for (uint32_t r = R_MEM; r <= R_SYNC; ++r) {
      if (row[r] + row[p.R + r] == 0) continue;   // no stall of this dependency kind at j
      live = true;
      uint32_t n_r = 0;
      for (uint32_t e = e0; e < e1; ++e) n_r += (p.cand[e] >> (r - 1)) & 1u;
      single_b &= (e1 - e0) <= 1;
      single_a &= n_r <= 1;
    }
    nodes += live;
    before += live && single_b;
    after += live && single_a;
  }
  __shared__ unsigned long long s[3];
  if (threadIdx.x < 3) s[threadIdx.x] = 0;
  __syncthreads();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nodes += __shfl_xor_sync(0xffffffffu, nodes, o);
    before += __shfl_xor_sync(0xffffffffu, before, o);
    after += __shfl_xor_sync(0xffffffffu, after, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&s[0], nodes);
    atomicAdd(&s[1], before);
    atomicAdd(&s[2], after);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    cov[k].nodes = s[0];
    cov[k].single_before = s[1];
    cov[k].single_after = s[2];
  }
}

}  // namespace

cudaError_t launch_advice(const DevProgram &p, const EstimatePlan &ep, const AdvicePlan &ap, cudaStream_t s,
                          uint64_t *launches) {
  const uint64_t blocks = (uint64_t)p.n_kernels * ep.n_pat;
  k_hotspots<<<(uint32_t)blocks, kAdvThreads, 0, s>>>(p, ep, ap);
  k_rank<<<(p.n_kernels + 127) / 128, 128, 0, s>>>(ep, p.n_kernels, ap.rank);
  k_coverage<<<p.n_kernels, kAdvThreads, 0, s>>>(p, ap.cov);
  *launches += 3;
  return cudaGetLastError();
}

}  // namespace gpa

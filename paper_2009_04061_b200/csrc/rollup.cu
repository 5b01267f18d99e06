// rollup.cu -- row a7: per-instruction blame vectors summed over program structure
// (line, loop exclusive/inclusive, function, kernel, Q16).
//
// Hand-written segmented reductions (no CUB), deterministic: every sum has a fixed order.
//   k_vrows            V[i] = {NCOL x (all, lat)} for every instruction, one
//                      warp per instruction row, stores coalesced; this is also the instruction
//                      level of the rollup (gpa_instr_vector).
//   k_rollup_chunks    one warp per <=128-instruction chunk of a create-time order (line-major |
//                      loop-major | function ranges); member ids are loaded once and broadcast by
//                      shuffles, lane s owns value slot s (and s+32) of the row, so each member
//                      row is one coalesced load and four interleaved accumulators keep loads in
//                      flight.  Slots NV, NV+1 carry (A_i, L_i).
//   k_rollup_segments  one warp per segment, same scheme over rows: chunk partials (stage 1:
//                      lines, loops-exclusive, functions) or earlier rows through a permutation
//                      (stage 2: loops-inclusive = preorder subtree ranges of the loop-exclusive
//                      rows; kernels = their function rows).
#include <algorithm>

#include "gpa_internal.cuh"

namespace gpa {
namespace {

// one warp per instruction row (lane = value slot): the row's loads are shared by the warp and
// V is written coalesced
__global__ void k_vrows(DevProgram p, double *__restrict__ vbuf) {
  const uint32_t nv = 2 * p.ncol, lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < p.n; i += warps)
    for (uint32_t s = lane; s < nv; s += 32) vbuf[(uint64_t)i * nv + s] = vvalue(p, i, s >> 1, s & 1);
}

// sum over positions [b, e) of rows it(pos): slot s < nv from vals, slots nv, nv+1 from al
template <typename ItemFn>
__device__ __forceinline__ void warp_sum_rows(uint32_t lane, uint32_t nv, uint32_t b, uint32_t e, ItemFn item,
                                              const double *__restrict__ vals, const uint64_t *__restrict__ al,
                                              double *__restrict__ out_v, uint64_t *__restrict__ out_al) {
  for (uint32_t s = lane; s < nv + 2; s += 32) {
    if (s < nv) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      uint32_t pos = b;
      for (; pos + 4 <= e; pos += 4) {
        const double x0 = vals[(uint64_t)item(pos) * nv + s], x1 = vals[(uint64_t)item(pos + 1) * nv + s];
        const double x2 = vals[(uint64_t)item(pos + 2) * nv + s], x3 = vals[(uint64_t)item(pos + 3) * nv + s];
        a0 = __dadd_rn(a0, x0);
        a1 = __dadd_rn(a1, x1);
        a2 = __dadd_rn(a2, x2);
        a3 = __dadd_rn(a3, x3);
      }
      for (; pos < e; ++pos) a0 = __dadd_rn(a0, vals[(uint64_t)item(pos) * nv + s]);
      out_v[s] = __dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3));
    } else {
      uint64_t acc = 0;
      for (uint32_t pos = b; pos < e; ++pos) acc += al[2 * (uint64_t)item(pos) + (s - nv)];
      out_al[s - nv] = acc;
    }
  }
}

// chunk of <= 128 members: member ids are loaded once (4 per lane) and broadcast by shuffles, so
// the row loads of consecutive members are independent and stay in flight together
__global__ void __launch_bounds__(128) k_rollup_chunks(RollupPlan rp, uint32_t nv, const double *__restrict__ vbuf,
                                                       const uint64_t *__restrict__ AL) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t ch = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; ch < rp.n_chunks; ch += warps) {
    const uint32_t b = rp.chunk_begin[ch], len = rp.chunk_end[ch] - b;
    uint32_t ids[kChunk / 32];
#pragma unroll
    for (int t = 0; t < kChunk / 32; ++t) ids[t] = (lane + 32 * t < len) ? rp.order[b + lane + 32 * t] : 0u;
    for (uint32_t s0 = 0; s0 < nv + 2; s0 += 32) {   // uniform trip count: shuffles need all lanes
      const uint32_t s = s0 + lane;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      uint64_t al = 0;
      const bool is_v = s < nv, is_al = s >= nv && s < nv + 2;
#pragma unroll
      for (int t = 0; t < kChunk / 32; ++t) {
        const uint32_t m_end = len > 32u * t ? min(32u, len - 32u * t) : 0u;
        for (uint32_t m = 0; m < m_end; m += 4) {
          const uint32_t i0 = __shfl_sync(0xffffffffu, ids[t], m);
          const uint32_t i1 = __shfl_sync(0xffffffffu, ids[t], m + 1 < 32 ? m + 1 : 31);
          const uint32_t i2 = __shfl_sync(0xffffffffu, ids[t], m + 2 < 32 ? m + 2 : 31);
          const uint32_t i3 = __shfl_sync(0xffffffffu, ids[t], m + 3 < 32 ? m + 3 : 31);
          if (is_v) {
            const double x0 = vbuf[(uint64_t)i0 * nv + s];
            const double x1 = m + 1 < m_end ? vbuf[(uint64_t)i1 * nv + s] : 0.0;
            const double x2 = m + 2 < m_end ? vbuf[(uint64_t)i2 * nv + s] : 0.0;
            const double x3 = m + 3 < m_end ? vbuf[(uint64_t)i3 * nv + s] : 0.0;
            a0 = __dadd_rn(a0, x0);
            a1 = __dadd_rn(a1, x1);
            a2 = __dadd_rn(a2, x2);
            a3 = __dadd_rn(a3, x3);
          } else if (is_al) {
            const uint32_t c = s - nv;
            al += AL[2 * (uint64_t)i0 + c];
            if (m + 1 < m_end) al += AL[2 * (uint64_t)i1 + c];
            if (m + 2 < m_end) al += AL[2 * (uint64_t)i2 + c];
            if (m + 3 < m_end) al += AL[2 * (uint64_t)i3 + c];
          }
        }
      }
      if (is_v) rp.part_v[(uint64_t)ch * nv + s] = __dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3));
      else if (is_al) rp.part_al[2 * (uint64_t)ch + (s - nv)] = al;
    }
  }
}

__global__ void __launch_bounds__(128) k_rollup_segments(uint32_t nv, const double *__restrict__ in_v,
                                                         const uint64_t *__restrict__ in_al,
                                                         const uint32_t *__restrict__ perm,
                                                         const uint32_t *__restrict__ seg_begin,
                                                         const uint32_t *__restrict__ seg_end, uint32_t n_seg,
                                                         double *__restrict__ out_v, uint64_t *__restrict__ out_al) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t sg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; sg < n_seg; sg += warps) {
    if (perm)
      warp_sum_rows(lane, nv, seg_begin[sg], seg_end[sg], [perm](uint32_t pos) { return perm[pos]; }, in_v, in_al,
                    out_v + (uint64_t)sg * nv, out_al + 2 * (uint64_t)sg);
    else
      warp_sum_rows(lane, nv, seg_begin[sg], seg_end[sg], [](uint32_t pos) { return pos; }, in_v, in_al,
                    out_v + (uint64_t)sg * nv, out_al + 2 * (uint64_t)sg);
  }
}

inline uint32_t warp_grid(uint64_t warps, int n_sms) {
  const uint64_t blocks = (warps + 3) / 4;   // 128 threads = 4 warps per block
  return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(blocks, (uint64_t)n_sms * 32));
}

}  // namespace

cudaError_t launch_vrows(const DevProgram &p, double *vbuf, int n_sms, cudaStream_t s) {
  const uint64_t total = (uint64_t)p.n * 32;
  const uint32_t g = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((total + 255) / 256, (uint64_t)n_sms * 32));
  k_vrows<<<g, 256, 0, s>>>(p, vbuf);
  return cudaGetLastError();
}

cudaError_t launch_rollup(const DevProgram &p, const RollupPlan &rp, int n_sms, cudaStream_t s,
                          uint64_t *launches) {
  const uint32_t nv = 2 * p.ncol;
  cudaError_t e = launch_vrows(p, rp.vbuf, n_sms, s);
  if (e != cudaSuccess) return e;
  if (rp.n_chunks) k_rollup_chunks<<<warp_grid(rp.n_chunks, n_sms), 128, 0, s>>>(rp, nv, rp.vbuf, p.AL);
  k_rollup_segments<<<warp_grid(rp.n_seg1, n_sms), 128, 0, s>>>(
      nv, rp.part_v, rp.part_al, nullptr, rp.seg1_begin, rp.seg1_end, rp.n_seg1, rp.rows_v, rp.rows_al);
  k_rollup_segments<<<warp_grid(rp.n_seg2, n_sms), 128, 0, s>>>(
      nv, rp.rows_v, rp.rows_al, rp.seg2_perm, rp.seg2_begin, rp.seg2_end, rp.n_seg2,
      rp.rows_v + (uint64_t)rp.n_seg1 * nv, rp.rows_al + 2 * (uint64_t)rp.n_seg1);
  *launches += rp.n_chunks ? 4 : 3;
  return cudaGetLastError();
}

}  // namespace gpa

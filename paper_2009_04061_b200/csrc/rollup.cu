// rollup.cu -- row a7: per-instruction blame vectors summed over program structure
// (line, loop exclusive/inclusive, function, kernel, Q16).
//
// Hand-written segmented reductions (no CUB), deterministic: every sum runs in a fixed order.
//   k_rollup_chunks    one warp per <=128-instruction chunk of a create-time order (line-major
//                      | loop-major | function ranges); lane s owns value slot s and s+32 of
//                      V[i] = {NCOL x (all, lat)} + (A_i, L_i) and sums it over the chunk.
//   k_rollup_segments  one warp per segment, summing rows (chunk partials, or earlier rows via
//                      a permutation) over [begin, end).  Stage 1: lines, loops-exclusive,
//                      functions from chunk partials.  Stage 2: loops-inclusive (subtree ranges
//                      of the preorder) from loop-exclusive rows, kernels from function rows.
#include <algorithm>

#include "gpa_internal.cuh"

namespace gpa {
namespace {

__global__ void k_rollup_chunks(DevProgram p, RollupPlan rp) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nv = 2 * p.ncol;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t ch = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; ch < rp.n_chunks; ch += warps) {
    const uint32_t b = rp.chunk_begin[ch], e = rp.chunk_end[ch];
    for (uint32_t s = lane; s < nv + 2; s += 32) {
      if (s < nv) {
        double acc = 0.0;
        for (uint32_t pos = b; pos < e; ++pos) acc = __dadd_rn(acc, vvalue(p, rp.order[pos], s >> 1, s & 1));
        rp.part_v[(uint64_t)ch * nv + s] = acc;
      } else {
        uint64_t acc = 0;
        for (uint32_t pos = b; pos < e; ++pos) acc += p.AL[2 * (uint64_t)rp.order[pos] + (s - nv)];
        rp.part_al[2 * (uint64_t)ch + (s - nv)] = acc;
      }
    }
  }
}

__global__ void k_rollup_segments(uint32_t nv, const double *__restrict__ in_v,
                                  const uint64_t *__restrict__ in_al, const uint32_t *__restrict__ perm,
                                  const uint32_t *__restrict__ seg_begin, const uint32_t *__restrict__ seg_end,
                                  uint32_t n_seg, double *__restrict__ out_v, uint64_t *__restrict__ out_al) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t sg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; sg < n_seg; sg += warps) {
    const uint32_t b = seg_begin[sg], e = seg_end[sg];
    for (uint32_t s = lane; s < nv + 2; s += 32) {
      if (s < nv) {
        double acc = 0.0;
        for (uint32_t pos = b; pos < e; ++pos) {
          const uint32_t it = perm ? perm[pos] : pos;
          acc = __dadd_rn(acc, in_v[(uint64_t)it * nv + s]);
        }
        out_v[(uint64_t)sg * nv + s] = acc;
      } else {
        uint64_t acc = 0;
        for (uint32_t pos = b; pos < e; ++pos) {
          const uint32_t it = perm ? perm[pos] : pos;
          acc += in_al[2 * (uint64_t)it + (s - nv)];
        }
        out_al[2 * (uint64_t)sg + (s - nv)] = acc;
      }
    }
  }
}

inline uint32_t warp_grid(uint64_t warps, int n_sms) {
  const uint64_t blocks = (warps + 3) / 4;   // 128 threads = 4 warps per block
  return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(blocks, (uint64_t)n_sms * 32));
}

}  // namespace

cudaError_t launch_rollup(const DevProgram &p, const RollupPlan &rp, int n_sms, cudaStream_t s,
                          uint64_t *launches) {
  const uint32_t nv = 2 * p.ncol;
  if (rp.n_chunks) k_rollup_chunks<<<warp_grid(rp.n_chunks, n_sms), 128, 0, s>>>(p, rp);
  k_rollup_segments<<<warp_grid(rp.n_seg1, n_sms), 128, 0, s>>>(
      nv, rp.part_v, rp.part_al, nullptr, rp.seg1_begin, rp.seg1_end, rp.n_seg1, rp.rows_v, rp.rows_al);
  k_rollup_segments<<<warp_grid(rp.n_seg2, n_sms), 128, 0, s>>>(
      nv, rp.rows_v, rp.rows_al, rp.seg2_perm, rp.seg2_begin, rp.seg2_end, rp.n_seg2,
      rp.rows_v + (uint64_t)rp.n_seg1 * nv, rp.rows_al + 2 * (uint64_t)rp.n_seg1);
  *launches += rp.n_chunks ? 3 : 2;
  return cudaGetLastError();
}

}  // namespace gpa

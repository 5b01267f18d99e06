// rollup.cu -- row a7: per-instruction blame vectors summed over program structure
// (line, loop exclusive/inclusive, function, kernel, Q16).
//
// Hand-written segmented reductions (no CUB), deterministic: every sum has a fixed order.
//   k_vrows            V[i] = {NCOL x (all, lat)} for every instruction, one
//                      thread per instruction with independent vector loads and 16-byte (all, lat)
//                      stores; this is also the instruction level of the rollup (gpa_instr_vector).
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

// one thread per instruction: the B row (64 B), the C row (16R B), class and self flags are
// loaded with independent loads before any store; the warp's 32 rows of V are staged in shared
// memory and written back as one contiguous, coalesced block (rows are consecutive in V).
// Same values as vvalue().
constexpr uint32_t kVrowsThreads = 128;
__global__ void __launch_bounds__(kVrowsThreads) k_vrows(DevProgram p, double *__restrict__ vbuf) {
  pdl_wait();
  extern __shared__ double2 vstage[];          // [kVrowsThreads / 32][32 rows][ncol]
  const uint32_t ncol = p.ncol, R = p.R, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double2 *ws = vstage + (size_t)warp * 32 * ncol;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; base < p.n; base += stride) {
    const uint32_t i = base + lane;
    if (i < p.n) {
      const double2 *b2 = reinterpret_cast<const double2 *>(p.B + 8 * (uint64_t)i);
      const double2 bm = b2[BG_MEM], be = b2[BG_EXEC], bw = b2[BG_WAR], bs = b2[BG_SYNC];
      const uint32_t cls = p.opclass[i], sf = p.selfm[i];
      const uint64_t *row = p.C + (uint64_t)i * 2 * R;
      uint64_t act[kReasonsMax], lat[kReasonsMax];
#pragma unroll
      for (uint32_t r = 1; r < kReasonsMax; ++r) {
        act[r] = r < R ? row[r] : 0ull;
        lat[r] = r < R ? row[R + r] : 0ull;
      }
      double2 *out = ws + (size_t)lane * ncol;
      const double2 z = make_double2(0.0, 0.0);
      out[COL_MEM_GLOBAL] = (cls != OC_LOCAL && cls != OC_CONSTANT) ? bm : z;
      out[COL_MEM_LOCAL] = cls == OC_LOCAL ? bm : z;
      out[COL_MEM_CONSTANT] = cls == OC_CONSTANT ? bm : z;
      out[COL_EXEC_SHARED] = cls == OC_SHARED ? be : z;
      out[COL_EXEC_ARITH] = cls != OC_SHARED ? be : z;
      out[COL_EXEC_WAR] = bw;
      out[COL_SYNC] = bs;
#pragma unroll
      for (uint32_t r = 1; r < kReasonsMax; ++r) {
        if (r >= R) break;
        const bool on = r > R_SYNC || ((sf >> (r - 1)) & 1u);
        out[6 + r] = on ? make_double2((double)(act[r] + lat[r]), (double)lat[r]) : z;
      }
    }
    __syncwarp();
    const uint32_t rows = min(32u, p.n - base);
    double2 *dst = reinterpret_cast<double2 *>(vbuf + (uint64_t)base * 2 * ncol);
    for (uint32_t x = lane; x < rows * ncol; x += 32) dst[x] = ws[x];
    __syncwarp();
  }
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
      for (; pos + 16 <= e; pos += 16) {   // 16 row loads in flight; member u still adds into a(u % 4)
        double x[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) x[u] = vals[(uint64_t)item(pos + u) * nv + s];
#pragma unroll
        for (int u = 0; u < 16; u += 4) {
          a0 = __dadd_rn(a0, x[u]);
          a1 = __dadd_rn(a1, x[u + 1]);
          a2 = __dadd_rn(a2, x[u + 2]);
          a3 = __dadd_rn(a3, x[u + 3]);
        }
      }
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

#ifndef GPA_ROLL_MEMBERS
#define GPA_ROLL_MEMBERS 16
#endif
constexpr int kRollMembers = GPA_ROLL_MEMBERS;   // members (row loads) in flight per lane

// chunk of <= 128 members: member ids are loaded once (4 per lane) and broadcast by shuffles, so
// the row loads of consecutive members are independent and stay in flight together
__global__ void __launch_bounds__(128) k_rollup_chunks(RollupPlan rp, uint32_t nv, const double *__restrict__ vbuf,
                                                       const uint64_t *__restrict__ AL) {
  pdl_wait();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t ch = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; ch < rp.n_chunks; ch += warps) {
    const uint32_t b = rp.chunk_begin[ch], len = rp.chunk_end[ch] - b;
    uint32_t ids[kChunk / 32];
#pragma unroll
    for (int t = 0; t < kChunk / 32; ++t) ids[t] = (lane + 32 * t < len) ? rp.order[b + lane + 32 * t] : 0u;
    for (uint32_t s0 = 0; s0 < nv + 2; s0 += 32) {   // uniform trip count: shuffles need all lanes
      const uint32_t s = s0 + lane;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};   // member u adds into acc[u % 4]: the order of the
      uint64_t al = 0;                          // four-accumulator scheme (a0..a3) is unchanged
      const bool is_v = s < nv, is_al = s >= nv && s < nv + 2;
#pragma unroll
      for (int t = 0; t < kChunk / 32; ++t) {
        const uint32_t m_end = len > 32u * t ? min(32u, len - 32u * t) : 0u;
        for (uint32_t m = 0; m < m_end; m += kRollMembers) {
          uint32_t id[kRollMembers];
#pragma unroll
          for (int u = 0; u < kRollMembers; ++u) id[u] = __shfl_sync(0xffffffffu, ids[t], (m + u) & 31);
          if (is_v) {
            double x[kRollMembers];
#pragma unroll
            for (int u = 0; u < kRollMembers; ++u) x[u] = m + u < m_end ? vbuf[(uint64_t)id[u] * nv + s] : 0.0;
#pragma unroll
            for (int u = 0; u < kRollMembers; ++u) acc[u & 3] = __dadd_rn(acc[u & 3], x[u]);
          } else if (is_al) {
            const uint32_t c = s - nv;
#pragma unroll
            for (int u = 0; u < kRollMembers; ++u)
              if (m + u < m_end) al += AL[2 * (uint64_t)id[u] + c];
          }
        }
      }
      if (is_v) rp.part_v[(uint64_t)ch * nv + s] = __dadd_rn(__dadd_rn(acc[0], acc[1]), __dadd_rn(acc[2], acc[3]));
      else if (is_al) rp.part_al[2 * (uint64_t)ch + (s - nv)] = al;
    }
  }
}

__global__ void __launch_bounds__(128) k_rollup_segments(uint32_t nv, const double *__restrict__ in_v,
                                                         const uint64_t *__restrict__ in_al,
                                                         const uint32_t *__restrict__ perm,
                                                         const uint32_t *__restrict__ seg_begin,
                                                         const uint32_t *__restrict__ seg_end, uint32_t n_seg,
                                                         const uint32_t *__restrict__ out_row,
                                                         double *__restrict__ out_v, uint64_t *__restrict__ out_al) {
  pdl_wait();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t sg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; sg < n_seg; sg += warps) {
    const uint64_t row = out_row ? out_row[sg] : sg;
    if (perm)
      warp_sum_rows(lane, nv, seg_begin[sg], seg_end[sg], [perm](uint32_t pos) { return perm[pos]; }, in_v, in_al,
                    out_v + row * nv, out_al + 2 * row);
    else
      warp_sum_rows(lane, nv, seg_begin[sg], seg_end[sg], [](uint32_t pos) { return pos; }, in_v, in_al,
                    out_v + row * nv, out_al + 2 * row);
  }
}

// packs of short segments (<= kChunk positions in all): one warp per pack, lane = value slot;
// member rows are fetched kRollMembers at a time across segment boundaries and added in member
// order into the current segment's sum, which is written to its row when the segment ends --
// the same left-to-right order as the oracle's per-instruction accumulation
__global__ void __launch_bounds__(128) k_rollup_packs(RollupPlan rp, uint32_t nv, const double *__restrict__ vbuf,
                                                      const uint64_t *__restrict__ AL) {
  pdl_wait();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t pk = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; pk < rp.n_packs; pk += warps) {
    const uint32_t sa = rp.pack_seg[pk], sb = rp.pack_seg[pk + 1];
    const uint32_t P0 = rp.segpos[sa], P1 = rp.segpos[sb], len = P1 - P0;
    if (len > (uint32_t)kChunk) continue;          // a long segment: chunked + k_rollup_segments
    uint32_t ids[kChunk / 32];
#pragma unroll
    for (int t = 0; t < kChunk / 32; ++t) ids[t] = (lane + 32 * t < len) ? rp.order[P0 + lane + 32 * t] : 0u;
    for (uint32_t s0 = 0; s0 < nv + 2; s0 += 32) {   // uniform trip count: shuffles need all lanes
      const uint32_t s = s0 + lane;
      const bool is_v = s < nv, is_al = s >= nv && s < nv + 2;
      uint32_t seg = sa, seg_end = rp.segpos[sa + 1];
      double acc = 0.0;
      uint64_t al = 0;
      auto flush_to = [&](uint32_t pos) {          // close every segment that ends at or before pos
        while (seg < sb && seg_end <= pos) {
          if (is_v) rp.rows_v[(uint64_t)seg * nv + s] = acc;
          else if (is_al) rp.rows_al[2 * (uint64_t)seg + (s - nv)] = al;
          acc = 0.0;
          al = 0;
          ++seg;
          if (seg < sb) seg_end = rp.segpos[seg + 1];
        }
      };
#pragma unroll
      for (int t = 0; t < kChunk / 32; ++t) {
        const uint32_t m_end = len > 32u * t ? min(32u, len - 32u * t) : 0u;
        for (uint32_t m = 0; m < m_end; m += kRollMembers) {
          uint32_t id[kRollMembers];
#pragma unroll
          for (int u = 0; u < kRollMembers; ++u) id[u] = __shfl_sync(0xffffffffu, ids[t], (m + u) & 31);
          double x[kRollMembers];
          uint64_t y[kRollMembers];
#pragma unroll
          for (int u = 0; u < kRollMembers; ++u) {
            const bool in = m + u < m_end;
            x[u] = (in && is_v) ? vbuf[(uint64_t)id[u] * nv + s] : 0.0;
            y[u] = (in && is_al) ? AL[2 * (uint64_t)id[u] + (s - nv)] : 0ull;
          }
#pragma unroll
          for (int u = 0; u < kRollMembers; ++u) {
            if (m + u >= m_end) break;
            flush_to(P0 + 32 * t + m + u);
            acc = __dadd_rn(acc, x[u]);
            al += y[u];
          }
        }
      }
      flush_to(P1);
    }
  }
}

inline uint32_t warp_grid(uint64_t warps, int n_sms) {
  const uint64_t blocks = (warps + 3) / 4;   // 128 threads = 4 warps per block
  return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(blocks, (uint64_t)n_sms * 32));
}

}  // namespace

cudaError_t launch_vrows(const DevProgram &p, double *vbuf, int n_sms, cudaStream_t s) {
  const uint64_t total = (uint64_t)p.n;
  const uint32_t g = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((total + kVrowsThreads - 1) / kVrowsThreads,
                                                                         (uint64_t)n_sms * 16));
  const size_t smem = (size_t)kVrowsThreads * p.ncol * sizeof(double2);   // 32 rows per warp
  cudaError_t e = cudaFuncSetAttribute(k_vrows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(p.n, k_vrows, g, kVrowsThreads, smem, s, p, vbuf);
}

// fork (optional, graph capture): the packs of short segments write rows disjoint from the
// chunked long segments', so they run on stream `side` between events fork / join
cudaError_t launch_rollup_fork(const DevProgram &p, const RollupPlan &rp, int n_sms, cudaStream_t s,
                               cudaStream_t side, cudaEvent_t fork, cudaEvent_t join, uint64_t *launches) {
  const uint32_t nv = 2 * p.ncol;
  cudaError_t e = launch_vrows(p, rp.vbuf, n_sms, s);
  if (e != cudaSuccess) return e;
  const bool split = side && rp.n_packs;
  if (split) {
    if ((e = cudaEventRecord(fork, s)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(side, fork, 0)) != cudaSuccess) return e;
  }
  cudaStream_t ps = split ? side : s;
  if (rp.n_packs) k_rollup_packs<<<warp_grid(rp.n_packs, n_sms), 128, 0, ps>>>(rp, nv, rp.vbuf, p.AL);
  if (split && (e = cudaEventRecord(join, side)) != cudaSuccess) return e;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (rp.n_chunks && (e = launch_pdl(p.n, k_rollup_chunks, warp_grid(rp.n_chunks, n_sms), 128, 0, s, rp, nv,
                                     (const double *)rp.vbuf, (const uint64_t *)p.AL)) != cudaSuccess)
    return e;
  if (rp.n_seg1 && (e = launch_pdl(p.n, k_rollup_segments, warp_grid(rp.n_seg1, n_sms), 128, 0, s, nv,
                                   (const double *)rp.part_v, (const uint64_t *)rp.part_al, (const uint32_t *)nullptr,
                                   (const uint32_t *)rp.seg1_begin, (const uint32_t *)rp.seg1_end, rp.n_seg1,
                                   (const uint32_t *)rp.seg1_id, rp.rows_v, rp.rows_al)) != cudaSuccess)
    return e;
  if (split && (e = cudaStreamWaitEvent(s, join, 0)) != cudaSuccess) return e;   // stage 2 reads the pack rows
  k_rollup_segments<<<warp_grid(rp.n_seg2, n_sms), 128, 0, s>>>(
      nv, rp.rows_v, rp.rows_al, rp.seg2_perm, rp.seg2_begin, rp.seg2_end, rp.n_seg2, nullptr,
      rp.rows_v + (uint64_t)rp.n_rows1 * nv, rp.rows_al + 2 * (uint64_t)rp.n_rows1);
  *launches += 2 + (rp.n_chunks ? 1 : 0) + (rp.n_packs ? 1 : 0) + (rp.n_seg1 ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_rollup(const DevProgram &p, const RollupPlan &rp, int n_sms, cudaStream_t s,
                          uint64_t *launches) {
  return launch_rollup_fork(p, rp, n_sms, s, nullptr, nullptr, nullptr, launches);
}

}  // namespace gpa

// rollup.cu -- row a7: per-instruction blame vectors summed over program structure
// (line, loop exclusive/inclusive, function, kernel, Q16).
//
// Hand-written segmented reductions (no CUB), deterministic: every sum has a fixed order.
//   k_rollup_tiles     one warp per tile of 32 consecutive instructions: lane = instruction builds
//                      V[i] = {NCOL x (all, lat)} from B, C, the class and the
//                      self flags into shared memory, then lane = value slot sums the tile's runs of
//                      equal line, equal innermost loop and equal function (create-time run lists)
//                      in member order -- a run that is its segment's only run is the segment's row,
//                      the others write partial rows.  B and C are read once, coalesced, in program
//                      order; V is never materialised in HBM.
//   k_rollup_segments  one warp per segment: stage 1 sums the partial rows of segments with several
//                      runs (functions, loops, lines that recur) in program order; stage 2 the
//                      loops-inclusive (preorder subtree ranges of the loop-exclusive rows) and the
//                      kernels (their function rows).
//   k_vrows            V for gpa_instr_vector (the instruction level, on request; not in the graph).
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
  double2 *vstage = &dyn_smem<double2>();      // [kVrowsThreads / 32][32 rows][ncol]
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
  // lane = value slot: slots < nv are the f64 values (fixed order: member u adds into a(u % 4)), the
  // two slots after them the u64 A / L sums; every slot walks the members with the same batched
  // 64-bit loads (16 in flight), so the A / L lanes no longer serialise behind the value lanes
  for (uint32_t s = lane; s < nv + 2; s += 32) {
    const bool isv = s < nv;
    const uint64_t *src = isv ? reinterpret_cast<const uint64_t *>(vals) : al;
    const uint32_t stride = isv ? nv : 2u, off = isv ? s : s - nv;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    uint64_t acc = 0;
    auto add = [&](double &a, uint64_t x) {
      if (isv) a = __dadd_rn(a, __longlong_as_double((long long)x));
      else acc += x;
    };
    uint32_t pos = b;
    for (; pos + 16 <= e; pos += 16) {   // 16 row loads in flight
      uint64_t x[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) x[u] = src[(uint64_t)item(pos + u) * stride + off];
#pragma unroll
      for (int u = 0; u < 16; u += 4) {
        add(a0, x[u]);
        add(a1, x[u + 1]);
        add(a2, x[u + 2]);
        add(a3, x[u + 3]);
      }
    }
    for (; pos + 4 <= e; pos += 4) {
      uint64_t x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = src[(uint64_t)item(pos + u) * stride + off];
      add(a0, x[0]);
      add(a1, x[1]);
      add(a2, x[2]);
      add(a3, x[3]);
    }
    for (; pos < e; ++pos) add(a0, src[(uint64_t)item(pos) * stride + off]);
    if (isv) out_v[s] = __dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3));
    else out_al[s - nv] = acc;
  }
}

__device__ __forceinline__ void body_rollup_segments(uint32_t nv, const double *__restrict__ in_v,
                                                         const uint64_t *__restrict__ in_al,
                                                         const uint32_t *__restrict__ perm,
                                                         const uint32_t *__restrict__ seg_begin,
                                                         const uint32_t *__restrict__ seg_end, uint32_t n_seg,
                                                         const uint32_t *__restrict__ out_row,
                                                         double *__restrict__ out_v, uint64_t *__restrict__ out_al, uint32_t bx, uint32_t gx) {
  pdl_wait();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = (gx * blockDim.x) >> 5;
  for (uint32_t sg = (bx * blockDim.x + threadIdx.x) >> 5; sg < n_seg; sg += warps) {
    const uint64_t row = out_row ? out_row[sg] : sg;
    if (perm)
      warp_sum_rows(lane, nv, seg_begin[sg], seg_end[sg], [perm](uint32_t pos) { return perm[pos]; }, in_v, in_al,
                    out_v + row * nv, out_al + 2 * row);
    else
      warp_sum_rows(lane, nv, seg_begin[sg], seg_end[sg], [](uint32_t pos) { return pos; }, in_v, in_al,
                    out_v + row * nv, out_al + 2 * row);
  }
}

__global__ void __launch_bounds__(128) k_rollup_segments(uint32_t nv, const double *__restrict__ in_v,
                                                         const uint64_t *__restrict__ in_al,
                                                         const uint32_t *__restrict__ perm,
                                                         const uint32_t *__restrict__ seg_begin,
                                                         const uint32_t *__restrict__ seg_end, uint32_t n_seg,
                                                         const uint32_t *__restrict__ out_row,
                                                         double *__restrict__ out_v, uint64_t *__restrict__ out_al) {
  body_rollup_segments(nv, in_v, in_al, perm, seg_begin, seg_end, n_seg, out_row, out_v, out_al, blockIdx.x, gridDim.x);
}

// one warp per tile of 32 instructions (4 warps per block): V rows built by lane = instruction into
// shared memory (the k_vrows arithmetic), then lane = value slot sums each run of the tile in member
// order and stores the run's row (or partial row) -- one coalesced row store per run
constexpr uint32_t kTileWarps = 4;
#ifndef GPA_ROLL_BATCH
#define GPA_ROLL_BATCH 8
#endif
constexpr uint32_t kRollBatch = GPA_ROLL_BATCH;   // count-row reasons loaded per batch (k_rollup_tiles)
// one tile: ws = the warp's [32 rows][ncol] double2 staging, wal = its [32][2] u64; kAcc: the tile's
// B rows come from the caller's registers (acc of the lane's instruction: the fused def + rollup
// tiles) instead of p.B
template <bool kAcc>
__device__ __forceinline__ void rollup_tile(const DevProgram &p, const RollupPlan &rp, uint32_t t, uint32_t lane,
                                            double2 *ws, uint64_t *wal, const double (&acc)[4][2]) {
  const uint32_t ncol = p.ncol, nv = 2 * ncol, R = p.R;
  const uint32_t i = 32 * t + lane;
  // the tile's run descriptors (at most 3 x 32: lines, loops, functions), one per lane, loaded
  // up front with the rows
  const uint32_t r0 = rp.tile_run_ptr[t], r1 = rp.tile_run_ptr[t + 1];
  uint32_t rbe[3], rdst[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const uint32_t r = r0 + 32 * k + lane;
    rbe[k] = r < r1 ? rp.run_be[r] : 0u;
    rdst[k] = r < r1 ? rp.run_dst[r] : 0u;
  }
  if (i < p.n) {
    double2 bm, be, bw, bs;
    if constexpr (kAcc) {
      bm = make_double2(acc[BG_MEM][0], acc[BG_MEM][1]);
      be = make_double2(acc[BG_EXEC][0], acc[BG_EXEC][1]);
      bw = make_double2(acc[BG_WAR][0], acc[BG_WAR][1]);
      bs = make_double2(acc[BG_SYNC][0], acc[BG_SYNC][1]);
    } else {
      const double2 *b2 = reinterpret_cast<const double2 *>(p.B + 8 * (uint64_t)i);
      bm = b2[BG_MEM]; be = b2[BG_EXEC]; bw = b2[BG_WAR]; bs = b2[BG_SYNC];
    }
    const uint32_t cls = p.opclass[i], sf = p.selfm[i];
    const uint64_t *row = p.C + (uint64_t)i * 2 * R;
    double2 *out = ws + (size_t)lane * ncol;
    const double2 z = make_double2(0.0, 0.0);
    out[COL_MEM_GLOBAL] = (cls != OC_LOCAL && cls != OC_CONSTANT) ? bm : z;
    out[COL_MEM_LOCAL] = cls == OC_LOCAL ? bm : z;
    out[COL_MEM_CONSTANT] = cls == OC_CONSTANT ? bm : z;
    out[COL_EXEC_SHARED] = cls == OC_SHARED ? be : z;
    out[COL_EXEC_ARITH] = cls != OC_SHARED ? be : z;
    out[COL_EXEC_WAR] = bw;
    out[COL_SYNC] = bs;
    // the count row in batches of kRollBatch reasons (all loads of a batch in flight together),
    // which bounds the live count registers; A_i, L_i are summed on the way and stored
    // as the instruction level of the A / L rollup (GPA_VIEW_INSTR_AL) unless k_summaries ran
    uint64_t a = 0, l = 0;
#pragma unroll
    for (uint32_t q0 = 0; q0 < kReasonsMax; q0 += kRollBatch) {
      if (q0 >= R) break;
      uint64_t act[kRollBatch], lat[kRollBatch];
#pragma unroll
      for (uint32_t u = 0; u < kRollBatch; ++u) {
        act[u] = q0 + u < R ? row[q0 + u] : 0ull;
        lat[u] = q0 + u < R ? row[R + q0 + u] : 0ull;
      }
#pragma unroll
      for (uint32_t u = 0; u < kRollBatch; ++u) {
        const uint32_t r = q0 + u;
        a += act[u];
        l += lat[u];
        if (r >= 1 && r < R) {
          const bool on = r > R_SYNC || ((sf >> (r - 1)) & 1u);
          out[6 + r] = on ? make_double2((double)(act[u] + lat[u]), (double)lat[u]) : z;
        }
      }
    }
    if (!p.al_pre) reinterpret_cast<ulonglong2 *>(p.AL)[i] = make_ulonglong2(a, l);
    wal[2 * lane] = a;
    wal[2 * lane + 1] = l;
  }
  __syncwarp();
  const double *wv = reinterpret_cast<const double *>(ws);
  for (uint32_t s0 = 0; s0 < nv + 2; s0 += 32) {
    const uint32_t s = s0 + lane;
    for (uint32_t r = r0; r < r1; ++r) {
      // the run's descriptor from the lane that loaded it (a dependent global load per run was
      // the serial tail of this loop)
      const uint32_t k = r - r0, src = k & 31u;
      const uint32_t be2 = __shfl_sync(0xffffffffu, k < 32 ? rbe[0] : k < 64 ? rbe[1] : rbe[2], src);
      const uint32_t dst = __shfl_sync(0xffffffffu, k < 32 ? rdst[0] : k < 64 ? rdst[1] : rdst[2], src);
      const uint32_t b = be2 & 0xffu, e = be2 >> 8;
      const bool part = (dst & kPartialBit) != 0;
      const uint64_t row_id = dst & ~kPartialBit;
      if (s < nv) {
        double acc_v = 0.0;
        for (uint32_t m = b; m < e; ++m) acc_v = __dadd_rn(acc_v, wv[(size_t)m * nv + s]);
        (part ? rp.part_v : rp.rows_v)[row_id * nv + s] = acc_v;
      } else if (s < nv + 2) {
        uint64_t acc_u = 0;
        for (uint32_t m = b; m < e; ++m) acc_u += wal[2 * m + (s - nv)];
        (part ? rp.part_al : rp.rows_al)[2 * row_id + (s - nv)] = acc_u;
      }
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void body_rollup_tiles(DevProgram p, RollupPlan rp, uint32_t bx, uint32_t gx) {
  pdl_wait();
  double2 *tstage = &dyn_smem<double2>();      // [kTileWarps][32 rows][ncol] + [kTileWarps][32][2] u64
  const uint32_t ncol = p.ncol, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2 *ws = tstage + (size_t)warp * 32 * ncol;
  uint64_t *wal = reinterpret_cast<uint64_t *>(tstage + (size_t)kTileWarps * 32 * ncol) + (size_t)warp * 64;
  const uint32_t warps = gx * kTileWarps;
  const double none[4][2] = {};
  for (uint32_t t = bx * kTileWarps + warp; t < rp.n_tiles; t += warps) rollup_tile<false>(p, rp, t, lane, ws, wal, none);
}

// Def reduction and rollup fused per tile (gpa_analyze): the rollup's tiles are the def tiles (32
// consecutive instructions), so a warp reduces its 32 defs (def_tile_acc: B stored for the views)
// and builds the same 32 V rows from the sums still in registers -- one kernel and one dependent
// level fewer in the graph, and no re-read of B.  Per warp one shared-memory region, used by the
// def staging, then by the V staging.
__host__ __device__ inline size_t def_roll_warp_bytes(uint32_t ncol) {
  const size_t roll = (size_t)32 * ncol * sizeof(double2) + 64 * sizeof(uint64_t);
  const size_t def = sizeof(DefWarpSmem);
  return ((roll > def ? roll : def) + 15) & ~(size_t)15;
}
__device__ __forceinline__ void body_def_rollup_tiles(DevProgram p, RollupPlan rp, uint32_t bx, uint32_t gx) {
  pdl_wait();
  uint8_t *base = &dyn_smem<uint8_t>();
  const uint32_t ncol = p.ncol, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t *region = base + (size_t)warp * def_roll_warp_bytes(ncol);
  DefWarpSmem &dsm = *reinterpret_cast<DefWarpSmem *>(region);
  double2 *ws = reinterpret_cast<double2 *>(region);
  uint64_t *wal = reinterpret_cast<uint64_t *>(region + (size_t)32 * ncol * sizeof(double2));
  const uint32_t warps = gx * kTileWarps;
  for (uint32_t t = bx * kTileWarps + warp; t < rp.n_tiles; t += warps) {
    double acc[4][2];
    def_tile_acc(p, t, lane, dsm, acc);   // ends converged: the region is free for the V rows
    rollup_tile<true>(p, rp, t, lane, ws, wal, acc);
  }
}

__global__ void __launch_bounds__(32 * kTileWarps) k_rollup_tiles(DevProgram p, RollupPlan rp) {
  body_rollup_tiles(p, rp, blockIdx.x, gridDim.x);
}

__global__ void __launch_bounds__(32 * kTileWarps) k_def_rollup_tiles(DevProgram p, RollupPlan rp) {
  body_def_rollup_tiles(p, rp, blockIdx.x, gridDim.x);
}

inline uint32_t warp_grid(uint64_t warps, int n_sms) {
  const uint64_t blocks = (warps + 3) / 4;   // 128 threads = 4 warps per block
  return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(blocks, (uint64_t)n_sms * 32));
}

}  // namespace

#ifndef GPA_FUSED_TU
cudaError_t launch_vrows(const DevProgram &p, double *vbuf, int n_sms, cudaStream_t s) {
  const uint64_t total = (uint64_t)p.n;
  const uint32_t g = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((total + kVrowsThreads - 1) / kVrowsThreads,
                                                                         (uint64_t)n_sms * 16));
  const size_t smem = (size_t)kVrowsThreads * p.ncol * sizeof(double2);   // 32 rows per warp
  cudaError_t e = cudaFuncSetAttribute(k_vrows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(p.n, k_vrows, g, kVrowsThreads, smem, s, p, vbuf);
}

cudaError_t launch_rollup(const DevProgram &p, const RollupPlan &rp, int n_sms, cudaStream_t s,
                          uint64_t *launches, bool with_def) {
  const uint32_t nv = 2 * p.ncol;
  auto tiles_kernel = with_def ? k_def_rollup_tiles : k_rollup_tiles;
  const size_t smem = with_def ? (size_t)kTileWarps * def_roll_warp_bytes(p.ncol)
                               : (size_t)kTileWarps * 32 * p.ncol * sizeof(double2) + (size_t)kTileWarps * 64 * sizeof(uint64_t);
  cudaError_t e = cudaFuncSetAttribute(tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const uint32_t g = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((rp.n_tiles + kTileWarps - 1) / kTileWarps,
                                                                         (uint64_t)n_sms * 16));
  if (rp.n_tiles && (e = launch_pdl(p.n, tiles_kernel, g, 32 * kTileWarps, smem, s, p, rp)) != cudaSuccess) return e;
  // stage 1: segments with several runs (and empty ones) from their partial rows
  if (rp.n_seg1 && (e = launch_pdl(p.n, k_rollup_segments, warp_grid(rp.n_seg1, n_sms), 128, 0, s, nv,
                                   (const double *)rp.part_v, (const uint64_t *)rp.part_al,
                                   (const uint32_t *)rp.seg1_perm, (const uint32_t *)rp.seg1_begin,
                                   (const uint32_t *)rp.seg1_end, rp.n_seg1, (const uint32_t *)rp.seg1_id, rp.rows_v,
                                   rp.rows_al)) != cudaSuccess)
    return e;
  // stage 2: loops inclusive and kernels over the stage-1 rows
  if (rp.n_seg2 && (e = launch_pdl(p.n, k_rollup_segments, warp_grid(rp.n_seg2, n_sms), 128, 0, s, nv,
                                   (const double *)rp.rows_v, (const uint64_t *)rp.rows_al,
                                   (const uint32_t *)rp.seg2_perm, (const uint32_t *)rp.seg2_begin,
                                   (const uint32_t *)rp.seg2_end, rp.n_seg2, (const uint32_t *)nullptr,
                                   rp.rows_v + (uint64_t)rp.n_rows1 * nv, rp.rows_al + 2 * (uint64_t)rp.n_rows1)) != cudaSuccess)
    return e;
  *launches += (rp.n_tiles ? 1 : 0) + (rp.n_seg1 ? 1 : 0) + (rp.n_seg2 ? 1 : 0);
  return cudaGetLastError();
}

#endif  // GPA_FUSED_TU

}  // namespace gpa

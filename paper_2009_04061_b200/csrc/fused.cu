// fused.cu -- the whole analysis (rows a2-a8) of a small program as ONE cooperative launch.
//
// For programs of a few thousand instructions (config 2: 2,000 instructions, ~3,500 edges) every
// analysis kernel does microseconds of work, and the 12-launch graph of gpa_analyze is bound by
// launch and drain latency, not by bytes.  k_analyze_fused runs the same device bodies as those
// kernels (blame.cu, rollup.cu and estimate.cu are compiled into this translation unit with their
// host launchers left out) on one persistent grid of 128-thread CTAs, in the graph's dependency
// order, with a grid-wide barrier between dependent phases:
//
//   1  blame tiles (rules 1-3, Eq. 1 shares, self flags)
//   2  def reduction (B)            | estimate rows / edges (matched samples per item)
//   3  rollup tiles (+ A_i, L_i)    | segment sums stage 1 (loops exclusive, functions)
//   4  rollup segments stage 1      | segment sums stage 2 (loops inclusive, kernels)
//   5  rollup segments stage 2
//   6  estimates (Eqs. 2-5, 10)
//
// Every body is the one the multi-kernel graph runs, with the same arithmetic and summation order,
// so both paths produce bit-identical results (tests/test_gpu_fused.py).
#define GPA_FUSED_TU
#include "blame.cu"
#include "rollup.cu"
#include "estimate.cu"

#include <cstdlib>

#include <cooperative_groups.h>

namespace gpa {
namespace {

constexpr uint32_t kFusedThreads = 128;   // every body is written for 128-thread CTAs (4 warps)

#ifdef GPA_FUSED_TIMING
// phase end times (globaltimer, ns) seen by CTA 0 (tuning: read with gpa_debug_fused_timing)
__device__ unsigned long long g_fused_t[16];
__device__ __forceinline__ void fmark(int i) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_fused_t[i] = t;
  }
}
#define FMARK(i) fmark(i)
#else
#define FMARK(i) do {} while (0)
#endif

__global__ void __launch_bounds__(kFusedThreads) k_analyze_fused(DevProgram p, RollupPlan rp, EstimatePlan ep,
                                                                 SegLaunch s1, SegLaunch s2, uint32_t any_slot) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  const uint32_t bx = blockIdx.x, gx = gridDim.x, nv = 2 * p.ncol;
  const bool est = ep.n_pat != 0;
  FMARK(0);
  if (p.al_pre) {
    body_summaries(p.C, p.n, p.R, p.AL, bx, gx);
    grid.sync();
    body_blame_tiles<true>(p, bx, gx);
  } else {
    body_blame_tiles<false>(p, bx, gx);
  }
  FMARK(1);
  grid.sync();
  FMARK(2);
  body_def_tiles(p, bx, gx);
  if (est) {
    body_est_rows(p, ep, bx, gx);
    if (any_slot) body_est_edges(p, ep, bx, gx);
  }
  FMARK(3);
  grid.sync();
  FMARK(4);
  if (rp.n_tiles) body_rollup_tiles(p, rp, bx, gx);
  if (est)
    for (uint32_t f = 0; f < s1.n_fam; ++f) body_segsum(s1, f, bx, gx);
  FMARK(5);
  grid.sync();
  FMARK(6);
  if (rp.n_seg1)
    body_rollup_segments(nv, rp.part_v, rp.part_al, rp.seg1_perm, rp.seg1_begin, rp.seg1_end, rp.n_seg1, rp.seg1_id,
                         rp.rows_v, rp.rows_al, bx, gx);
  if (est)
    for (uint32_t f = 0; f < s2.n_fam; ++f) body_segsum(s2, f, bx, gx);
  FMARK(7);
  grid.sync();
  FMARK(8);
  if (rp.n_seg2)
    body_rollup_segments(nv, rp.rows_v, rp.rows_al, rp.seg2_perm, rp.seg2_begin, rp.seg2_end, rp.n_seg2, nullptr,
                         rp.rows_v + (uint64_t)rp.n_rows1 * nv, rp.rows_al + 2 * (uint64_t)rp.n_rows1, bx, gx);
  if (est) {
    FMARK(9);
    grid.sync();
    FMARK(10);
    body_est_final(p, ep, bx, gx);
  }
  FMARK(15);
}

}  // namespace

bool fused_feasible(uint32_t n_pat) { return (n_pat + kEstGroup - 1) / kEstGroup <= kFusedThreads / 32; }

// one dynamic region, reused phase by phase (the grid barriers order every phase's last use before
// the next phase's first)
size_t fused_smem_bytes(const DevProgram &p) {
  const size_t roll = (size_t)kTileWarps * 32 * p.ncol * sizeof(double2) + (size_t)kTileWarps * 64 * sizeof(uint64_t);
  return std::max({roll, sizeof(BlameSmem), sizeof(DefSmem)});
}

cudaError_t launch_analyze_fused(const DevProgram &p, const RollupPlan &rp, const EstimatePlan &ep, int n_sms,
                                 uint32_t max_ctas, cudaStream_t s, uint64_t *launches) {
  static_assert(32 * kBlameWarps == kFusedThreads && 32 * kTileWarps == kFusedThreads, "bodies assume 4 warps");
  if (!fused_feasible(ep.n_pat)) return cudaErrorInvalidValue;   // one warp per pattern group
  const size_t smem = fused_smem_bytes(p);
  cudaError_t e = cudaFuncSetAttribute(k_analyze_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_analyze_fused, kFusedThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  // enough CTAs for the widest phase (32-row tiles, 4 per CTA), never more than can be co-resident
  uint64_t want = std::max<uint64_t>(1, ((uint64_t)p.n + 127) / 128);
  if (const char *env = getenv("GPA_FUSED_GRID")) want = strtoull(env, nullptr, 10);   // tuning probe
  const uint32_t grid = (uint32_t)std::min<uint64_t>({want, (uint64_t)per_sm * n_sms, (uint64_t)max_ctas});
  SegLaunch s1, s2;
  make_seg_launches(p, ep, s1, s2);
  DevProgram pa = p;
  RollupPlan ra = rp;
  EstimatePlan ea = ep;
  uint32_t any_slot = 0;
  for (uint32_t q = 0; q < ep.n_pat; ++q) any_slot |= ep.loop_slot[q] >= 0 && p.E ? 1u : 0u;
  void *args[] = {&pa, &ra, &ea, &s1, &s2, &any_slot};
  e = cudaLaunchCooperativeKernel((const void *)k_analyze_fused, dim3(grid), dim3(kFusedThreads), args, smem, s);
  *launches += 1;
  return e;
}

#ifdef GPA_FUSED_TIMING
extern "C" int gpa_debug_fused_timing(unsigned long long *out) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(out, g_fused_t, sizeof(g_fused_t));
}
#endif

}  // namespace gpa

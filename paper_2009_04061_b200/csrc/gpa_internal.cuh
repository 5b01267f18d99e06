// gpa_internal.cuh -- private declarations shared by the runtime and the sm_100a kernels.
// Product code (the CUDA path).  Independent of oracle/ (no shared code or tables).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <utility>

#include <vector>

#include "../../include/gpa.h"

namespace gpa {

constexpr int kReasonsMax = 16;
constexpr int kColsMax = kReasonsMax + 6;   // NCOL = R + 6
constexpr int kSlotsMax = 2 * kColsMax + 2; // V values + (A, L)
constexpr int kPatternsMax = 32;
#ifndef GPA_ROLL_CHUNK
#define GPA_ROLL_CHUNK 64
#endif
constexpr int kChunk = GPA_ROLL_CHUNK;      // rollup chunk length (instructions), a multiple of 32
constexpr int kMaxIngestCtas = 256;         // per-CTA partial tables reserved (smem variant)
constexpr size_t kSmemTableMax = 224 * 1024;// largest CTA-private table (bytes; sm_100a opt-in is 227 KB)
// Programmatic dependent launch (sm_90+): the analysis kernels start with griddepcontrol.wait, so
// a kernel launched with the programmatic-serialization attribute may be scheduled while its
// predecessor drains and waits for its completion (and memory flush) before touching any data.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// The tile kernels carve their staging buffers out of dynamic shared memory (a struct per kernel),
// so the fused analysis kernel, whose phases run one after another, reuses one region for all.
#ifdef __CUDACC__
template <typename T>
__device__ __forceinline__ T &dyn_smem() {
  extern __shared__ __align__(16) uint8_t gpa_dyn_smem[];
  return *reinterpret_cast<T *>(gpa_dyn_smem);
}
#endif
#ifndef GPA_PDL
#define GPA_PDL 1
#endif
// Only for programs below kPdlMaxInstr instructions: there the analysis kernels are short and
// latency-bound (config 3: 92 -> 82 us); on config 4's 4.5 M instructions the overlap cost 1 %.
constexpr uint32_t kPdlMaxInstr = 1u << 20;
#ifndef GPA_FUSED_CTAS
#define GPA_FUSED_CTAS 4096
#endif
constexpr uint32_t kFusedMaxCtas = GPA_FUSED_CTAS;   // grid of the fused analysis kernel (at most)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(uint32_t n_instr, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = GPA_PDL && n_instr < kPdlMaxInstr;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
// partitioned ingest (variant P): bucket exchange through L2
// GPA_* macros below (and in ingest.cu / rollup.cu / estimate.cu / runtime.cu) are tuning knobs:
// tools/variant_build.py builds alternative libraries with other values for A/B timing on the GPU
// (tools/variant_time.py, tools/seg_time.py); the defaults are the measured best.
#ifndef GPA_PART_THREADS
#define GPA_PART_THREADS 1024
#endif
constexpr int kPartThreads = GPA_PART_THREADS;
#ifndef GPA_PART_CHUNK
#define GPA_PART_CHUNK 6400
#endif
constexpr int kPartChunk = GPA_PART_CHUNK;  // largest exchange chunk: records per CTA per round (50 KB)
#ifndef GPA_PART_BUFS
#define GPA_PART_BUFS 16
#endif
constexpr int kPartBufs = GPA_PART_BUFS;    // exchange buffers in flight
#ifndef GPA_PART_CAP
#define GPA_PART_CAP 56
#endif
constexpr int kPartCap = GPA_PART_CAP;                // keys per (src, dst) slot per chunk (mean 43 at G=148);
                                            // excess -> L2 atomics
constexpr int kPartMaxCtas = 160;           // < 255: bucket ids fit a byte
size_t part_smem_bytes(uint32_t bpb, uint32_t G);
constexpr size_t kPartZeroBytes = 64 * 1024;  // >= one staging buffer of any exchange shape

// stall reasons
constexpr uint32_t R_NONE = 0, R_MEM = 1, R_EXEC = 2, R_SYNC = 3;
// opcode classes
constexpr uint32_t OC_GLOBAL = 0, OC_LOCAL = 1, OC_SHARED = 2, OC_CONSTANT = 3, OC_TEXTURE = 4,
                   OC_SYNC = 9, OC_COUNT = 11;
constexpr uint8_t K_WAR = 8;
// blame column indices
constexpr uint32_t COL_MEM_GLOBAL = 0, COL_MEM_LOCAL = 1, COL_MEM_CONSTANT = 2,
                   COL_EXEC_SHARED = 3, COL_EXEC_ARITH = 4, COL_EXEC_WAR = 5, COL_SYNC = 6,
                   COL_MEM_SELF = 7, COL_PASS0 = 10;
// per-instruction edge-blame groups (GPA_VIEW_INSTR_BLAME)
constexpr uint32_t BG_MEM = 0, BG_EXEC = 1, BG_WAR = 2, BG_SYNC = 3;

enum : int { ST_COUNTS = 1, ST_BLAMED = 2, ST_AGGREGATED = 4, ST_PATTERNS = 8, ST_ESTIMATED = 16, ST_ADVISED = 32 };
enum : int { VAR_SMEM = 0, VAR_PART = 1, VAR_L2 = 2 };

// Device-side view of a program: plain pointers into the workspace.
// The fields a def-use edge gathers from its def (blame: latency, class; estimate matching: class,
// flags, loop), packed per instruction at create time so a gather is one 16-byte load (one
// sector) instead of one per array
struct __align__(16) DefInfo {
  uint32_t latency;
  int32_t loop;
  uint32_t cls_flags;   // opclass | iflags << 8
  uint32_t pad;
};

struct DevProgram {
  uint32_t n, E, R, ncol, n_lines, n_loops, n_funcs, n_kernels;
  const uint8_t *opclass, *iflags;
  const uint32_t *latency, *line_id;
  const int32_t *loop_id;
  const uint32_t *func_begin, *kernel_func_begin, *kernel_grid_blocks;
  const uint32_t *row_ptr, *edge_def, *edge_min, *edge_max, *edge_use;
  const int32_t *edge_dom, *edge_lca;
  const uint8_t *edge_kind;
  const uint32_t *def_ptr, *def_perm;
  uint64_t *C, *stats, *AL;
  uint32_t *partials;               // [kMaxIngestCtas][n*2R] per-CTA tables (smem variant)
  uint32_t *part_x;                 // [kPartBufs][kPartMaxCtas dst][G src][kPartCap] 2-byte exchange keys
  unsigned int *part_sync;          // [2*kPartBufs]: per exchange buffer, CTAs that produced / consumed it
  const uint16_t *part_zero;        // [kPartZeroBytes] zeros (GPA_PART_TMA_ZERO staging clears)
  uint8_t *cand, *selfm;
  double *share, *B;
  uint32_t al_pre;                  // 1: k_summaries fills AL before the blame (n >= kPdlMaxInstr)
  const DefInfo *dinfo;             // [n] packed latency / loop / class / flags
};

// Rollup plan (create-time).  Tiles of 32 consecutive instructions; in each tile the
// maximal runs of equal line, equal innermost loop (loop members only) and equal function.  A run
// whose segment (line / loop-exclusive / function) has no other run is written straight into the
// segment's row; the other runs write partial rows, summed per segment in program order (stage 1).
struct RollupPlan {
  const uint32_t *tile_run_ptr; // [n_tiles+1] runs of tile t
  const uint32_t *run_be;       // [n_runs] begin | end << 8 (offsets in the tile, end exclusive)
  const uint32_t *run_dst;      // [n_runs] row id, or kPartialBit | partial row id
  uint32_t n_tiles;
  double *part_v;               // [n_partials][2*ncol]
  uint64_t *part_al;            // [n_partials][2]
  // stage 1: segments with 0 or >= 2 runs, summed over their partial rows (seg1_perm positions)
  const uint32_t *seg1_perm, *seg1_begin, *seg1_end, *seg1_id;
  uint32_t n_seg1, n_rows1;
  // stage 2: segments (loops incl, kernels) over rows via perm -> rows [n_rows1, n_rows1 + n_seg2)
  const uint32_t *seg2_perm, *seg2_begin, *seg2_end;
  uint32_t n_seg2;
  double *rows_v;               // [n_rows][2*ncol]
  uint64_t *rows_al;            // [n_rows][2]
};
constexpr uint32_t kPartialBit = 0x80000000u;

// per-kernel occupancy (gpa_set_launches) for parallel_rule 3 / 4
struct KernOcc {
  double W, W_new_block, W_new_thread;
  uint32_t match_block, match_thread;
};

struct EstimatePlan {
  const gpa_pattern *pats;
  const KernOcc *occ;           // [n_kernels]; zeroed until gpa_set_launches
  uint32_t n_pat;
  int8_t loop_slot[kPatternsMax];   // pattern -> slot in mval (models 2, 4) or -1
  double *mval;                 // [n_pat][E + n]: edge part then instruction part
  double *mrow;                 // [n_pat][n]: per use row (edges of the row + instruction part)
  const uint32_t *loop_items;   // [n_items] item ids (edge e, or E + instruction) by scope loop
  const uint32_t *loop_item_ptr;// [n_loops+1]
  const uint32_t *pre_perm;     // [n_loops] loops in preorder
  const uint32_t *pre_begin, *pre_end; // [n_loops] subtree range in preorder positions
  const uint32_t *kloop_ptr, *kloops;  // kernel -> its loops
  const int32_t *loop_func;     // [n_loops]
  double *lM_excl, *lM_incl;    // [n_pat][n_loops]
  double *fM, *kM;              // [n_pat][n_funcs], [n_pat][n_kernels]
  const uint64_t *loop_incl_al, *func_al, *kern_al;
  gpa_estimate_out *out;        // [n_kernels][n_pat]
};

// advice (NEXT #2): hotspots [n_kernels][n_pat][kTopKMax], counts, ranks, coverage
constexpr uint32_t kTopKMax = GPA_TOP_K_MAX;
struct AdvicePlan {
  gpa_hotspot *hot;
  uint32_t *n_hot;              // [n_kernels][n_pat]
  uint32_t *rank;               // [n_kernels][n_pat] pattern at each rank
  gpa_coverage *cov;            // [n_kernels]
  uint32_t top_k;
};

// kernel launchers (return cudaError_t of the launch)
cudaError_t launch_ingest(const DevProgram &p, int variant, const void *records, uint64_t n,
                          int n_sms, size_t smem_optin, cudaStream_t s);
cudaError_t launch_blame(const DevProgram &p, int n_sms, cudaStream_t s, uint64_t *launches);
cudaError_t launch_blame_rows(const DevProgram &p, int n_sms, cudaStream_t s, uint64_t *launches);
cudaError_t launch_def_reduce(const DevProgram &p, int n_sms, cudaStream_t s, uint64_t *launches);
cudaError_t launch_estimate_sums(const DevProgram &p, const EstimatePlan &ep, int n_sms, cudaStream_t s,
                                 uint64_t *launches);
cudaError_t launch_estimate_final(const DevProgram &p, const EstimatePlan &ep, int n_sms, cudaStream_t s,
                                  uint64_t *launches);
// with_def: the def reduction runs inside the rollup tiles (k_def_rollup_tiles), replacing
// launch_def_reduce before it
cudaError_t launch_rollup(const DevProgram &p, const RollupPlan &rp, int n_sms, cudaStream_t s,
                          uint64_t *launches, bool with_def = false);
cudaError_t launch_estimate(const DevProgram &p, const EstimatePlan &ep, int n_sms,
                            cudaStream_t s, uint64_t *launches);
cudaError_t launch_vrows(const DevProgram &p, double *vbuf, int n_sms, cudaStream_t s);
cudaError_t launch_slice(const gpa_sass_desc *h, uint32_t *h_row_ptr, uint64_t cap_edges, uint32_t *h_def,
                         uint8_t *h_kind, uint32_t *h_min, uint32_t *h_max, int32_t *h_dom, uint64_t *n_edges,
                         int n_sms, cudaStream_t st, int *status);
cudaError_t launch_simulate(const gpa_sass_desc *h, const uint8_t *h_cls, const uint32_t *h_lat, uint32_t func,
                            const gpa_simcfg &cfg, uint32_t n_sm, uint64_t cap, gpa_sample *d_out, int32_t *d_truth,
                            uint64_t *h_counts, cudaStream_t st);
cudaError_t launch_advice(const DevProgram &p, const EstimatePlan &ep, const AdvicePlan &ap, cudaStream_t s,
                          uint64_t *launches);
cudaError_t launch_ingest_segments(const DevProgram &p, const void *records, uint64_t n, const uint64_t *seg_begin,
                                   const uint32_t *seg_kernel, uint32_t n_seg, uint32_t pc_base, uint32_t max_tab_bins,
                                   int n_sms, cudaStream_t s);
size_t ingest_smem_bytes(const DevProgram &p);
// the whole analysis as one cooperative launch (fused.cu; small programs, <= 16 patterns)
bool fused_feasible(uint32_t n_pat);
cudaError_t launch_analyze_fused(const DevProgram &p, const RollupPlan &rp, const EstimatePlan &ep, int n_sms,
                                 uint32_t max_ctas, cudaStream_t s, uint64_t *launches);
bool part_feasible(const DevProgram &p, int n_sms, size_t smem_optin);

#ifdef __CUDACC__
// Full per-instruction vector V[i][NCOL][2] from B, self flags and C.
__device__ __forceinline__ double vvalue(const DevProgram &p, uint32_t i, uint32_t col, uint32_t c) {
  const uint32_t cls = p.opclass[i];
  if (col < 7) {
    const double *b = p.B + 8 * (uint64_t)i;
    switch (col) {
      case COL_MEM_GLOBAL: return (cls != OC_LOCAL && cls != OC_CONSTANT) ? b[2 * BG_MEM + c] : 0.0;
      case COL_MEM_LOCAL: return cls == OC_LOCAL ? b[2 * BG_MEM + c] : 0.0;
      case COL_MEM_CONSTANT: return cls == OC_CONSTANT ? b[2 * BG_MEM + c] : 0.0;
      case COL_EXEC_SHARED: return cls == OC_SHARED ? b[2 * BG_EXEC + c] : 0.0;
      case COL_EXEC_ARITH: return cls != OC_SHARED ? b[2 * BG_EXEC + c] : 0.0;
      case COL_EXEC_WAR: return b[2 * BG_WAR + c];
      default: return b[2 * BG_SYNC + c];
    }
  }
  const uint32_t r = col - 6;   // 7..9 -> MEM..SYNC (self); >= 10 -> pass-through reason
  if (col < COL_PASS0 && !((p.selfm[i] >> (r - 1)) & 1u)) return 0.0;
  const uint64_t *row = p.C + (uint64_t)i * 2 * p.R;
  const uint64_t lat = row[p.R + r];
  return (double)(c ? lat : row[r] + lat);
}


// ---- def-side reduction (rows a5-a6), shared by the def tiles (blame.cu) and the
// fused def + rollup tiles (rollup.cu): one def's S_j[r]*share and SL_j[r]*share over its
// out-edges in def-major order, summed into its four Fig. 6 groups
__device__ __forceinline__ void def_acc_one(const DevProgram &p, uint32_t i, double (&acc)[4][2]) {
#pragma unroll
  for (int g = 0; g < 4; ++g) acc[g][0] = acc[g][1] = 0.0;
  for (uint32_t k = p.def_ptr[i]; k < p.def_ptr[i + 1]; ++k) {
    const uint32_t e = p.def_perm[k];
    const uint32_t m = p.cand[e];
    if (!m) continue;
    const uint64_t *row = p.C + (uint64_t)p.edge_use[e] * 2 * p.R;
#pragma unroll
    for (uint32_t r = R_MEM; r <= R_SYNC; ++r) {
      if (!(m & (1u << (r - 1)))) continue;
      const double sh = p.share[3 * (uint64_t)e + (r - 1)];
      const uint64_t lat = row[p.R + r], all = row[r] + lat;
      const uint32_t g = r == R_MEM ? BG_MEM : r == R_SYNC ? BG_SYNC : ((p.edge_kind[e] & K_WAR) ? BG_WAR : BG_EXEC);
      acc[g][0] = __dadd_rn(acc[g][0], __dmul_rn((double)all, sh));
      acc[g][1] = __dadd_rn(acc[g][1], __dmul_rn((double)lat, sh));
    }
  }
}
__device__ __forceinline__ void store_B(const DevProgram &p, uint32_t i, const double (&acc)[4][2]) {
  double2 *out = reinterpret_cast<double2 *>(p.B + 8 * (uint64_t)i);
#pragma unroll
  for (int g = 0; g < 4; ++g) out[g] = make_double2(acc[g][0], acc[g][1]);
}

// Warp-cooperative def reduction of a tile of 32 consecutive defs.  (1) lanes over the tile's
// out-edge positions (def-major order, coalesced def_perm): the products S_j[r]*share and
// SL_j[r]*share of every candidate reason, gathered from the use rows by 32 lanes at once and staged
// in shared memory with the Fig. 6 group of the EXEC reason; (2) lane = def: the sums over its
// positions in order, reasons MEM, EXEC, SYNC -- the sequential order of def_acc_one, so B is
// bit-identical.  Tiles with more than kDefTileEdges positions take def_acc_one per lane.  Stores
// B and leaves the lane's def sums in acc (i < n); ends with the warp converged.
constexpr uint32_t kDefTileEdges = 128;
struct DefWarpSmem {
  double2 prod[3][kDefTileEdges];   // (all, lat) * share per dependency reason
  uint8_t m[kDefTileEdges];         // candidate mask | exec group is WAR << 3
};
__device__ __forceinline__ void def_tile_acc(const DevProgram &p, uint32_t tile, uint32_t lane, DefWarpSmem &S,
                                             double (&acc)[4][2]) {
  const uint32_t i0 = tile * 32, i = i0 + lane;
  const uint32_t K0 = p.def_ptr[i0], K1 = p.def_ptr[min(i0 + 32, p.n)];
  if (K1 - K0 > kDefTileEdges) {   // rare: a long tile
    if (i < p.n) {
      def_acc_one(p, i, acc);
      store_B(p, i, acc);
    }
    __syncwarp();
    return;
  }
  // (1) lanes over positions
  for (uint32_t k = K0 + lane; k < K1; k += 32) {
    const uint32_t e = p.def_perm[k];
    const uint32_t m = p.cand[e];
    uint32_t mm = m;
    if (m) {
      const uint64_t *row = p.C + (uint64_t)p.edge_use[e] * 2 * p.R;
      if (p.edge_kind[e] & K_WAR) mm |= 8u;
#pragma unroll
      for (uint32_t r = R_MEM; r <= R_SYNC; ++r) {
        if (!(m & (1u << (r - 1)))) continue;
        const double sh = p.share[3 * (uint64_t)e + (r - 1)];
        const uint64_t lat = row[p.R + r], all = row[r] + lat;
        S.prod[r - 1][k - K0] = make_double2(__dmul_rn((double)all, sh), __dmul_rn((double)lat, sh));
      }
    }
    S.m[k - K0] = (uint8_t)mm;
  }
  __syncwarp();
  // (2) lane = def: sums in position order
  if (i < p.n) {
#pragma unroll
    for (int g = 0; g < 4; ++g) acc[g][0] = acc[g][1] = 0.0;
    const uint32_t k0 = p.def_ptr[i] - K0, k1 = p.def_ptr[i + 1] - K0;
    for (uint32_t k = k0; k < k1; ++k) {
      const uint32_t mm = S.m[k];
      if (!(mm & 7u)) continue;
#pragma unroll
      for (uint32_t r = R_MEM; r <= R_SYNC; ++r) {
        if (!(mm & (1u << (r - 1)))) continue;
        const uint32_t g = r == R_MEM ? BG_MEM : r == R_SYNC ? BG_SYNC : ((mm & 8u) ? BG_WAR : BG_EXEC);
        const double2 v = S.prod[r - 1][k];
        acc[g][0] = __dadd_rn(acc[g][0], v.x);
        acc[g][1] = __dadd_rn(acc[g][1], v.y);
      }
    }
    store_B(p, i, acc);
  }
  __syncwarp();
}

// ---- pattern matching shared by the estimate and advice kernels (Table 2)
__device__ __forceinline__ uint32_t classify(uint32_t r, uint32_t cls, uint32_t kind) {
  if (r == R_MEM) return cls == OC_LOCAL ? COL_MEM_LOCAL : cls == OC_CONSTANT ? COL_MEM_CONSTANT : COL_MEM_GLOBAL;
  if (r == R_EXEC) return (kind & K_WAR) ? COL_EXEC_WAR : cls == OC_SHARED ? COL_EXEC_SHARED : COL_EXEC_ARITH;
  return COL_SYNC;
}

__device__ __forceinline__ bool passes(const gpa_pattern &q, uint32_t cls, uint32_t flags) {
  return ((q.class_mask >> cls) & 1u) && (!q.flag_filter || (flags & q.flag_filter));
}

// matched samples of edge e (def d -> use j) under pattern q: X = all / latency samples of j
struct EdgeInfo {
  uint32_t m, cls, flags, c_mem, c_exec;
  bool same;
  double sh0, sh1, sh2;
};
__device__ __forceinline__ EdgeInfo edge_info(const DevProgram &p, uint32_t e, int32_t loop_j) {
  EdgeInfo x{};
  x.m = p.cand[e];
  uint32_t kind = 0;
  if (x.m) {
    const uint32_t d = p.edge_def[e];
    const DefInfo di = p.dinfo[d];
    x.cls = di.cls_flags & 0xffu;
    x.flags = di.cls_flags >> 8;
    kind = p.edge_kind[e];
    x.same = di.loop >= 0 && di.loop == loop_j;
    const double *sh = p.share + 3 * (uint64_t)e;
    x.sh0 = sh[0]; x.sh1 = sh[1]; x.sh2 = sh[2];
  }
  x.c_mem = classify(R_MEM, x.cls, kind);
  x.c_exec = classify(R_EXEC, x.cls, kind);
  return x;
}
__device__ __forceinline__ double edge_match(const gpa_pattern &q, const EdgeInfo &x, const double *X) {
  double me = 0.0;
  if (x.m && passes(q, x.cls, x.flags) && (!q.same_loop || x.same)) {
    if ((x.m & 1u) && ((q.column_mask >> x.c_mem) & 1u)) me = __dadd_rn(me, __dmul_rn(X[1], x.sh0));
    if ((x.m & 2u) && ((q.column_mask >> x.c_exec) & 1u)) me = __dadd_rn(me, __dmul_rn(X[2], x.sh1));
    if ((x.m & 4u) && ((q.column_mask >> COL_SYNC) & 1u)) me = __dadd_rn(me, __dmul_rn(X[3], x.sh2));
  }
  return me;
}

// the use's own matched samples (self and pass-through columns) under pattern q (k_est_rows,
// k_hotspots): X = all / latency samples of the dependency reasons, row = C row of j
__device__ __forceinline__ double instr_match(const gpa_pattern &q, uint32_t R, const uint64_t *row, const double *X,
                                              uint32_t cls_j, uint32_t flags_j, uint32_t self_j, int32_t loop_j) {
  double mi = 0.0;
  const bool L = q.sample_class != 0;
  if (passes(q, cls_j, flags_j) && (!q.same_loop || loop_j >= 0)) {
    for (uint32_t r = R_MEM; r <= R_SYNC; ++r)
      if (((self_j >> (r - 1)) & 1u) && ((q.column_mask >> (COL_MEM_SELF + r - 1)) & 1u)) mi = __dadd_rn(mi, X[r]);
    for (uint32_t r = 4; r < R; ++r)
      if ((q.column_mask >> (COL_PASS0 + r - 4)) & 1u) mi = __dadd_rn(mi, (double)(row[R + r] + (L ? 0ull : row[r])));
  }
  return mi;
}

#endif

}  // namespace gpa

struct gpa_program {
  int device = 0;
  int n_sms = 148;
  size_t smem_optin = 0;
  uint8_t *ws = nullptr;
  size_t ws_bytes = 0;
  gpa::DevProgram d{};
  gpa::RollupPlan rp{};
  gpa::EstimatePlan ep{};
  gpa::AdvicePlan ap{};
  gpa::KernOcc *occ_dev = nullptr;
  std::vector<uint32_t> grid_host;   // kernel_grid_blocks (empty if not given)
  int state = 0;
  int variant = gpa::VAR_SMEM;
  bool part_ok = false;
  uint32_t seg_tab_bins = 0;        // shared-memory table of the segment ingest (bins)
  uint64_t launches = 0;
  uint64_t view_off[GPA_VIEW_COUNT_] = {};
  uint64_t view_bytes[GPA_VIEW_COUNT_] = {};
  gpa_pattern *pats_dev = nullptr;
  // host ingest staging ring
  void *staging = nullptr;
  size_t staging_bytes = 0;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr};
  // blame + aggregate + estimate captured once as a CUDA graph (gpa_analyze)
  cudaStream_t capture_stream = nullptr;
  cudaStream_t side_stream = nullptr;          // analyze graph: the estimate branch
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaGraphExec_t analyze_exec = nullptr;
  uint32_t analyze_npat = 0xffffffffu;
  uint64_t analyze_launches = 0;
  int analyze_mode = GPA_ANALYZE_AUTO;   // gpa_set_analyze_mode
};

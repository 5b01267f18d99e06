/*
 * gpa.h -- C ABI of the B200-native GPA hot path.
 *
 * GPA (Zhou, Meng, Sai, Mellor-Crummey, "GPA: A GPU Performance Advisor Based on Instruction
 * Sampling", arXiv 2009.04061).  Citations "P:n" are lines of the paper's text;
 * readings of silent or ambiguous passages are the Q-numbers of DESIGN.md §3.2.
 *
 * The problem statement: static program structure (instruction table, def-use
 * graph with path lengths, line/loop/function maps) + a stream of PC samples  ->  stalls
 * attributed to the instructions that cause them, rolled up to program structure, and the
 * estimated speedup of each optimizer.  Calls, in order:
 *
 *   gpa_workspace_size / gpa_program_create   static structure -> device workspace
 *   gpa_reset_counts                          zero the sample histogram
 *   gpa_ingest_samples (repeatable)           records -> C[pc][class][reason]
 *   [multi-GPU: all-reduce the counts view]
 *   gpa_blame                                 rules 1-3, Eq. 1, Fig. 6
 *   gpa_aggregate                             line / loop / function / kernel
 *   gpa_set_patterns + gpa_estimate           Table 2 + Eqs. 2-10
 *
 * Conventions:
 *   stall reason r : 0 NONE, 1 MEM, 2 EXEC, 3 SYNC (dependency reasons), r >= 4 are
 *                    pass-through reasons; R = n_reasons in [4, 16].
 *   sample class c : 0 ACT (scheduler issuing), 1 LAT (not issuing).
 *   opcode class   : 0 GLOBAL 1 LOCAL 2 SHARED 3 CONSTANT 4 TEXTURE 5 ARITH_FIXED 6 ARITH_LONG
 *                    7 CONVERT 8 CONTROL 9 SYNC 10 MISC.
 *   edge kind bits : 1 REG, 2 PRED, 4 BAR (virtual barrier register), 8 WAR.
 *   instr flags    : 1 IN_MATH, 2 IN_DEVICE_FN, 4 CALLSITE.
 *   blame columns  : 0 MEM_GLOBAL 1 MEM_LOCAL 2 MEM_CONSTANT 3 EXEC_SHARED 4 EXEC_ARITH
 *                    5 EXEC_WAR 6 SYNC 7 MEM_SELF 8 EXEC_SELF 9 SYNC_SELF 10+(r-4) reason r;
 *                    NCOL = R + 6; every column holds {all samples, latency samples}.
 *
 * Memory and ownership: every pointer in gpa_program_desc is a HOST pointer, read only during
 * gpa_program_create and copied into the caller-owned DEVICE workspace.  The library never
 * allocates device memory except the staging ring of gpa_ingest_samples_host.  Views
 * (gpa_view) are byte ranges of that workspace, valid until gpa_program_destroy.
 *
 * Asynchrony: reset / ingest / blame / aggregate / estimate only enqueue work on `stream`
 * (a cudaStream_t passed as void*; NULL = legacy default stream).  gpa_program_create,
 * gpa_set_patterns, gpa_read_estimates, gpa_get_stats and gpa_ingest_samples_host synchronize.
 *
 * Errors: every call returns gpa_status; negative = error, with a message in gpa_last_error()
 * (thread-local).  Malformed sample RECORDS are data, not errors: they are excluded and counted
 * (gpa_get_stats).  A CUDA launch failure returns GPA_ERR_CUDA and leaves the program unusable.
 */
#ifndef GPA_H
#define GPA_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GPA_OK = 0,
  GPA_ERR_INVALID_ARGUMENT = -1, /* NULL pointer, size mismatch, misaligned buffer */
  GPA_ERR_INVALID_PROGRAM = -2,  /* desc violates a structural rule (see gpa_validate_program) */
  GPA_ERR_BAD_STATE = -3,        /* call order violated (e.g. aggregate before blame) */
  GPA_ERR_CUDA = -4,             /* CUDA runtime / launch error */
  GPA_ERR_WORKSPACE = -5,        /* workspace too small or not 256-byte aligned */
  GPA_ERR_DOMAIN = -6,           /* estimator input outside its domain (W <= 0, R_I not in [0,1]) */
  GPA_ERR_OVERFLOW = -7          /* an output capacity or search budget was exceeded (gpa_slice) */
} gpa_status;

/* One PC-sampling record: `count` identical samples of instruction `pc`
 * (global instruction index), stall `reason`, flags bit0 = latency sample.  8 bytes, little
 * endian.  Valid iff pc < n_instr, reason < R, flags <= 1 and not (LAT and reason == NONE). */
typedef struct {
  uint32_t pc;
  uint16_t count;
  uint8_t reason;
  uint8_t flags;
} gpa_sample;

/* Static program structure (the outputs of GPA's static analyzer). */
typedef struct {
  uint32_t n_instr;             /* instructions, >= 1 */
  uint32_t n_reasons;           /* R in [4, 16] */
  uint32_t n_lines, n_loops, n_funcs, n_kernels;
  const uint8_t *opclass;       /* [n_instr] opcode class, < 11 */
  const uint8_t *iflags;        /* [n_instr] IN_MATH | IN_DEVICE_FN | CALLSITE */
  const uint32_t *latency;      /* [n_instr] cycles; upper bound for variable latency */
  const uint32_t *line_id;      /* [n_instr] < n_lines */
  const int32_t *loop_id;       /* [n_instr] innermost loop or -1 */
  const int32_t *loop_parent;   /* [n_loops] parent loop or -1; the loop forest must be acyclic */
  const uint32_t *func_begin;   /* [n_funcs+1] contiguous instruction ranges, [0] = 0, [n_funcs] = n_instr */
  const uint32_t *kernel_func_begin; /* [n_kernels+1] contiguous function ranges */
  const uint32_t *kernel_grid_blocks; /* [n_kernels] launch blocks, or NULL (Block Increase) */
  /* def-use graph, CSR keyed by the USE instruction j; one edge per (def, use) (Q10) */
  const uint32_t *row_ptr;      /* [n_instr+1] */
  const uint32_t *edge_def;     /* [E] def instruction i, same function as j */
  const uint8_t *edge_kind;     /* [E] REG | PRED | BAR | WAR, nonzero */
  const uint32_t *edge_min_len; /* [E] fewest instructions on an i->j CFG path, >= 1 (rule 3) */
  const uint32_t *edge_max_len; /* [E] most instructions on an i->j path, >= min_len (Eq. 1) */
  const int32_t *edge_dom_k;    /* [E] rule-2 interposer instruction or -1 (Q7) */
} gpa_program_desc;

/* Optimizer pattern (one Table 2 row), see DESIGN.md §3.4. */
typedef struct {
  uint32_t column_mask;  /* blame columns matched */
  uint16_t class_mask;   /* opcode classes of the blamed instruction matched (bit per class) */
  uint8_t sample_class;  /* 0: all samples (M), 1: latency samples (M^L) */
  uint8_t model;         /* 0 Eq.2, 1 Eq.4, 2 Eq.5 over loops, 3 Eq.5 over functions,
                            4 Eq.5 over loops and functions, 5 Eq.10 (parallel) */
  uint8_t flag_filter;   /* nonzero: blamed instruction must have (iflags & flag_filter) */
  uint8_t same_loop;     /* def and use in the same innermost loop (Q15) */
  uint8_t parallel_rule; /* model 5 match: 0 never, 1 always, 2 grid_blocks < sm_count (W, W_new
                            below); 3 Block Increase, 4 Thread Increase with W,
                            W_new from the occupancy model (gpa_set_launches) */
  uint8_t pad;
  uint32_t sm_count;
  double ratio;          /* Eq. 2 uses ratio * M (Q17); 1 = the paper's Eq. 2 */
  double W, W_new, f;    /* Eqs. 6-10 inputs (Q18) */
} gpa_pattern;

typedef struct {
  double speedup;        /* the pattern's model; +inf when unbounded */
  double M;              /* matched samples at kernel level (pattern's sample class) */
  double eq3, eq4;       /* T/(T-M) and T/(T-min(A,M)) for reference */
  uint64_t T, A;         /* kernel samples and active samples */
  int32_t best_scope;    /* Eq. 5: loop id, or n_loops + function id; -1 otherwise */
  uint8_t unbounded, matched, model, pad;
} gpa_estimate_out;

/* SASS fields for backward slicing (Table 1) and the
 * control flow graph.  Host pointers, read during gpa_slice only. */
typedef struct {
  uint32_t n_instr, n_funcs, n_blocks;
  const uint32_t *func_begin;   /* [n_funcs+1] contiguous instruction ranges (block boundaries) */
  const uint32_t *block_begin;  /* [n_blocks+1] contiguous basic blocks, [0] = 0, [n_blocks] = n_instr */
  const uint32_t *succ_ptr;     /* [n_blocks+1] CSR of successor blocks */
  const uint32_t *succ;         /* successor block ids, in the same function */
  const uint8_t *guard;         /* [n_instr] bits 0-2 predicate P0..P6 (7 = none, '_'), bit 3 = negated (!P) */
  const uint16_t *dst, *src;    /* [n_instr][4] operands: 0..254 R0..R254, 255 RZ (ignored),
                                   256..262 P0..P6, 0xFFFF = none */
  const uint8_t *wbar, *rbar;   /* [n_instr] write / read barrier masks over B0..B5 */
  const uint8_t *wait;          /* [n_instr] wait mask over B0..B5 */
} gpa_sass_desc;

/* PC-sampling simulator (DESIGN.md §3.2 Q40-Q44). */
typedef struct {
  uint32_t schedulers, warps_per_scheduler;  /* warps of one simulated SM */
  uint32_t period;                           /* a sample every `period` cycles, schedulers in turn */
  uint32_t trip_count;                       /* iterations of every self-loop block */
  uint32_t rbar_latency;                     /* cycles until a read barrier clears */
  uint32_t max_cycles;                       /* per SM; exceeding it is an error */
  uint64_t seed;                             /* predicate values per warp */
} gpa_simcfg;

/* Occupancy model (DESIGN.md §3.2 Q34): the GPU the profile came from and
 * each kernel's launch, for parallel_rule 3 / 4 of the parallel estimator (Eqs. 6-10). */
typedef struct {
  uint32_t sm_count, max_warps_per_sm, max_blocks_per_sm, regs_per_sm, smem_per_sm,
           schedulers_per_sm, warp_size, reg_alloc_unit;
} gpa_arch;
typedef struct {
  uint32_t threads_per_block, regs_per_thread, smem_per_block, pad;   /* 0 = unknown / none */
} gpa_launch;

/* Advice report data (after the path; DESIGN.md §3.2 Q30-Q32). */
#define GPA_TOP_K_MAX 8
typedef struct {
  uint32_t def_pc;       /* blamed instruction: def of an edge, or the use for its own samples */
  uint32_t use_pc;       /* instruction where the samples were observed */
  uint32_t distance;     /* the edge's max_len ("their distance"); 0 for own samples */
  uint32_t item;         /* edge index e, or E + instruction */
  double samples;        /* matched samples of the pattern (its sample class) on this item */
} gpa_hotspot;           /* 24 bytes */

typedef struct {
  uint64_t nodes;          /* instructions with dependency-stall samples */
  uint64_t single_before;  /* single-dependency nodes before pruning */
  uint64_t single_after;   /* after rules 1-3 */
} gpa_coverage;

typedef struct gpa_program gpa_program;

/* Views of device results (byte ranges of the workspace), for gpa_view(): */
typedef enum {
  GPA_VIEW_COUNTS = 0,     /* u64 [n_instr][2][R]: C[pc][class][reason]; all-reduce this (SUM) */
  GPA_VIEW_STATS = 1,      /* u64 [4]: valid samples, invalid records, invalid samples, reserved;
                              starts right after GPA_VIEW_COUNTS' last byte, so one SUM
                              all-reduce of [counts | stats] combines ranks */
  GPA_VIEW_INSTR_AL = 2,   /* u64 [n_instr][2]: A_i, L_i (after gpa_aggregate / gpa_analyze) */
  GPA_VIEW_CAND = 3,       /* u8 [E]: candidate mask bit r-1, r in {MEM,EXEC,SYNC} */
  GPA_VIEW_SELF = 4,       /* u8 [n_instr]: self-attribution flags bit r-1 (Q5) */
  GPA_VIEW_SHARE = 5,      /* f64 [E][3]: Eq. 1 share per dependency reason, 0 if not candidate */
  GPA_VIEW_INSTR_BLAME = 6,/* f64 [n_instr][4][2]: edge blame at the def by {MEM, EXEC, EXEC_WAR,
                              SYNC} x {all, latency}; MEM/EXEC sub-category = def class (Fig. 6) */
  GPA_VIEW_LINE = 7,       /* f64 [n_lines][NCOL][2] */
  GPA_VIEW_LINE_AL = 8,    /* u64 [n_lines][2] */
  GPA_VIEW_LOOP_EXCL = 9,  /* f64 [n_loops][NCOL][2]: instructions whose innermost loop is l */
  GPA_VIEW_LOOP_EXCL_AL = 10,
  GPA_VIEW_LOOP_INCL = 11, /* f64 [n_loops][NCOL][2]: l and all loops nested in it (Eq. 5) */
  GPA_VIEW_LOOP_INCL_AL = 12,
  GPA_VIEW_FUNC = 13,      /* f64 [n_funcs][NCOL][2] */
  GPA_VIEW_FUNC_AL = 14,
  GPA_VIEW_KERNEL = 15,    /* f64 [n_kernels][NCOL][2] */
  GPA_VIEW_KERNEL_AL = 16, /* u64 [n_kernels][2]: A, L; T = A + L */
  GPA_VIEW_ESTIMATES = 17, /* gpa_estimate_out [n_kernels][n_patterns] */
  GPA_VIEW_COUNT_ = 18
} gpa_view_id;

/* Host-only structural validation: row_ptr monotone, def < n_instr, def and use in the same
 * function, no duplicate (def, use) in a row, 1 <= min_len <= max_len, kinds nonzero, classes
 * < 11, line_id < n_lines, loops acyclic with every loop inside one function, function and
 * kernel ranges contiguous and covering.  GPA_ERR_INVALID_PROGRAM with a message otherwise. */
gpa_status gpa_validate_program(const gpa_program_desc *desc);

/* Device workspace bytes for `desc` (validates it).  The workspace must be 256-byte aligned. */
gpa_status gpa_workspace_size(const gpa_program_desc *desc, size_t *bytes);

/* Validates, builds the create-time transposes/permutations on the host, copies everything
 * into `d_workspace` on `stream` and synchronizes.  The device is the current CUDA device. */
gpa_status gpa_program_create(const gpa_program_desc *desc, void *d_workspace, size_t bytes,
                              void *stream, gpa_program **out);
gpa_status gpa_program_destroy(gpa_program *prog);

/* Advice (enqueue; needs estimates of the current counts: gpa_estimate or gpa_analyze with
 * patterns set): per (kernel, pattern) the top_k hotspots (1 <= top_k <= GPA_TOP_K_MAX; items
 * with matched samples > 0 by samples descending, ties by item), the patterns of every kernel
 * ranked by estimated speedup (+inf first, ties by pattern index) and the single
 * dependency coverage before / after pruning per kernel. */
gpa_status gpa_advise(gpa_program *prog, uint32_t top_k, void *stream);

/* Copy the advice to HOST buffers (synchronizes); any pointer may be NULL to skip it:
 *   h_hotspots [n_kernels][n_patterns][top_k], h_n_hotspots u32 [n_kernels][n_patterns],
 *   h_rank u32 [n_kernels][n_patterns] (pattern index at each rank), h_coverage [n_kernels].
 * GPA_ERR_BAD_STATE before gpa_advise. */
gpa_status gpa_read_advice(gpa_program *prog, gpa_hotspot *h_hotspots, uint32_t *h_n_hotspots, uint32_t *h_rank,
                           gpa_coverage *h_coverage, void *stream);

/* Backward slicing (DESIGN.md §3.2 Q35-Q39): the def-use CSR keyed by the use -- what
 * gpa_program_desc's row_ptr / edge_* fields take -- from SASS fields and the CFG, computed on
 * the device (one thread per use).  Host output arrays: h_row_ptr [n_instr+1] and cap_edges
 * entries of each edge array; *n_edges receives the edge count.  GPA_ERR_OVERFLOW if cap_edges
 * is too small (nothing but *n_edges and h_row_ptr written) or a search exceeds its state budget
 * (4 x the longest function + 256 states).  Synchronizes. */
gpa_status gpa_slice(const gpa_sass_desc *h_sass, uint64_t cap_edges, uint32_t *h_row_ptr, uint32_t *h_edge_def,
                     uint8_t *h_edge_kind, uint32_t *h_edge_min_len, uint32_t *h_edge_max_len,
                     int32_t *h_edge_dom_k, uint64_t *n_edges, void *stream);

/* Simulate n_sm SMs (one GPU thread each) running function `func` of a SASS program and write each
 * SM's PC samples to DEVICE d_records + sm * cap_per_sm (gpa_sample: pc within the program, count
 * 1, reason, class) and, if d_truth is not NULL, the ground truth (the instruction whose result a
 * dependency-stalled sample waits for, else -1) at the same positions.  h_counts[sm] receives the
 * SM's record count.  h_opclass / h_latency: HOST [n_instr].  GPA_ERR_OVERFLOW if an SM exceeds
 * cap_per_sm records or cfg.max_cycles.  Synchronizes. */
gpa_status gpa_simulate(const gpa_sass_desc *h_sass, const uint8_t *h_opclass, const uint32_t *h_latency,
                        uint32_t func, const gpa_simcfg *cfg, uint32_t n_sm, uint64_t cap_per_sm,
                        gpa_sample *d_records, int32_t *d_truth, uint64_t *h_counts, void *stream);

/* Set the kernels' launch statistics (HOST array [n_kernels]; with the program's
 * kernel_grid_blocks) and the GPU's limits; computes, per kernel, the resident warps per
 * scheduler W and the W_new of Block Increase (same warps over all SMs when grid < #SM) and
 * Thread Increase (block slots bind; larger blocks up to the warp / register limit).  Used by
 * patterns with parallel_rule 3 / 4; without this call those never match.  Synchronizes. */
gpa_status gpa_set_launches(gpa_program *prog, const gpa_launch *h_launches, const gpa_arch *arch, void *stream);

/* Zero the count table and stats (enqueue). */
gpa_status gpa_reset_counts(gpa_program *prog, void *stream);

/* Histogram n records at DEVICE pointer d_samples (8-byte aligned) into the count table
 * (enqueue; accumulates across calls).  n = 0 is a no-op. */
gpa_status gpa_ingest_samples(gpa_program *prog, const gpa_sample *d_samples, uint64_t n,
                              void *stream);

/* Same from HOST memory: copies through a double-buffered device staging ring in chunks and
 * ingests each chunk; pinned memory overlaps copy and histogram.  Synchronizes. */
gpa_status gpa_ingest_samples_host(gpa_program *prog, const gpa_sample *h_samples, uint64_t n,
                                   void *stream);

/* Histogram a stream grouped by kernel launch (enqueue; accumulates).  GPA's profiler collects
 * the PC samples of each kernel launch and the blamer analyses each invocation,
 * so a whole-application batch (BASELINE config 4) arrives as per-launch segments:
 *   segment s = records [d_seg_begin[s], d_seg_begin[s+1]) of d_samples, drawn from kernel
 *   d_seg_kernel[s] of this program (any value >= n_kernels: unknown kernel).
 * d_seg_begin: DEVICE u64 [n_segments + 1], non-decreasing (offsets past n_samples are clipped;
 * records outside [d_seg_begin[0], d_seg_begin[n_segments]) are not ingested).
 * d_seg_kernel: DEVICE u32 [n_segments].  pc_base is subtracted from every record's pc before
 * decoding (a program holding a slice of an application's kernels).
 * Counts and stats are identical to gpa_ingest_samples over the same records (with pc - pc_base):
 * records outside their segment's kernel are still counted, only more slowly.  Non-monotone
 * offsets are memory-safe but give unspecified counts.  n_segments = 0 is a no-op. */
gpa_status gpa_ingest_segments(gpa_program *prog, const gpa_sample *d_samples, uint64_t n_samples,
                               const uint64_t *d_seg_begin, const uint32_t *d_seg_kernel,
                               uint32_t n_segments, uint32_t pc_base, void *stream);

/* Rules 1-3, Eq. 1 (all and latency samples), self flags, Fig. 6 classes, def-side
 * reduction (enqueue).  GPA_ERR_BAD_STATE before any reset/ingest. */
gpa_status gpa_blame(gpa_program *prog, void *stream);

/* Rollups to line, loop (exclusive, inclusive), function, kernel (enqueue); needs gpa_blame. */
gpa_status gpa_aggregate(gpa_program *prog, void *stream);

/* Copy n_patterns (<= 32) patterns into the workspace (synchronizes). */
gpa_status gpa_set_patterns(gpa_program *prog, const gpa_pattern *patterns, uint32_t n_patterns,
                            void *stream);

/* Matching + Eqs. 2-10 per (kernel, pattern) into GPA_VIEW_ESTIMATES (enqueue); needs
 * gpa_aggregate and gpa_set_patterns. */
gpa_status gpa_estimate(gpa_program *prog, void *stream);

/* gpa_blame + gpa_aggregate + (gpa_estimate when patterns are set) as one CUDA graph, captured
 * on first use (and again after gpa_set_patterns changes the pattern count), replayed on `stream`
 * (enqueue).  Same results as the three calls; fewer launch gaps. */
gpa_status gpa_analyze(gpa_program *prog, void *stream);

/* How gpa_analyze runs the analysis.  GPA_ANALYZE_GRAPH: the CUDA graph of per-step kernels
 * above.  GPA_ANALYZE_FUSED: one cooperative kernel running the same device code phase by phase
 * with grid-wide barriers between dependent phases (no launch gaps; both give bit-identical
 * results).  GPA_ANALYZE_AUTO (default) is the graph: on B200 the fused kernel measured slower at
 * every program size tried (config 2: 40 vs 53-90 us), because the graph runs the
 * independent branches (def reduction | estimate sums) side by side while every CTA of the fused
 * kernel runs them one after the other.  Errors: GPA_ERR_INVALID_ARGUMENT for an unknown mode. */
#define GPA_ANALYZE_AUTO 0
#define GPA_ANALYZE_GRAPH 1
#define GPA_ANALYZE_FUSED 2
gpa_status gpa_set_analyze_mode(gpa_program *prog, int mode);

/* Copy the estimates to host memory h_out[n_kernels * n_patterns] (synchronizes). */
gpa_status gpa_read_estimates(gpa_program *prog, gpa_estimate_out *h_out, void *stream);

/* Copy the 4 stats words to host (synchronizes). */
gpa_status gpa_get_stats(gpa_program *prog, uint64_t out[4], void *stream);

/* Byte offset (from the workspace base) and size of a device result. */
gpa_status gpa_view(gpa_program *prog, int view, uint64_t *offset, uint64_t *bytes);

/* Expand the per-instruction blame vector V[n_instr][NCOL][2] (f64) into the caller's
 * DEVICE buffer d_out (enqueue; needs gpa_blame).  Instruction-level rollup level. */
gpa_status gpa_instr_vector(gpa_program *prog, double *d_out, void *stream);

/* Program shape queries. */
gpa_status gpa_program_info(gpa_program *prog, uint64_t info[8]); /* n_instr, E, R, NCOL, n_lines,
                                                                      n_loops, n_funcs, n_kernels */
/* Which ingest kernel the program uses: 0 smem-private table, 1 partitioned smem, 2 L2 atomics. */
gpa_status gpa_ingest_variant(gpa_program *prog, int *variant);
gpa_status gpa_set_ingest_variant(gpa_program *prog, int variant);

/* Number of kernel launches the last blame+aggregate+estimate enqueued (self-reported). */
gpa_status gpa_launch_count(gpa_program *prog, uint64_t *launches);

const char *gpa_last_error(void);
const char *gpa_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GPA_H */

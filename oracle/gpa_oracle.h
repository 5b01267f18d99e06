/*
 * gpa_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU statement of what GPA's instruction blamer,
 * rollup and estimators compute (arXiv 2009.04061, "GPA: A GPU Performance Advisor
 * Based on Instruction Sampling").  Citations "P:n" are lines of PAPER.md; the
 * adopted readings of silent/ambiguous passages are the Q-numbers of DESIGN.md §3.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library.  It shares no code, header, table or constant with the
 * CUDA path under paper_2009_04061_b200/ and never calls it.
 *
 * Conventions fixed here (own copy; the product header states them independently):
 *   stall reasons  r: 0 NONE, 1 MEM (memory dependency), 2 EXEC (execution dependency),
 *                     3 SYNC (synchronization), >=4 pass-through reasons (throttle,
 *                     fetch, pipe, not-selected, misc ...), R <= 16 reasons in total.
 *   sample class   c: 0 ACT (active: scheduler issuing), 1 LAT (latency) -- P:137.
 *   opcode class     : 0 GLOBAL 1 LOCAL 2 SHARED 3 CONSTANT 4 TEXTURE 5 ARITH_FIXED
 *                      6 ARITH_LONG 7 CONVERT 8 CONTROL 9 SYNC 10 MISC.
 *   record (8 bytes, little endian): u32 pc | u16 count | u8 reason | u8 flags(bit0=LAT).
 *   blame columns    : 0 MEM_GLOBAL 1 MEM_LOCAL 2 MEM_CONSTANT 3 EXEC_SHARED 4 EXEC_ARITH
 *                      5 EXEC_WAR 6 SYNC 7 MEM_SELF 8 EXEC_SELF 9 SYNC_SELF,
 *                      10+(r-4) pass-through reason r  (NCOL = 10 + R - 4).
 *   per column two values: [0] = all samples (ACT+LAT), [1] = latency samples only.
 *
 * "parity pinned" / "parity unpinned" status of every function: DESIGN.md §3.3.
 */
#ifndef GPA_ORACLE_H
#define GPA_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint32_t n_instr, n_reasons, n_lines, n_loops, n_funcs, n_kernels;
  const uint8_t  *opclass;        /* [n_instr] */
  const uint8_t  *iflags;         /* [n_instr] bit0 IN_MATH, bit1 IN_DEVICE_FN, bit2 CALLSITE */
  const uint32_t *latency;        /* [n_instr] cycles; upper bound if variable */
  const uint32_t *line_id;        /* [n_instr] */
  const int32_t  *loop_id;        /* [n_instr] innermost loop or -1 */
  const int32_t  *loop_parent;    /* [n_loops] -1 = outermost */
  const uint32_t *func_begin;     /* [n_funcs+1] contiguous instruction ranges */
  const uint32_t *kernel_func_begin; /* [n_kernels+1] contiguous function ranges */
  const uint32_t *kernel_grid_blocks; /* [n_kernels] or NULL */
  const uint32_t *row_ptr;        /* [n_instr+1] def-use CSR keyed by the use */
  const uint32_t *edge_def;       /* [E] */
  const uint8_t  *edge_kind;      /* [E] bit0 REG bit1 PRED bit2 BAR bit3 WAR */
  const uint32_t *edge_min_len;   /* [E] fewest instructions on any def->use path */
  const uint32_t *edge_max_len;   /* [E] most instructions on any def->use path */
  const int32_t  *edge_dom_k;     /* [E] rule-2 interposer instruction or -1 */
} or_program;

typedef struct {
  uint32_t column_mask;   /* bit per blame column */
  uint16_t class_mask;    /* bit per opcode class of the blamed instruction */
  uint8_t  sample_class;  /* 0 all samples, 1 latency samples */
  uint8_t  model;         /* 0 Eq.2, 1 Eq.4, 2 Eq.5 loops, 3 Eq.5 functions, 4 Eq.5 loops+functions, 5 Eq.10 */
  uint8_t  flag_filter;   /* nonzero: blamed instruction must have (iflags & flag_filter) != 0 */
  uint8_t  same_loop;     /* def and use in the same innermost loop */
  uint8_t  parallel_rule; /* Eq.10 match: 0 never, 1 always, 2 grid_blocks < sm_count with
                            the caller's W / W_new; 3 Block Increase, 4 Thread Increase from the
                            occupancy model (or_occupancy) */
  uint8_t  pad;
  uint32_t sm_count;
  double ratio, W, W_new, f;
} or_pattern;

typedef struct {
  double speedup, M, eq3, eq4;
  uint64_t T, A;
  int32_t best_scope;      /* loop id, n_loops + function id, or -1 */
  uint8_t unbounded, matched, model, pad;
} or_estimate;

/* Step 1: per-record validity + C[pc][c][r] += count.  stats[0] valid samples,
   stats[1] invalid records, stats[2] invalid samples.  records: n*8 raw bytes. */
int or_histogram(const or_program *p, const uint8_t *records, uint64_t n,
                 uint64_t *C /* n_instr*2*R, accumulated into */, uint64_t stats[3]);

/* Steps 2-6: live rows, candidates (rules 1-3), Eq.1 shares, self flags, and the
   per-instruction blame vector V[n_instr][NCOL][2]. */
int or_blame(const or_program *p, const uint64_t *C,
             uint8_t *cand /* [E] bit r-1 for r in {MEM,EXEC,SYNC} */,
             uint8_t *self_flags /* [n_instr] bit r-1 */,
             double *share /* [E][3] */, double *V /* [n_instr][NCOL][2] */);

/* Step 7: rollups of V and of (A,L) counts.
   Any output pointer may be NULL.  *_v are [seg][NCOL][2], *_al are [seg][2]. */
int or_rollup(const or_program *p, const uint64_t *C, const double *V,
              double *line_v, uint64_t *line_al,
              double *loop_excl_v, uint64_t *loop_excl_al,
              double *loop_incl_v, uint64_t *loop_incl_al,
              double *func_v, uint64_t *func_al,
              double *kern_v, uint64_t *kern_al);

/* Step 8: optimizer matching and Eqs. 2-10.  out[k*n_pat + q]. */
int or_estimate_all(const or_program *p, const uint64_t *C, const uint8_t *cand,
                    const uint8_t *self_flags, const double *share,
                    const or_pattern *pats, uint32_t n_pat, or_estimate *out);

/* ---- backward slicing: the def-use CSR from SASS fields
 * (Table 1: wait mask, write / read barrier, predicate, destination and source
 * operands) and the CFG; DESIGN.md §3.2 Q35-Q39 state the readings. */
typedef struct {
  uint32_t n_instr, n_funcs, n_blocks;
  const uint32_t *func_begin;   /* [n_funcs+1] */
  const uint32_t *block_begin;  /* [n_blocks+1] contiguous instruction ranges inside functions */
  const uint32_t *succ_ptr;     /* [n_blocks+1] */
  const uint32_t *succ;         /* successor blocks, same function */
  const uint8_t  *guard;        /* [n_instr] bits 0-2 predicate register P0..P6, 7 = none ('_'); bit 3 = negated */
  const uint16_t *dst, *src;    /* [n_instr][4]: 0..254 R0..R254, 255 RZ (ignored), 256..262 P0..P6, 0xFFFF none */
  const uint8_t  *wbar, *rbar, *wait;   /* [n_instr] barrier masks over B0..B5 */
} or_sass;

/* Def-use CSR keyed by the use (one edge per (def, use), defs ascending), as gpa_program_desc
 * takes it: kind bits REG 1, PRED 2, BAR 4, WAR 8; min_len / max_len; dom_k (rule 2) or -1.
 * cap = capacity of the edge arrays; returns the edge count, or -1 if cap is too small. */
int64_t or_slice(const or_sass *s, uint64_t cap, uint32_t *row_ptr, uint32_t *edge_def, uint8_t *edge_kind,
                 uint32_t *edge_min, uint32_t *edge_max, int32_t *edge_dom);

/* ---- sampling simulator (P:119-142 PC sampling model, DESIGN.md §3.2
 * Q40-Q44): one SM running warps of one SASS function with an in-order scoreboard, loose
 * round-robin warp schedulers, and a sample every `period` cycles from the schedulers in turn. */
typedef struct {
  uint32_t schedulers, warps_per_scheduler, period, trip_count, rbar_latency, max_cycles;
  uint64_t seed;          /* predicate values: P_k of warp w = bit 0 of mix(seed, w, k) */
} or_simcfg;

/* Simulate SM `sm` (its warps are sm*W .. sm*W+W-1 globally) running function `func`; writes up to
 * cap records (8 bytes: pc | count 1 | reason | class) and truth[] (the instruction that produced
 * the value a dependency-stalled sample waits for, else -1).  Returns the record count, -1 if cap is
 * too small, -2 on a scheduling deadlock or max_cycles. */
int64_t or_simulate(const or_sass *s, const uint8_t *opclass, const uint32_t *latency, uint32_t func,
                    const or_simcfg *cfg, uint32_t sm, uint64_t cap, uint64_t *records, int32_t *truth);

/* ---- occupancy model feeding W, W_new of the parallel estimator
 * for Block Increase and Thread Increase; DESIGN.md §3.2 Q34. */
typedef struct {
  uint32_t sm_count, max_warps_per_sm, max_blocks_per_sm, regs_per_sm, smem_per_sm,
           schedulers_per_sm, warp_size, reg_alloc_unit;
} or_arch;
typedef struct { uint32_t threads_per_block, regs_per_thread, smem_per_block, pad; } or_launch;
typedef struct {
  double W;              /* active warps per scheduler */
  double W_new_block;    /* Block Increase: the same warps spread over all SMs */
  double W_new_thread;   /* Thread Increase: larger blocks up to the warp / register limit */
  uint32_t blocks_per_sm, limiter;   /* limiter 0 warps, 1 block slots, 2 registers, 3 shared memory */
  uint32_t match_block, match_thread;
} or_occ;
int or_occupancy(const or_arch *arch, const or_launch *launch, const uint32_t *grid_blocks,
                 uint32_t n_kernels, or_occ *out);

/* same, with the occupancy model per kernel for parallel_rule 3 / 4 (occ may be NULL) */
int or_estimate_all_occ(const or_program *p, const uint64_t *C, const uint8_t *cand,
                        const uint8_t *self_flags, const double *share,
                        const or_pattern *pats, uint32_t n_pat, const or_occ *occ, or_estimate *out);

/* ---- after the path: the advice report's data (P:261, P:658-661,
 * P:684-686).  DESIGN.md §3.2 Q30-Q33 state the readings. */
typedef struct {
  uint32_t def_pc;    /* blamed instruction (def of an edge; the use itself for self/pass-through) */
  uint32_t use_pc;    /* instruction where the samples were observed */
  uint32_t distance;  /* max_len of the edge (instructions on the longest path), 0 for own samples */
  uint32_t item;      /* edge index e, or E + instruction for the use's own samples */
  double samples;     /* matched samples of the pattern carried by this item */
} or_hotspot;

/* Per (kernel k, pattern q): the top_k items with matched samples > 0, by samples descending,
 * ties by item ascending.  out[(k*n_pat + q)*top_k + t], n_out[k*n_pat + q] = count. */
int or_hotspots(const or_program *p, const uint64_t *C, const uint8_t *cand,
                const uint8_t *self_flags, const double *share, const or_pattern *pats,
                uint32_t n_pat, uint32_t top_k, or_hotspot *out, uint32_t *n_out);

/* Optimizers of each kernel ranked by estimated speedup: order[k*n_pat + t] =
 * pattern at rank t; +inf first, ties by pattern index. */
int or_rank(const or_estimate *est, uint32_t n_kernels, uint32_t n_pat, uint32_t *order);

/* Single dependency coverage per kernel, before and after pruning:
 * out[3k] = nodes, out[3k+1] = single-dependency nodes before, out[3k+2] = after. */
int or_coverage(const or_program *p, const uint64_t *C, const uint8_t *cand, uint64_t *out);

/* Closed forms, exposed for the equation pins. */
double or_eq2(double T, double M);
double or_eq4(double T, double A, double ML);
double or_eq5(double T, double A_nested, double ML_scope);
double or_eq10(double W, double W_new, double R_I, double f);

uint32_t or_ncol(uint32_t n_reasons);

#ifdef __cplusplus
}
#endif
#endif

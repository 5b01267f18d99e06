/*
 * gpa_oracle.c -- TEST INFRASTRUCTURE ONLY (see gpa_oracle.h).
 *
 * Plain single-threaded C99, fp64, u64 counts, sums in the order the definitions are
 * written (CSR order, instruction order).  No blocking, no fusion, no reordering.
 * Each function cites the PAPER.md passage it follows ("P:n") and the DESIGN.md
 * reading ("Q#") where the paper is silent.  Build: gcc -O2 -shared -fPIC.
 */
#include "gpa_oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { R_NONE = 0, R_MEM = 1, R_EXEC = 2, R_SYNC = 3 };
enum { C_GLOBAL = 0, C_LOCAL = 1, C_SHARED = 2, C_CONSTANT = 3, C_TEXTURE = 4,
       C_ARITH_FIXED = 5, C_ARITH_LONG = 6, C_CONVERT = 7, C_CONTROL = 8, C_SYNC = 9, C_MISC = 10 };
enum { K_REG = 1, K_PRED = 2, K_BAR = 4, K_WAR = 8 };
enum { COL_MEM_GLOBAL = 0, COL_MEM_LOCAL = 1, COL_MEM_CONSTANT = 2, COL_EXEC_SHARED = 3,
       COL_EXEC_ARITH = 4, COL_EXEC_WAR = 5, COL_SYNC = 6, COL_MEM_SELF = 7, COL_EXEC_SELF = 8,
       COL_SYNC_SELF = 9, COL_PASS0 = 10 };

uint32_t or_ncol(uint32_t R) { return 10u + (R - 4u); }

static uint64_t cnt(const or_program *p, const uint64_t *C, uint32_t i, int c, uint32_t r) {
  return C[((uint64_t)i * 2u + (uint64_t)c) * p->n_reasons + r];
}

/* ---------------------------------------------------------------- step 1: histogram
 * every sample is an active sample (scheduler issuing) or a latency sample,
 * with a stall reason "if any".  A record is a pre-aggregated run of `count` identical
 * samples.  Q12: a latency sample without a stall reason is malformed and excluded;
 * records with pc >= n_instr, reason >= R or unknown flag bits are excluded too and
 * counted in the stats. */
int or_histogram(const or_program *p, const uint8_t *rec, uint64_t n, uint64_t *C,
                 uint64_t stats[3]) {
  uint64_t k;
  for (k = 0; k < n; ++k) {
    const uint8_t *b = rec + 8u * k;
    uint32_t pc = (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) |
                  ((uint32_t)b[3] << 24);
    uint32_t count = (uint32_t)b[4] | ((uint32_t)b[5] << 8);
    uint32_t reason = b[6];
    uint32_t flags = b[7];
    int lat = (int)(flags & 1u);
    int valid = pc < p->n_instr && reason < p->n_reasons && (flags & ~1u) == 0u &&
                !(lat && reason == R_NONE);
    if (!valid) {
      stats[1] += 1u;
      stats[2] += count;
      continue;
    }
    C[((uint64_t)pc * 2u + (uint64_t)lat) * p->n_reasons + reason] += count;
    stats[0] += count;
  }
  return 0;
}

/* ---------------------------------------------------------------- step 2-6: blame */

/* Rule 1, opcode based pruning: memory dependency stalls only to memory
 * instructions, synchronization stalls only to synchronization instructions.
 * Q6: memory = {GLOBAL, LOCAL, CONSTANT, TEXTURE}; shared memory is an execution
 * dependency source (Fig. 6); execution dependency has no opcode rule. */
static int rule1_keeps(uint32_t r, uint32_t def_class) {
  if (r == R_MEM)
    return def_class == C_GLOBAL || def_class == C_LOCAL || def_class == C_CONSTANT ||
           def_class == C_TEXTURE;
  if (r == R_SYNC) return def_class == C_SYNC;
  return 1;
}

/* Fig. 6: detailed category of an attributed dependency stall, chosen by
 * the opcode of the source (def) instruction; WAR is the execution sub-category of
 * P:412 (Q13); texture counts as global memory (Q14). */
static uint32_t classify(uint32_t r, uint32_t def_class, uint32_t kind) {
  if (r == R_MEM) {
    if (def_class == C_LOCAL) return COL_MEM_LOCAL;
    if (def_class == C_CONSTANT) return COL_MEM_CONSTANT;
    return COL_MEM_GLOBAL;
  }
  if (r == R_EXEC) {
    if (kind & K_WAR) return COL_EXEC_WAR;
    if (def_class == C_SHARED) return COL_EXEC_SHARED;
    return COL_EXEC_ARITH;
  }
  return COL_SYNC;
}

int or_blame(const or_program *p, const uint64_t *C, uint8_t *cand, uint8_t *self_flags,
             double *share, double *V) {
  const uint32_t n = p->n_instr, R = p->n_reasons, NC = or_ncol(R);
  const uint32_t E = p->row_ptr[n];
  uint32_t j, r, e;
  memset(cand, 0, E);
  memset(self_flags, 0, n);
  memset(share, 0, sizeof(double) * 3u * E);
  memset(V, 0, sizeof(double) * 2u * NC * n);

  for (j = 0; j < n; ++j) {
    /* S_j[r] (all samples of reason r at j) and SL_j[r] (latency samples) */
    uint64_t S[16], SL[16];
    uint64_t dep_total = 0;
    for (r = 0; r < R; ++r) {
      S[r] = cnt(p, C, j, 0, r) + cnt(p, C, j, 1, r);
      SL[r] = cnt(p, C, j, 1, r);
    }
    for (r = R_MEM; r <= R_SYNC; ++r) dep_total += S[r];

    /* the dependency graph is built from the def-use chains of instructions that
     * carry samples; only rows with dependency stalls get in-edges. */
    if (dep_total > 0) {
      for (r = R_MEM; r <= R_SYNC; ++r) {
        double W = 0.0;
        int any = 0;
        /* an edge i->j survives for reason r unless pruned by rule 1 (opcode),
         * rule 2 (a non-predicated k reading the operand lies on every i->j path: the
         * static field dom_k >= 0, Q7) or rule 3 (every i->j path is longer than
         * latency(i): min_len > latency, Q8). */
        for (e = p->row_ptr[j]; e < p->row_ptr[j + 1]; ++e) {
          uint32_t d = p->edge_def[e];
          int keep = rule1_keeps(r, p->opclass[d]) && p->edge_dom_k[e] < 0 &&
                     p->edge_min_len[e] <= p->latency[d];
          if (keep) {
            cand[e] |= (uint8_t)(1u << (r - 1u));
            any = 1;
          }
        }
        if (!any) {
          /* Q5: no surviving source -> the stall stays at j (self), never dropped. */
          self_flags[j] |= (uint8_t)(1u << (r - 1u));
          continue;
        }
        /* Eq. 1: weight R_path * R_issue with R_issue = issued (active)
         * samples of the def (Q3; at least 1, Q4) and R_path = 1 / longest path
         * length in instructions (Q1/Q2). */
        for (e = p->row_ptr[j]; e < p->row_ptr[j + 1]; ++e) {
          if (cand[e] & (1u << (r - 1u))) {
            uint32_t d = p->edge_def[e];
            uint64_t A_d = 0;
            uint32_t rr;
            for (rr = 0; rr < R; ++rr) A_d += cnt(p, C, d, 0, rr);
            W += (double)(A_d > 0 ? A_d : 1u) / (double)p->edge_max_len[e];
          }
        }
        for (e = p->row_ptr[j]; e < p->row_ptr[j + 1]; ++e) {
          if (cand[e] & (1u << (r - 1u))) {
            uint32_t d = p->edge_def[e];
            uint64_t A_d = 0;
            uint32_t rr, col;
            double w, sh;
            for (rr = 0; rr < R; ++rr) A_d += cnt(p, C, d, 0, rr);
            w = (double)(A_d > 0 ? A_d : 1u) / (double)p->edge_max_len[e];
            sh = w / W;
            share[3u * e + (r - 1u)] = sh;
            /* S_i = share * S_j, and the same share for latency samples. */
            col = classify(r, p->opclass[d], p->edge_kind[e]);
            V[((uint64_t)d * NC + col) * 2u + 0u] += (double)S[r] * sh;
            V[((uint64_t)d * NC + col) * 2u + 1u] += (double)SL[r] * sh;
          }
        }
      }
    }
    /* self-attributed dependency stalls stay at j */
    for (r = R_MEM; r <= R_SYNC; ++r) {
      if (self_flags[j] & (1u << (r - 1u))) {
        uint32_t col = COL_MEM_SELF + (r - 1u);
        V[((uint64_t)j * NC + col) * 2u + 0u] += (double)S[r];
        V[((uint64_t)j * NC + col) * 2u + 1u] += (double)SL[r];
      }
    }
    /* other stall reasons are caused by the instruction that suffers them. */
    for (r = 4; r < R; ++r) {
      uint32_t col = COL_PASS0 + (r - 4u);
      V[((uint64_t)j * NC + col) * 2u + 0u] += (double)S[r];
      V[((uint64_t)j * NC + col) * 2u + 1u] += (double)SL[r];
    }
  }
  return 0;
}

/* ---------------------------------------------------------------- step 7: rollup */

static int is_ancestor_or_self(const or_program *p, int32_t anc, int32_t l) {
  while (l >= 0) {
    if (l == anc) return 1;
    l = p->loop_parent[l];
  }
  return 0;
}

/* function f with func_begin[f] <= i < func_begin[f+1] (binary search over the ranges) */
static uint32_t func_of(const or_program *p, uint32_t i) {
  uint32_t lo = 0, hi = p->n_funcs;
  while (hi - lo > 1u) {
    uint32_t mid = (lo + hi) / 2u;
    if (p->func_begin[mid] <= i) lo = mid; else hi = mid;
  }
  return lo;
}

static uint32_t kernel_of_func(const or_program *p, uint32_t f) {
  uint32_t lo = 0, hi = p->n_kernels;
  while (hi - lo > 1u) {
    uint32_t mid = (lo + hi) / 2u;
    if (p->kernel_func_begin[mid] <= f) lo = mid; else hi = mid;
  }
  return lo;
}

static void add_row(double *dst, const double *src, uint32_t NC) {
  uint32_t q;
  for (q = 0; q < 2u * NC; ++q) dst[q] += src[q];
}

/* Program structure levels ("line, loop, function"), with loops both
 * exclusive and inclusive of nested loops (Eq. 5's nested(l) contains l, Q16).
 * Every instruction contributes its own V row (edge blame at the def, self and
 * pass-through at the use) and its (A_i, L_i) counts. */
int or_rollup(const or_program *p, const uint64_t *C, const double *V, double *line_v,
              uint64_t *line_al, double *loop_excl_v, uint64_t *loop_excl_al,
              double *loop_incl_v, uint64_t *loop_incl_al, double *func_v, uint64_t *func_al,
              double *kern_v, uint64_t *kern_al) {
  const uint32_t n = p->n_instr, R = p->n_reasons, NC = or_ncol(R);
  uint32_t i, r, l;
  if (line_v) memset(line_v, 0, sizeof(double) * 2u * NC * p->n_lines);
  if (line_al) memset(line_al, 0, sizeof(uint64_t) * 2u * p->n_lines);
  if (loop_excl_v) memset(loop_excl_v, 0, sizeof(double) * 2u * NC * p->n_loops);
  if (loop_excl_al) memset(loop_excl_al, 0, sizeof(uint64_t) * 2u * p->n_loops);
  if (loop_incl_v) memset(loop_incl_v, 0, sizeof(double) * 2u * NC * p->n_loops);
  if (loop_incl_al) memset(loop_incl_al, 0, sizeof(uint64_t) * 2u * p->n_loops);
  if (func_v) memset(func_v, 0, sizeof(double) * 2u * NC * p->n_funcs);
  if (func_al) memset(func_al, 0, sizeof(uint64_t) * 2u * p->n_funcs);
  if (kern_v) memset(kern_v, 0, sizeof(double) * 2u * NC * p->n_kernels);
  if (kern_al) memset(kern_al, 0, sizeof(uint64_t) * 2u * p->n_kernels);

  for (i = 0; i < n; ++i) {
    const double *row = V + (uint64_t)i * NC * 2u;
    uint64_t A = 0, L = 0;
    uint32_t f, k, ln = p->line_id[i];
    int32_t lp = p->loop_id[i];
    for (r = 0; r < R; ++r) {
      A += cnt(p, C, i, 0, r);
      L += cnt(p, C, i, 1, r);
    }
    if (line_v) add_row(line_v + (uint64_t)ln * NC * 2u, row, NC);
    if (line_al) { line_al[2u * ln] += A; line_al[2u * ln + 1u] += L; }
    if (lp >= 0) {
      if (loop_excl_v) add_row(loop_excl_v + (uint64_t)lp * NC * 2u, row, NC);
      if (loop_excl_al) { loop_excl_al[2u * lp] += A; loop_excl_al[2u * lp + 1u] += L; }
      /* nested(l) contains l: the instruction counts for its loop and every ancestor */
      for (l = (uint32_t)lp; ; l = (uint32_t)p->loop_parent[l]) {
        if (loop_incl_v) add_row(loop_incl_v + (uint64_t)l * NC * 2u, row, NC);
        if (loop_incl_al) { loop_incl_al[2u * l] += A; loop_incl_al[2u * l + 1u] += L; }
        if (p->loop_parent[l] < 0) break;
      }
    }
    f = func_of(p, i);
    k = kernel_of_func(p, f);
    if (func_v) add_row(func_v + (uint64_t)f * NC * 2u, row, NC);
    if (func_al) { func_al[2u * f] += A; func_al[2u * f + 1u] += L; }
    if (kern_v) add_row(kern_v + (uint64_t)k * NC * 2u, row, NC);
    if (kern_al) { kern_al[2u * k] += A; kern_al[2u * k + 1u] += L; }
  }
  return 0;
}

/* ---------------------------------------------------------------- step 8: estimators */

/* Eq. 2: S^e = T / (T - M).  T = 0 -> 1 (no samples, nothing to gain);
 * M >= T -> +inf (Q19). */
double or_eq2(double T, double M) {
  if (T <= 0.0) return 1.0;
  if (M >= T) return INFINITY;
  return T / (T - M);
}

/* Eq. 4: S^h = T / (T - min(A, M^L)). */
double or_eq4(double T, double A, double ML) {
  double m = A < ML ? A : ML;
  return or_eq2(T, m);
}

/* Eq. 5: S^h_l = T / (T - min(sum_{l' in nested(l)} A_l', M^L_l)). */
double or_eq5(double T, double A_nested, double ML_scope) {
  double m = A_nested < ML_scope ? A_nested : ML_scope;
  return or_eq2(T, m);
}

/* Eqs. 6-10: C_W = W_new / W; I = 1 - (1 - R_I)^W; I_new likewise;
 * C_I = I_new / I (:= 1 when I = 0, Q18); S^p = (1 / C_W) * C_I * f. */
double or_eq10(double W, double W_new, double R_I, double f) {
  double C_W = W_new / W;
  double I = 1.0 - pow(1.0 - R_I, W);
  double I_new = 1.0 - pow(1.0 - R_I, W_new);
  double C_I = (I == 0.0) ? 1.0 : I_new / I;
  return (1.0 / C_W) * C_I * f;
}

static int32_t lca_loop(const or_program *p, int32_t a, int32_t b) {
  int32_t x;
  for (x = a; x >= 0; x = p->loop_parent[x])
    if (is_ancestor_or_self(p, x, b)) return x;
  return -1;
}

static int instr_passes(const or_program *p, const or_pattern *q, uint32_t i) {
  if (!((q->class_mask >> p->opclass[i]) & 1u)) return 0;
  if (q->flag_filter && !(p->iflags[i] & q->flag_filter)) return 0;
  return 1;
}

/* Matched samples of pattern q contributed by one blamed item, and the loop it lives in
 * (-2 = not matched).  Edge contributions live at lca(def loop, use loop); self and
 * pass-through contributions at the use's loop (Q16). */
static double match_edge(const or_program *p, const uint64_t *C, const uint8_t *cand,
                         const double *share, const or_pattern *q, uint32_t e, uint32_t j) {
  uint32_t d = p->edge_def[e], r;
  double m = 0.0;
  if (!instr_passes(p, q, d)) return 0.0;
  if (q->same_loop && !(p->loop_id[d] >= 0 && p->loop_id[d] == p->loop_id[j])) return 0.0;
  for (r = R_MEM; r <= R_SYNC; ++r) {
    if (cand[e] & (1u << (r - 1u))) {
      uint32_t col = classify(r, p->opclass[d], p->edge_kind[e]);
      if ((q->column_mask >> col) & 1u) {
        uint64_t X = cnt(p, C, j, 1, r) + (q->sample_class ? 0u : cnt(p, C, j, 0, r));
        m += (double)X * share[3u * e + (r - 1u)];
      }
    }
  }
  return m;
}

static double match_instr(const or_program *p, const uint64_t *C, const uint8_t *self_flags,
                          const or_pattern *q, uint32_t j) {
  uint32_t r;
  double m = 0.0;
  if (!instr_passes(p, q, j)) return 0.0;
  if (q->same_loop && p->loop_id[j] < 0) return 0.0;
  for (r = R_MEM; r <= R_SYNC; ++r) {
    if ((self_flags[j] & (1u << (r - 1u))) && ((q->column_mask >> (COL_MEM_SELF + r - 1u)) & 1u))
      m += (double)(cnt(p, C, j, 1, r) + (q->sample_class ? 0u : cnt(p, C, j, 0, r)));
  }
  for (r = 4; r < p->n_reasons; ++r) {
    if ((q->column_mask >> (COL_PASS0 + r - 4u)) & 1u)
      m += (double)(cnt(p, C, j, 1, r) + (q->sample_class ? 0u : cnt(p, C, j, 0, r)));
  }
  return m;
}

/* Table 2 optimizers as patterns, the Loop Unrolling workflow,
 * and the estimators of §5.2 per kernel launch context. */
int or_estimate_all(const or_program *p, const uint64_t *C, const uint8_t *cand,
                    const uint8_t *self_flags, const double *share, const or_pattern *pats,
                    uint32_t n_pat, or_estimate *out) {
  return or_estimate_all_occ(p, C, cand, self_flags, share, pats, n_pat, NULL, out);
}

int or_estimate_all_occ(const or_program *p, const uint64_t *C, const uint8_t *cand,
                        const uint8_t *self_flags, const double *share, const or_pattern *pats,
                        uint32_t n_pat, const or_occ *occ, or_estimate *out) {
  const uint32_t n = p->n_instr, R = p->n_reasons;
  uint32_t k, qi, i, r, e, l, f;
  double *loopM = (double *)calloc(p->n_loops ? p->n_loops : 1u, sizeof(double));
  double *loopA = (double *)calloc(p->n_loops ? p->n_loops : 1u, sizeof(double));
  double *funcM = (double *)calloc(p->n_funcs ? p->n_funcs : 1u, sizeof(double));
  double *funcA = (double *)calloc(p->n_funcs ? p->n_funcs : 1u, sizeof(double));
  int32_t *loop_func = (int32_t *)malloc(sizeof(int32_t) * (p->n_loops ? p->n_loops : 1u));
  if (!loopM || !loopA || !funcM || !funcA || !loop_func) return -1;

  /* function owning each loop: that of any instruction in the loop's subtree */
  for (l = 0; l < p->n_loops; ++l) loop_func[l] = -1;
  for (i = 0; i < n; ++i) {
    int32_t x;
    for (x = p->loop_id[i]; x >= 0; x = p->loop_parent[x])
      if (loop_func[x] < 0) loop_func[x] = (int32_t)func_of(p, i);
  }

  for (k = 0; k < p->n_kernels; ++k) {
    uint32_t f0 = p->kernel_func_begin[k], f1 = p->kernel_func_begin[k + 1];
    uint32_t i0 = p->func_begin[f0], i1 = p->func_begin[f1];
    uint64_t T = 0, A = 0;
    double R_I;
    /* T, A, L of the kernel; R_I = issued / all samples */
    for (i = i0; i < i1; ++i)
      for (r = 0; r < R; ++r) {
        A += cnt(p, C, i, 0, r);
        T += cnt(p, C, i, 0, r) + cnt(p, C, i, 1, r);
      }
    R_I = T ? (double)A / (double)T : 0.0;

    for (qi = 0; qi < n_pat; ++qi) {
      const or_pattern *q = &pats[qi];
      or_estimate *o = &out[(uint64_t)k * n_pat + qi];
      double M = 0.0, best = 1.0;
      int32_t best_scope = -1;
      memset(o, 0, sizeof(*o));
      o->T = T;
      o->A = A;
      o->model = q->model;
      o->best_scope = -1;

      if (q->model == 5) {
        /* Parallel optimizers (Table 2): Block Increase matches when the
         * kernel has fewer blocks than SMs; Eq. 10 otherwise from caller W, W_new, f. */
        int matched = q->parallel_rule == 1 ||
                      (q->parallel_rule == 2 && p->kernel_grid_blocks &&
                       p->kernel_grid_blocks[k] < q->sm_count);
        double W = q->W, W_new = q->W_new;
        if (q->parallel_rule == 3 || q->parallel_rule == 4) {   /* occupancy model (Q34) */
          matched = occ && (q->parallel_rule == 3 ? occ[k].match_block : occ[k].match_thread);
          if (matched) {
            W = occ[k].W;
            W_new = q->parallel_rule == 3 ? occ[k].W_new_block : occ[k].W_new_thread;
          }
        }
        o->matched = (uint8_t)matched;
        o->speedup = matched ? or_eq10(W, W_new, R_I, q->f) : 1.0;
        o->eq3 = o->eq4 = 1.0;
        continue;
      }

      for (l = 0; l < p->n_loops; ++l) { loopM[l] = 0.0; loopA[l] = 0.0; }
      for (f = 0; f < p->n_funcs; ++f) { funcM[f] = 0.0; funcA[f] = 0.0; }

      for (i = i0; i < i1; ++i) {
        uint32_t fi = func_of(p, i);
        uint64_t Ai = 0;
        double mi;
        for (r = 0; r < R; ++r) Ai += cnt(p, C, i, 0, r);
        int32_t x;
        funcA[fi] += (double)Ai;
        for (x = p->loop_id[i]; x >= 0; x = p->loop_parent[x]) loopA[x] += (double)Ai;
        /* contributions of in-edges of use i */
        for (e = p->row_ptr[i]; e < p->row_ptr[i + 1]; ++e) {
          double me = match_edge(p, C, cand, share, q, e, i);
          int32_t sc;
          if (me == 0.0) continue;
          M += me;
          funcM[fi] += me;
          sc = lca_loop(p, p->loop_id[p->edge_def[e]], p->loop_id[i]);
          for (x = sc; x >= 0; x = p->loop_parent[x]) loopM[x] += me;
        }
        mi = match_instr(p, C, self_flags, q, i);
        if (mi != 0.0) {
          M += mi;
          funcM[fi] += mi;
          for (x = p->loop_id[i]; x >= 0; x = p->loop_parent[x]) loopM[x] += mi;
        }
      }
      o->M = M;
      o->matched = M > 0.0;
      o->eq3 = or_eq2((double)T, M);                 /* Eq. 3 */
      o->eq4 = or_eq4((double)T, (double)A, M);      /* Eq. 4 */
      if (q->model == 0) {
        o->speedup = or_eq2((double)T, q->ratio * M); /* Eq. 2 (x ratio, Q17) */
      } else if (q->model == 1) {
        o->speedup = o->eq4;
      } else {
        /* Eq. 5 per scope; the optimizer's estimate is its best scope (Q16). */
        if (q->model == 2 || q->model == 4) {
          for (l = 0; l < p->n_loops; ++l) {
            double s;
            if (loop_func[l] < (int32_t)f0 || loop_func[l] >= (int32_t)f1) continue;
            s = or_eq5((double)T, loopA[l], loopM[l]);
            if (best_scope < 0 || s > best) { best = s; best_scope = (int32_t)l; }
          }
        }
        if (q->model == 3 || q->model == 4) {
          for (f = f0; f < f1; ++f) {
            double s = or_eq5((double)T, funcA[f], funcM[f]);
            if (best_scope < 0 || s > best) { best = s; best_scope = (int32_t)(p->n_loops + f); }
          }
        }
        o->speedup = best_scope < 0 ? 1.0 : best;
        o->best_scope = best_scope;
      }
      o->unbounded = isinf(o->speedup) ? 1u : 0u;
    }
  }
  free(loopM); free(loopA); free(funcM); free(funcA); free(loop_func);
  return 0;
}

/* ---------------------------------------------------------------- after the path: advice */

/* Hotspots ("Each optimizer ... lists several hotspots to focus on.  Each hotspot
 * consists of the def and use locations and their distance"; "the top five hotspots").
 * The items of a kernel are its edges (def -> use, matched samples of match_edge) and its
 * instructions (own self / pass-through samples, match_instr); Q30. */
static int hot_before(double sa, uint32_t ia, double sb, uint32_t ib) {
  return sa > sb || (sa == sb && ia < ib);
}

int or_hotspots(const or_program *p, const uint64_t *C, const uint8_t *cand,
                const uint8_t *self_flags, const double *share, const or_pattern *pats,
                uint32_t n_pat, uint32_t top_k, or_hotspot *out, uint32_t *n_out) {
  const uint32_t E = p->row_ptr[p->n_instr];
  uint32_t k, qi, j, e;
  for (k = 0; k < p->n_kernels; ++k) {
    uint32_t i0 = p->func_begin[p->kernel_func_begin[k]], i1 = p->func_begin[p->kernel_func_begin[k + 1]];
    for (qi = 0; qi < n_pat; ++qi) {
      const or_pattern *q = &pats[qi];
      or_hotspot *h = &out[((uint64_t)k * n_pat + qi) * top_k];
      uint32_t n = 0;
      if (q->model != 5) {
        for (j = i0; j < i1; ++j) {
          for (e = p->row_ptr[j]; e <= p->row_ptr[j + 1]; ++e) {
            or_hotspot x;
            uint32_t t;
            if (e < p->row_ptr[j + 1]) {   /* an in-edge of j */
              x.def_pc = p->edge_def[e]; x.use_pc = j; x.distance = p->edge_max_len[e]; x.item = e;
              x.samples = match_edge(p, C, cand, share, q, e, j);
            } else {                       /* j's own samples */
              x.def_pc = j; x.use_pc = j; x.distance = 0; x.item = E + j;
              x.samples = match_instr(p, C, self_flags, q, j);
            }
            if (!(x.samples > 0.0)) continue;
            /* insertion into the sorted top list */
            if (n == top_k && !hot_before(x.samples, x.item, h[n - 1].samples, h[n - 1].item)) continue;
            t = n < top_k ? n++ : n - 1;
            while (t > 0 && hot_before(x.samples, x.item, h[t - 1].samples, h[t - 1].item)) {
              h[t] = h[t - 1];
              --t;
            }
            h[t] = x;
          }
        }
      }
      n_out[(uint64_t)k * n_pat + qi] = n;
    }
  }
  return 0;
}

/* P:261 "an advice report that contains suggestions from its top optimizers sorted by their
 * estimated speedups"; Q31. */
int or_rank(const or_estimate *est, uint32_t n_kernels, uint32_t n_pat, uint32_t *order) {
  uint32_t k, a, b;
  for (k = 0; k < n_kernels; ++k) {
    uint32_t *o = &order[(uint64_t)k * n_pat];
    const or_estimate *x = &est[(uint64_t)k * n_pat];
    for (a = 0; a < n_pat; ++a) o[a] = a;
    for (a = 1; a < n_pat; ++a) {          /* stable insertion sort, descending speedup */
      uint32_t v = o[a];
      b = a;
      while (b > 0 && x[o[b - 1]].speedup < x[v].speedup) {
        o[b] = o[b - 1];
        --b;
      }
      o[b] = v;
    }
  }
  return 0;
}

/* P:658-659 "a node is a single dependency node if the node does not have any incoming edge,
 * or each incoming edge represents a different dependency.  ... single dependency coverage as
 * the ratio of single dependency nodes to the total number of nodes."  Q32: nodes are the
 * instructions with dependency-stall samples; before pruning every in-edge may represent each
 * dependency, after pruning an edge represents the reasons of its candidate mask (rules 1-3). */
int or_coverage(const or_program *p, const uint64_t *C, const uint8_t *cand, uint64_t *out) {
  uint32_t k, j, e, r;
  for (k = 0; k < p->n_kernels; ++k) {
    uint32_t i0 = p->func_begin[p->kernel_func_begin[k]], i1 = p->func_begin[p->kernel_func_begin[k + 1]];
    uint64_t nodes = 0, before = 0, after = 0;
    for (j = i0; j < i1; ++j) {
      int live = 0, single_b = 1, single_a = 1;
      uint32_t deg = p->row_ptr[j + 1] - p->row_ptr[j];
      for (r = R_MEM; r <= R_SYNC; ++r) {
        uint32_t n_r = 0;
        if (cnt(p, C, j, 0, r) + cnt(p, C, j, 1, r) == 0) continue;   /* no stall of this kind */
        live = 1;
        for (e = p->row_ptr[j]; e < p->row_ptr[j + 1]; ++e)
          if (cand[e] & (1u << (r - 1u))) ++n_r;
        if (deg > 1) single_b = 0;
        if (n_r > 1) single_a = 0;
      }
      if (!live) continue;
      ++nodes;
      before += (uint64_t)single_b;
      after += (uint64_t)single_a;
    }
    out[3 * (uint64_t)k] = nodes;
    out[3 * (uint64_t)k + 1] = before;
    out[3 * (uint64_t)k + 2] = after;
  }
  return 0;
}

/* ---------------------------------------------------------------- occupancy (NEXT #4)
 * The standard occupancy calculation (SPEC's invented plumbing; the paper names the limits,
 * P:443-444, without a formula): blocks per SM = min over the warp, block-slot, register and
 * shared-memory limits; W = resident warps per scheduler.  Block Increase (grid < #SM) spreads
 * the same warps over all SMs, W_new = W * grid / #SM; Thread Increase matches when block slots
 * bind and a full grid stays resident, W_new = the warp or register limit.  Q34. */
int or_occupancy(const or_arch *a, const or_launch *L, const uint32_t *grid_blocks, uint32_t n_kernels,
                 or_occ *out) {
  uint32_t k;
  for (k = 0; k < n_kernels; ++k) {
    or_occ *o = &out[k];
    const or_launch *l = &L[k];
    uint32_t wpb, rpw, lim[4], i, grid, want, resident;
    memset(o, 0, sizeof(*o));
    if (!l->threads_per_block || !a->warp_size || !a->schedulers_per_sm || !a->sm_count) continue;
    wpb = (l->threads_per_block + a->warp_size - 1) / a->warp_size;
    rpw = l->regs_per_thread
              ? (l->regs_per_thread * a->warp_size + a->reg_alloc_unit - 1) / a->reg_alloc_unit * a->reg_alloc_unit
              : 0;
    lim[0] = a->max_warps_per_sm / wpb;
    lim[1] = a->max_blocks_per_sm;
    lim[2] = rpw ? a->regs_per_sm / (rpw * wpb) : 0xffffffffu;
    lim[3] = l->smem_per_block ? a->smem_per_sm / l->smem_per_block : 0xffffffffu;
    o->blocks_per_sm = lim[0];
    o->limiter = 0;
    for (i = 1; i < 4; ++i)
      if (lim[i] < o->blocks_per_sm) { o->blocks_per_sm = lim[i]; o->limiter = i; }
    if (!o->blocks_per_sm) continue;   /* the launch cannot run */
    grid = grid_blocks ? grid_blocks[k] : 0;
    if (!grid) continue;
    want = (grid + a->sm_count - 1) / a->sm_count;
    resident = want < o->blocks_per_sm ? want : o->blocks_per_sm;
    o->W = (double)resident * wpb / a->schedulers_per_sm;
    if (grid < a->sm_count) {
      o->match_block = 1;
      o->W_new_block = o->W * grid / a->sm_count;
    }
    if (o->limiter == 1 && resident == o->blocks_per_sm) {
      uint32_t warps = a->max_warps_per_sm;
      if (rpw && a->regs_per_sm / rpw < warps) warps = a->regs_per_sm / rpw;
      o->W_new_thread = (double)warps / a->schedulers_per_sm;
      o->match_thread = o->W_new_thread > o->W;
    }
  }
  return 0;
}

/* ---------------------------------------------------------------- backward slicing (NEXT #1)
 * P:289-321; readings DESIGN.md §3.2 Q35-Q39 (definitions over backward paths, the same
 * ones tests/slice_enum.py evaluates by listing paths).
 *
 * For a use j and a register r that j reads (a source operand, its guard predicate, or a virtual
 * barrier register B0-B5 of its wait mask), a backward path is x_1, x_2, ... with
 * x_1 in prev(j) and x_{t+1} in prev(x_t), inside j's function; prev(x) = x-1 inside a block, else
 * the last instruction of every predecessor block.  P = the union of the predicates of the defs of
 * r passed so far; the path stops after a def x_t of r once P contains j's predicate.
 * Every def of r met at step t is a dependency source at length t.  A step from the first
 * instruction x of a block to the last instruction y of a predecessor block crosses a back edge
 * when y >= x.  For a def i:
 *   min_len = the fewest steps over the paths reaching i,
 *   K*      = the fewest back-edge crossings over those paths,
 *   max_len = the most steps over the paths with exactly K* crossings ("the longest one"; the
 *             unrolled-once convention of SPEC S:185: a back edge only when the pair needs it),
 *   dom_k   = the smallest unpredicated k (k != i, j) reading every register linking i and j that
 *             lies on every such path (rule 2), else -1.
 * A search state is (x, P); states with the crossing count added, (x, P, k), form "layers" k in
 * which every step goes to a lower address, so each layer is a DAG processed by descending x. */

#define SL_ALL 0x4000u   /* the '_' predicate */
#define SL_NONE 0xFFFFu
#define SL_NIL 0xFFFFFFFFu

static uint32_t sl_pbit(uint8_t g) {          /* predicate of an instruction as a P-set bit */
  uint32_t r = g & 7u;
  if (r == 7u) return SL_ALL;
  return (g & 8u) ? (1u << (7u + r)) : (1u << r);
}
static uint32_t sl_union(uint32_t P, uint32_t b) {   /* P + {b}, with {p_i, !p_i} = {_} */
  uint32_t i;
  P |= b;
  for (i = 0; i < 7; ++i)
    if ((P >> i & 1u) && (P >> (7 + i) & 1u)) P |= SL_ALL;
  return P;
}
static int sl_contains(uint32_t P, uint32_t b) { return (P & SL_ALL) || (P & b); }

/* registers read by x: out[] = 0..254 (R), 256..262 (P), 512+b (B_b); kinds[] = REG / PRED / BAR */
static int sl_reads(const or_sass *s, uint32_t x, uint32_t *out, uint8_t *kinds) {
  int n = 0, t;
  for (t = 0; t < 4; ++t) {
    uint16_t r = s->src[4u * x + t];
    if (r == SL_NONE || r == 255u) continue;
    out[n] = r; kinds[n] = r >= 256u ? 2u : 1u; ++n;
  }
  if ((s->guard[x] & 7u) != 7u) { out[n] = 256u + (s->guard[x] & 7u); kinds[n] = 2u; ++n; }
  for (t = 0; t < 6; ++t)
    if (s->wait[x] >> t & 1u) { out[n] = 512u + t; kinds[n] = 4u; ++n; }
  return n;
}
static int sl_defines(const or_sass *s, uint32_t x, uint32_t r) {   /* P:301-302 for barriers */
  int t;
  if (r >= 512u) return ((s->wbar[x] | s->rbar[x]) >> (r - 512u)) & 1u;
  for (t = 0; t < 4; ++t)
    if (s->dst[4u * x + t] == r) return 1;
  return 0;
}
static int sl_reads_reg(const or_sass *s, uint32_t x, uint32_t r) {
  uint32_t rr[16];
  uint8_t kk[16];
  int n = sl_reads(s, x, rr, kk), t;
  for (t = 0; t < n; ++t)
    if (rr[t] == r) return 1;
  return 0;
}

typedef struct {                 /* the CFG at instruction level */
  const or_sass *s;
  uint32_t *blk_of, *pred_ptr, *pred;
  uint32_t *kids, *roots;        /* prev() output buffers (max predecessor count + 1) */
} sl_cfg;

/* prev(x): x-1 inside its block, else the last instruction of each predecessor block */
static int sl_prev(const sl_cfg *c, uint32_t x, uint32_t *out) {
  uint32_t b = c->blk_of[x], e;
  int n = 0;
  if (x > c->s->block_begin[b]) { out[0] = x - 1; return 1; }
  for (e = c->pred_ptr[b]; e < c->pred_ptr[b + 1]; ++e) out[n++] = c->s->block_begin[c->pred[e] + 1] - 1;
  return n;
}

/* a growable list of search states (x, P, k) with a per-instruction chain for lookups; states are
 * appended in discovery order, so a breadth-first search walks the list itself as its queue */
typedef struct {
  uint32_t n, cap;
  uint32_t *x, *P, *k, *next, *val;   /* val: distance (BFS) or longest length (layers) */
  uint8_t *flag;
  uint32_t *head;                     /* [n_instr] latest state of instruction x, SL_NIL if none */
} sl_states;

static void sl_states_init(sl_states *S, uint32_t n_instr) {
  uint32_t i;
  S->n = 0; S->cap = 64;
  S->x = (uint32_t *)malloc(4u * S->cap); S->P = (uint32_t *)malloc(4u * S->cap);
  S->k = (uint32_t *)malloc(4u * S->cap); S->next = (uint32_t *)malloc(4u * S->cap);
  S->val = (uint32_t *)malloc(4u * S->cap); S->flag = (uint8_t *)malloc(S->cap);
  S->head = (uint32_t *)malloc(4u * (n_instr ? n_instr : 1));
  for (i = 0; i < n_instr; ++i) S->head[i] = SL_NIL;
}
static void sl_states_clear(sl_states *S) {
  uint32_t i;
  for (i = 0; i < S->n; ++i) S->head[S->x[i]] = SL_NIL;
  S->n = 0;
}
static void sl_states_free(sl_states *S) {
  free(S->x); free(S->P); free(S->k); free(S->next); free(S->val); free(S->flag); free(S->head);
}
static uint32_t sl_find(const sl_states *S, uint32_t x, uint32_t P, uint32_t k) {
  uint32_t i;
  for (i = S->head[x]; i != SL_NIL; i = S->next[i])
    if (S->P[i] == P && S->k[i] == k) return i;
  return SL_NIL;
}
static uint32_t sl_add(sl_states *S, uint32_t x, uint32_t P, uint32_t k, uint32_t val) {
  uint32_t i = S->n++;
  if (i == S->cap) {
    S->cap *= 2;
    S->x = (uint32_t *)realloc(S->x, 4u * S->cap); S->P = (uint32_t *)realloc(S->P, 4u * S->cap);
    S->k = (uint32_t *)realloc(S->k, 4u * S->cap); S->next = (uint32_t *)realloc(S->next, 4u * S->cap);
    S->val = (uint32_t *)realloc(S->val, 4u * S->cap); S->flag = (uint8_t *)realloc(S->flag, S->cap);
  }
  S->x[i] = x; S->P[i] = P; S->k[i] = k; S->val[i] = val; S->flag[i] = 0;
  S->next[i] = S->head[x]; S->head[x] = i;
  return i;
}

/* what a path carries past state (x, P): the new P, and whether the path stops at x */
static uint32_t sl_pass(const or_sass *s, uint32_t x, uint32_t P, uint32_t r, uint32_t pj, int *stop) {
  *stop = 0;
  if (!sl_defines(s, x, r)) return P;
  P = sl_union(P, sl_pbit(s->guard[x]));
  *stop = sl_contains(P, pj);
  return P;
}

/* per (use j, def i) accumulator over the registers linking them */
typedef struct {
  uint32_t def, mn, kstar, mx;
  uint8_t kind;
  uint8_t *dom_ok;   /* [function length]: k = f0 + index still qualifies for rule 2 */
  uint8_t *sep;      /* scratch: k separates the def from j for the current register */
} sl_acc;

/* breadth-first search from the roots over (x, P) (k = 0), never entering instruction `blocked`
 * (SL_NIL: none); val = path length */
static void sl_bfs(const sl_cfg *c, const uint32_t *roots, int nroot, uint32_t r, uint32_t pj, uint32_t blocked,
                   sl_states *S) {
  uint32_t u;
  int q, nk, stop;
  sl_states_clear(S);
  for (q = 0; q < nroot; ++q)
    if (roots[q] != blocked && sl_find(S, roots[q], 0u, 0u) == SL_NIL) sl_add(S, roots[q], 0u, 0u, 1u);
  for (u = 0; u < S->n; ++u) {
    const uint32_t Pout = sl_pass(c->s, S->x[u], S->P[u], r, pj, &stop);
    if (stop) continue;
    nk = sl_prev(c, S->x[u], c->kids);
    for (q = 0; q < nk; ++q)
      if (c->kids[q] != blocked && sl_find(S, c->kids[q], Pout, 0u) == SL_NIL)
        sl_add(S, c->kids[q], Pout, 0u, S->val[u] + 1u);
  }
}

/* One register r of use j (function [f0, f1)): merges into acc[] the defs of r the search reaches
 * -- their kinds, minimum lengths (breadth-first over (x, P)), K* and the longest length at K*
 * (layers), and the rule-2 candidates (the breadth-first search with each candidate removed). */
static void sl_register(const sl_cfg *c, uint32_t f0, uint32_t f1, uint32_t j, uint32_t r, uint8_t kind,
                        sl_states *bfs, sl_states *lay, sl_acc *acc, uint32_t *n_acc) {
  const or_sass *s = c->s;
  const uint32_t pj = sl_pbit(s->guard[j]), nf = f1 - f0;
  uint32_t i, a, L, x, k;
  const int nroot = sl_prev(c, j, c->roots);
  int q, nk, stop;

  /* ---- minimum lengths; the defs reached, their kinds */
  sl_bfs(c, c->roots, nroot, r, pj, SL_NIL, bfs);
  for (i = 0; i < bfs->n; ++i) {
    const uint32_t d = bfs->x[i];
    uint8_t kk = kind;
    if (!sl_defines(s, d, r)) continue;
    for (a = 0; a < *n_acc && acc[a].def != d; ++a) {}
    if (a == *n_acc) {                           /* first register linking d to j */
      acc[a].def = d; acc[a].mn = SL_NIL; acc[a].kstar = SL_NIL; acc[a].mx = 0; acc[a].kind = 0;
      memset(acc[a].dom_ok, 1, nf);
      ++*n_acc;
    }
    if (bfs->val[i] < acc[a].mn) acc[a].mn = bfs->val[i];
    if (r >= 512u && ((s->rbar[d] >> (r - 512u)) & 1u)) {   /* WAR: j overwrites what d reads */
      int tt, uu;
      for (tt = 0; tt < 4; ++tt)
        for (uu = 0; uu < 4; ++uu) {
          const uint16_t w = s->dst[4u * j + tt];
          if (w != SL_NONE && w != 255u && w == s->src[4u * d + uu]) kk |= 8u;
        }
    }
    acc[a].kind |= kk;
  }

  /* ---- layers k = 0, 1, ...: the longest length of every (x, P, k); stop after a layer that
   *      adds no (x, P) pair absent from the layers below (no later layer can add one then).
   *      bfs->flag marks the (x, P) pairs met in some layer so far. */
  sl_states_clear(lay);
  for (i = 0; i < bfs->n; ++i) bfs->flag[i] = 0;
  for (q = 0; q < nroot; ++q) {
    const uint32_t k0 = c->roots[q] >= j ? 1u : 0u;
    if (sl_find(lay, c->roots[q], 0u, k0) == SL_NIL) sl_add(lay, c->roots[q], 0u, k0, 1u);
  }
  for (L = 0;; ++L) {
    int any = 0, fresh = 0;
    for (x = f1; x-- > f0;) {                    /* descending address: in-layer steps go down */
      uint32_t st;
      for (st = lay->head[x]; st != SL_NIL; st = lay->next[st]) {
        uint32_t Pout, pair;
        if (lay->k[st] != L) continue;
        any = 1;
        pair = sl_find(bfs, x, lay->P[st], 0u);
        if (!bfs->flag[pair]) { bfs->flag[pair] = 1; fresh = 1; }
        Pout = sl_pass(s, x, lay->P[st], r, pj, &stop);
        if (stop) continue;
        nk = sl_prev(c, x, c->kids);
        for (q = 0; q < nk; ++q) {
          const uint32_t k2 = L + (c->kids[q] >= x ? 1u : 0u);
          const uint32_t t = sl_find(lay, c->kids[q], Pout, k2);
          if (t == SL_NIL) sl_add(lay, c->kids[q], Pout, k2, lay->val[st] + 1u);
          else if (lay->val[st] + 1u > lay->val[t]) lay->val[t] = lay->val[st] + 1u;
        }
      }
    }
    /* layer 0 is empty only when every root is behind a back edge: go on to layer 1 then */
    if (any ? !fresh : L > 0) break;
  }
  for (i = 0; i < lay->n; ++i) {                 /* K* and the longest length at K* */
    const uint32_t d = lay->x[i];
    if (!sl_defines(s, d, r)) continue;
    for (a = 0; a < *n_acc && acc[a].def != d; ++a) {}
    if (lay->k[i] < acc[a].kstar) { acc[a].kstar = lay->k[i]; acc[a].mx = lay->val[i]; }
    else if (lay->k[i] == acc[a].kstar && lay->val[i] > acc[a].mx) acc[a].mx = lay->val[i];
  }

  /* ---- rule 2 for this register: k separates def d from j iff k reads r, has no guard, k is
   *      neither d nor j, and the search with k removed reaches no state of d */
  for (a = 0; a < *n_acc; ++a) memset(acc[a].sep, 0, nf);
  for (k = f0; k < f1; ++k) {
    if (k == j || (s->guard[k] & 7u) != 7u || !sl_reads_reg(s, k, r)) continue;
    sl_bfs(c, c->roots, nroot, r, pj, k, lay);   /* lay reused */
    for (a = 0; a < *n_acc; ++a)
      if (acc[a].def != k && lay->head[acc[a].def] == SL_NIL) acc[a].sep[k - f0] = 1;
  }
  for (a = 0; a < *n_acc; ++a)                   /* the defs r links to j: dom_ok &= sep */
    if (sl_defines(s, acc[a].def, r) && bfs->head[acc[a].def] != SL_NIL)
      for (k = 0; k < nf; ++k) acc[a].dom_ok[k] &= acc[a].sep[k];
}

int64_t or_slice(const or_sass *s, uint64_t cap, uint32_t *row_ptr, uint32_t *edge_def, uint8_t *edge_kind,
                 uint32_t *edge_min, uint32_t *edge_max, int32_t *edge_dom) {
  const uint32_t n = s->n_instr, NB = s->n_blocks;
  sl_cfg c;
  uint32_t *fill = (uint32_t *)calloc(NB + 1, sizeof(uint32_t));
  uint32_t b, e, j, f, maxf = 1, maxp = 1, a, a2;
  uint64_t E = 0;
  int64_t ret = -1;
  sl_states bfs, lay;
  sl_acc *acc;
  c.s = s;
  c.blk_of = (uint32_t *)malloc(sizeof(uint32_t) * (n ? n : 1));
  c.pred_ptr = (uint32_t *)calloc(NB + 1, sizeof(uint32_t));
  c.pred = (uint32_t *)malloc(sizeof(uint32_t) * (s->succ_ptr[NB] ? s->succ_ptr[NB] : 1));
  for (b = 0; b < NB; ++b)
    for (j = s->block_begin[b]; j < s->block_begin[b + 1]; ++j) c.blk_of[j] = b;
  for (b = 0; b < NB; ++b)
    for (e = s->succ_ptr[b]; e < s->succ_ptr[b + 1]; ++e) c.pred_ptr[s->succ[e] + 1]++;
  for (b = 0; b < NB; ++b) {
    if (c.pred_ptr[b + 1] > maxp) maxp = c.pred_ptr[b + 1];
    c.pred_ptr[b + 1] += c.pred_ptr[b];
  }
  for (b = 0; b < NB; ++b)                       /* ascending source block id per target */
    for (e = s->succ_ptr[b]; e < s->succ_ptr[b + 1]; ++e) {
      uint32_t t = s->succ[e];
      c.pred[c.pred_ptr[t] + fill[t]++] = b;
    }
  c.kids = (uint32_t *)malloc(4u * (maxp + 1u));
  c.roots = (uint32_t *)malloc(4u * (maxp + 1u));
  for (f = 0; f < s->n_funcs; ++f)
    if (s->func_begin[f + 1] - s->func_begin[f] > maxf) maxf = s->func_begin[f + 1] - s->func_begin[f];
  sl_states_init(&bfs, n);
  sl_states_init(&lay, n);
  acc = (sl_acc *)malloc(sizeof(sl_acc) * maxf);
  for (a = 0; a < maxf; ++a) { acc[a].dom_ok = (uint8_t *)malloc(maxf); acc[a].sep = (uint8_t *)malloc(maxf); }
  row_ptr[0] = 0;
  for (f = 0, j = 0; j < n; ++j) {
    uint32_t reads[16], n_acc = 0;
    uint8_t kinds[16];
    const int nr = sl_reads(s, j, reads, kinds);
    int ri;
    while (s->func_begin[f + 1] <= j) ++f;
    for (ri = 0; ri < nr; ++ri)
      sl_register(&c, s->func_begin[f], s->func_begin[f + 1], j, reads[ri], kinds[ri], &bfs, &lay, acc, &n_acc);
    for (a = 1; a < n_acc; ++a)                  /* defs ascending */
      for (a2 = a; a2 > 0 && acc[a2 - 1].def > acc[a2].def; --a2) {
        const sl_acc t0 = acc[a2]; acc[a2] = acc[a2 - 1]; acc[a2 - 1] = t0;
      }
    for (a = 0; a < n_acc; ++a) {
      int32_t dom = -1;
      uint32_t k;
      if (E >= cap) goto fail;
      for (k = 0; k < s->func_begin[f + 1] - s->func_begin[f] && dom < 0; ++k)
        if (acc[a].dom_ok[k]) dom = (int32_t)(s->func_begin[f] + k);
      edge_def[E] = acc[a].def; edge_kind[E] = acc[a].kind;
      edge_min[E] = acc[a].mn; edge_max[E] = acc[a].mx; edge_dom[E] = dom;
      ++E;
    }
    row_ptr[j + 1] = (uint32_t)E;
  }
  ret = (int64_t)E;
fail:
  free(fill); free(c.blk_of); free(c.pred_ptr); free(c.pred); free(c.kids); free(c.roots);
  sl_states_free(&bfs); sl_states_free(&lay);
  for (a = 0; a < maxf; ++a) { free(acc[a].dom_ok); free(acc[a].sep); }
  free(acc);
  return ret;
}

/* ---------------------------------------------------------------- sampling simulator (NEXT #3)
 * each SM has warp schedulers with active warps; every sampling period the SM records
 * a sample for one of its schedulers, cycling round-robin: an active sample if that scheduler is
 * issuing, a latency sample otherwise, with the sampled warp's stall reason if any.  The model
 * (SPEC's invented plumbing; Q40-Q44): in-order issue, one instruction per scheduler per cycle,
 * loose round-robin among ready warps; a register is ready `latency` cycles after its producer
 * issues, a write barrier clears `latency` cycles after, a read barrier `rbar_latency` after; a
 * warp waits for its sources and the barriers of its wait mask.  Predicated-off instructions issue
 * as no-ops.  Loops (self-loop blocks) run trip_count times; a two-way branch goes to successor
 * (warp mod 2). */

#define SIM_REGS 263u    /* R0-R254, RZ, P0-P6 */
#define R_NOTSEL 7u

static uint64_t sim_mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

typedef struct {
  uint32_t pc, done, loop_count, last_pc;
  int64_t last_issue;
  int64_t ready[SIM_REGS];  int32_t prod[SIM_REGS];
  int64_t bclear[6];        int32_t bprod[6];
  uint32_t predv;           /* bit k = value of P_k */
} sim_warp;

static int sim_is_mem(uint8_t c) { return c == 0 || c == 1 || c == 3 || c == 4; }   /* GLOBAL LOCAL CONSTANT TEXTURE */

/* blocking requirement of the warp's next instruction at cycle t: returns 1 if ready; else the
 * reason (MEM / EXEC / SYNC) and the producing instruction via *why / *who */
static int sim_ready(const or_sass *s, const uint8_t *opclass, const sim_warp *w, int64_t t, uint32_t *why, int32_t *who) {
  const uint32_t j = w->pc;
  int64_t worst = -1;
  int32_t p = -1;
  int t2, bar = 0;
  uint32_t b;
  for (b = 0; b < 6; ++b)
    if ((s->wait[j] >> b & 1u) && w->bclear[b] > t && w->bclear[b] > worst) { worst = w->bclear[b]; p = w->bprod[b]; bar = 1; }
  for (t2 = 0; t2 < 4; ++t2) {
    const uint16_t r = s->src[4u * j + t2];
    if (r == 0xFFFFu || r == 255u) continue;
    if (w->ready[r] > t && w->ready[r] > worst) { worst = w->ready[r]; p = w->prod[r]; bar = 0; }
  }
  if ((s->guard[j] & 7u) != 7u) {
    const uint32_t r = 256u + (s->guard[j] & 7u);
    if (w->ready[r] > t && w->ready[r] > worst) { worst = w->ready[r]; p = w->prod[r]; bar = 0; }
  }
  (void)bar;
  if (worst < 0) return 1;
  *who = p;
  *why = p < 0 ? R_EXEC : (opclass[p] == 9 ? R_SYNC : sim_is_mem(opclass[p]) ? R_MEM : R_EXEC);
  return 0;
}

int64_t or_simulate(const or_sass *s, const uint8_t *opclass, const uint32_t *latency, uint32_t func,
                    const or_simcfg *cfg, uint32_t sm, uint64_t cap, uint64_t *records, int32_t *truth) {
  const uint32_t S = cfg->schedulers, WP = cfg->warps_per_scheduler, W = S * WP;
  const uint32_t f0 = s->func_begin[func];
  uint32_t *blk_of = (uint32_t *)malloc(4u * s->n_instr);
  sim_warp *w = (sim_warp *)calloc(W, sizeof(sim_warp));
  uint32_t *rr = (uint32_t *)calloc(S, 4), *srr = (uint32_t *)calloc(S, 4);
  int32_t *issued = (int32_t *)malloc(4u * S);
  uint32_t b, k, live = W;
  uint64_t n_rec = 0;
  int64_t c, ret = -2;
  for (b = 0; b < s->n_blocks; ++b)
    for (k = s->block_begin[b]; k < s->block_begin[b + 1]; ++k) blk_of[k] = b;
  for (k = 0; k < W; ++k) {
    uint32_t r, q;
    w[k].pc = f0;
    w[k].last_issue = -1;
    for (r = 0; r < SIM_REGS; ++r) { w[k].ready[r] = 0; w[k].prod[r] = -1; }
    for (r = 0; r < 6; ++r) { w[k].bclear[r] = 0; w[k].bprod[r] = -1; }
    for (q = 0; q < 7; ++q)
      w[k].predv |= (uint32_t)(sim_mix(cfg->seed ^ ((uint64_t)(sm * W + k) << 8) ^ q) & 1u) << q;
  }
  for (c = 0; live > 0; ++c) {
    uint32_t sc;
    if (c >= (int64_t)cfg->max_cycles) goto out;
    /* ---- issue: per scheduler the first ready warp from its round-robin pointer */
    for (sc = 0; sc < S; ++sc) {
      uint32_t i;
      issued[sc] = -1;
      for (i = 0; i < WP; ++i) {
        const uint32_t lw = (rr[sc] + i) % WP, wi = lw * S + sc;   /* warp wi belongs to scheduler wi % S */
        sim_warp *x = &w[wi];
        uint32_t why;
        int32_t who;
        if (x->done || x->last_issue == c || !sim_ready(s, opclass, x, c, &why, &who)) continue;
        {
          const uint32_t j = x->pc;
          const uint32_t g = s->guard[j];
          const int on = (g & 7u) == 7u || ((((x->predv >> (g & 7u)) & 1u) != 0) != ((g & 8u) != 0));
          int t2;
          if (on) {
            for (t2 = 0; t2 < 4; ++t2) {
              const uint16_t d = s->dst[4u * j + t2];
              if (d == 0xFFFFu || d == 255u) continue;
              x->ready[d] = c + latency[j];
              x->prod[d] = (int32_t)j;
            }
            for (t2 = 0; t2 < 6; ++t2) {
              if (s->wbar[j] >> t2 & 1u) { x->bclear[t2] = c + latency[j]; x->bprod[t2] = (int32_t)j; }
              else if (s->rbar[j] >> t2 & 1u) { x->bclear[t2] = c + cfg->rbar_latency; x->bprod[t2] = (int32_t)j; }
            }
          }
          x->last_issue = c;
          x->last_pc = j;
          issued[sc] = (int32_t)wi;
          rr[sc] = (lw + 1u) % WP;
          /* advance the pc: next instruction, or the next block by the control policy */
          if (j + 1 < s->block_begin[blk_of[j] + 1]) {
            x->pc = j + 1;
          } else {
            const uint32_t bb = blk_of[j], e0 = s->succ_ptr[bb], e1 = s->succ_ptr[bb + 1];
            uint32_t e, self = 0, other = 0xFFFFFFFFu, n_other = 0, first_other = 0xFFFFFFFFu;
            for (e = e0; e < e1; ++e) {
              if (s->succ[e] == bb) self = 1;
              else { if (first_other == 0xFFFFFFFFu) first_other = s->succ[e]; ++n_other; }
            }
            if (self && x->loop_count + 1 < cfg->trip_count) {
              ++x->loop_count;
              other = bb;
            } else {
              x->loop_count = 0;
              if (n_other == 1 || (self && n_other >= 1)) other = first_other;
              else if (n_other >= 2) {
                uint32_t pick = wi % 2u, cnt = 0;
                for (e = e0; e < e1; ++e)
                  if (s->succ[e] != bb) { if (cnt == pick) { other = s->succ[e]; break; } ++cnt; }
              }
            }
            if (other == 0xFFFFFFFFu) { x->done = 1; --live; }
            else x->pc = s->block_begin[other];
          }
        }
        break;
      }
    }
    /* ---- sample at c = period, 2 period, ...: scheduler (c/period - 1) mod S, its warps in turn */
    if (c > 0 && c % cfg->period == 0) {
      const uint32_t sc2 = (uint32_t)((c / cfg->period - 1) % S);
      uint32_t i;
      for (i = 0; i < WP; ++i) {
        const uint32_t lw = (srr[sc2] + i) % WP, wi = lw * S + sc2;
        sim_warp *x = &w[wi];
        uint32_t why = 0, pc, reason, cls;
        int32_t who = -1;
        if (x->done && issued[sc2] != (int32_t)wi) continue;
        srr[sc2] = (lw + 1u) % WP;
        cls = issued[sc2] >= 0 ? 0u : 1u;
        if (issued[sc2] == (int32_t)wi) {          /* the issuing warp: its issued instruction */
          pc = x->last_pc;
          reason = R_NONE;
        } else {
          pc = x->pc;
          reason = sim_ready(s, opclass, x, c, &why, &who) ? R_NOTSEL : why;
        }
        if (n_rec >= cap) { ret = -1; goto out; }
        records[n_rec] = (uint64_t)pc | (1ull << 32) | ((uint64_t)reason << 48) | ((uint64_t)cls << 56);
        truth[n_rec] = (reason == R_MEM || reason == R_EXEC || reason == R_SYNC) ? who : -1;
        ++n_rec;
        break;
      }
    }
  }
  ret = (int64_t)n_rec;
out:
  free(blk_of); free(w); free(rr); free(srr); free(issued);
  return ret;
}

// slice.cu -- the step before the path: backward slicing of SASS fields into
// the def-use CSR that gpa_program_create takes (readings DESIGN.md §3.2 Q35-Q39).
//
// One thread per use instruction j (grid-stride), independent of all others.  For every register r j
// reads (source operands, its guard predicate, the virtual barrier registers of its wait mask) the
// thread explores the backward state graph of j's function -- states (instruction x about to be
// examined, P = predicates of the defs of r passed so far), P:310-320 -- and evaluates the
// definitions of DESIGN.md §3.2 Q36-Q38 (tests/slice_enum.py lists them path by path):
//   * min_len: breadth-first distances over the (x, P) pairs;
//   * K* and max_len: the pairs counting-sorted by descending address once, then "layers" L = 0, 1,
//     ... of back-edge crossings, two length arrays over the pair ids (layer L, layer L+1): inside
//     a layer every step goes to a lower address, so one descending sweep per layer settles its
//     longest lengths; the sweep stops after a layer that meets no new pair;
//   * rule 2: per def, candidates k ascending (unpredicated readers of every linking register met
//     by the search), each tested by a breadth-first search with k removed, on the pair table of
//     each linking register in turn (rebuilt only when the register changes).
// Each thread owns a slice of a scratch buffer (pair arrays, an open-addressing index, the layer
// arrays), so the work is an irregular per-thread graph walk with no communication.  Two launches:
// edge counts per use, then (after a host prefix sum) the edges.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "gpa_internal.cuh"

namespace gpa {
namespace {

constexpr uint32_t kSlNone = 0xFFFFu;
constexpr uint32_t kSlAll = 0x4000u;   // the '_' predicate
constexpr uint32_t kSlEmpty = 0xFFFFFFFFu;
constexpr uint32_t kSlMaxKids = 64;
constexpr uint32_t kSlThreads = 64;

struct SliceIn {
  uint32_t n, n_blocks;
  const uint32_t *block_begin, *blk_of, *pred_ptr, *pred, *func_begin, *func_of;
  const uint8_t *guard, *wbar, *rbar, *wait;
  const uint16_t *dst, *src;
};

struct SliceScratch {   // per-thread views into the scratch buffer
  uint32_t *x, *P, *dist, *hslot, *order, *cur, *nxt, *stamp, *queue, *cnt, *cand;
  uint32_t *hx, *hp, *hv;
  uint8_t *seen;
  uint32_t cap, hcap, n, gen, nfmax;
};

__device__ __forceinline__ uint32_t pbit(uint8_t g) {
  const uint32_t r = g & 7u;
  if (r == 7u) return kSlAll;
  return (g & 8u) ? (1u << (7u + r)) : (1u << r);
}
__device__ __forceinline__ uint32_t pnorm(uint32_t P) {
  for (uint32_t i = 0; i < 7; ++i)
    if (((P >> i) & 1u) && ((P >> (7 + i)) & 1u)) P |= kSlAll;
  return P;
}
__device__ __forceinline__ bool pcontains(uint32_t P, uint32_t b) { return (P & kSlAll) || (P & b); }

__device__ int reads_of(const SliceIn &s, uint32_t x, uint32_t *out, uint8_t *kinds) {
  int n = 0;
  for (int t = 0; t < 4; ++t) {
    const uint32_t r = s.src[4u * x + t];
    if (r == kSlNone || r == 255u) continue;
    out[n] = r;
    kinds[n] = r >= 256u ? 2u : 1u;
    ++n;
  }
  if ((s.guard[x] & 7u) != 7u) { out[n] = 256u + (s.guard[x] & 7u); kinds[n] = 2u; ++n; }
  for (int t = 0; t < 6; ++t)
    if ((s.wait[x] >> t) & 1u) { out[n] = 512u + t; kinds[n] = 4u; ++n; }
  return n;
}
__device__ __forceinline__ bool defines(const SliceIn &s, uint32_t x, uint32_t r) {
  if (r >= 512u) return (((s.wbar[x] | s.rbar[x]) >> (r - 512u)) & 1u) != 0;
  for (int t = 0; t < 4; ++t)
    if (s.dst[4u * x + t] == r) return true;
  return false;
}
__device__ bool reads_reg(const SliceIn &s, uint32_t x, uint32_t r) {
  uint32_t rr[16];
  uint8_t kk[16];
  const int n = reads_of(s, x, rr, kk);
  for (int t = 0; t < n; ++t)
    if (rr[t] == r) return true;
  return false;
}
__device__ int prev_of(const SliceIn &s, uint32_t x, uint32_t *out) {
  const uint32_t b = s.blk_of[x];
  if (x > s.block_begin[b]) { out[0] = x - 1; return 1; }
  int n = 0;
  for (uint32_t e = s.pred_ptr[b]; e < s.pred_ptr[b + 1] && n < (int)kSlMaxKids; ++e) out[n++] = s.block_begin[s.pred[e] + 1] - 1;
  return n;
}
__device__ __forceinline__ uint32_t out_mask(const SliceIn &s, uint32_t x, uint32_t P, uint32_t r, uint32_t pj, bool &term) {
  const bool d = defines(s, x, r);
  if (d) P = pnorm(P | pbit(s.guard[x]));
  term = d && pcontains(P, pj);
  return P;
}
__device__ __forceinline__ uint32_t hhash(const SliceScratch &g, uint32_t x, uint32_t P) {
  return (x * 2654435761u ^ (P + 1u) * 40503u) & (g.hcap - 1u);
}
__device__ uint32_t hfind(const SliceScratch &g, uint32_t x, uint32_t P) {
  uint32_t h = hhash(g, x, P);
  while (g.hv[h] != kSlEmpty) {
    if (g.hx[h] == x && g.hp[h] == P) return g.hv[h];
    h = (h + 1u) & (g.hcap - 1u);
  }
  return kSlEmpty;
}
__device__ uint32_t hinsert(SliceScratch &g, uint32_t x, uint32_t P) {
  uint32_t h = hhash(g, x, P);
  while (g.hv[h] != kSlEmpty) {
    if (g.hx[h] == x && g.hp[h] == P) return g.hv[h];
    h = (h + 1u) & (g.hcap - 1u);
  }
  g.hx[h] = x; g.hp[h] = P; g.hv[h] = g.n;
  g.x[g.n] = x; g.P[g.n] = P; g.hslot[g.n] = h;
  return g.n++;
}

struct RowAcc {
  uint32_t def, mn, kstar, mx;
  uint16_t regs;   // read indices of j linking the def
  uint8_t kind;
};

// breadth-first search from j over (x, P) for register r: the pair table (x, P, dist) and its index;
// false when the per-search budget is exceeded
__device__ bool build_pairs(const SliceIn &s, SliceScratch &g, uint32_t j, uint32_t r, uint32_t pj,
                            const uint32_t *roots, int nroot) {
  uint32_t kids[kSlMaxKids];
  bool stop;
  for (uint32_t i = 0; i < g.n; ++i) g.hv[g.hslot[i]] = kSlEmpty;
  g.n = 0;
  for (int q = 0; q < nroot; ++q)
    if (hfind(g, roots[q], 0u) == kSlEmpty) {
      const uint32_t id = hinsert(g, roots[q], 0u);
      g.dist[id] = 1u;
    }
  for (uint32_t u = 0; u < g.n; ++u) {    // pairs are appended in discovery order: the list is the queue
    const uint32_t Pout = out_mask(s, g.x[u], g.P[u], r, pj, stop);
    if (stop) continue;
    const int nk = prev_of(s, g.x[u], kids);
    for (int q = 0; q < nk; ++q)
      if (hfind(g, kids[q], Pout) == kSlEmpty) {
        if (g.n + 1u >= g.cap) return false;
        const uint32_t v = hinsert(g, kids[q], Pout);
        g.dist[v] = g.dist[u] + 1u;
      }
  }
  return true;
}

// with instruction k removed, does the search of the current pair table reach a state of def i?
__device__ bool reaches_without(const SliceIn &s, SliceScratch &g, uint32_t r, uint32_t pj, const uint32_t *roots,
                                int nroot, uint32_t k, uint32_t i) {
  uint32_t kids[kSlMaxKids];
  bool stop;
  const uint32_t gen = ++g.gen;
  uint32_t head = 0, tail = 0;
  for (int q = 0; q < nroot; ++q) {
    if (roots[q] == k) continue;
    const uint32_t c = hfind(g, roots[q], 0u);
    if (g.stamp[c] != gen) { g.stamp[c] = gen; g.queue[tail++] = c; }
  }
  while (head < tail) {
    const uint32_t u = g.queue[head++];
    if (g.x[u] == i) return true;
    const uint32_t Pout = out_mask(s, g.x[u], g.P[u], r, pj, stop);
    if (stop) continue;
    const int nk = prev_of(s, g.x[u], kids);
    for (int q = 0; q < nk; ++q) {
      if (kids[q] == k) continue;
      const uint32_t v = hfind(g, kids[q], Pout);
      if (g.stamp[v] != gen) { g.stamp[v] = gen; g.queue[tail++] = v; }
    }
  }
  return false;
}

// the edges of use j (function [f0, f1)), defs ascending, into out[] (when non-null); returns the
// count, or -1 when the per-search state budget or the row capacity is exceeded
__device__ int slice_row(const SliceIn &s, SliceScratch &g, RowAcc *acc, uint32_t acc_cap, uint32_t j, uint32_t f0,
                         uint32_t f1, uint32_t *o_def, uint8_t *o_kind, uint32_t *o_min, uint32_t *o_max,
                         int32_t *o_dom) {
  uint32_t reads[16];
  uint8_t kinds[16];
  const int nr = reads_of(s, j, reads, kinds);
  const uint32_t pj = pbit(s.guard[j]), nf = f1 - f0;
  uint32_t n_acc = 0;
  uint32_t roots[kSlMaxKids], kids[kSlMaxKids];
  const int nroot = prev_of(s, j, roots);
  bool stop;
  for (int ri = 0; ri < nr; ++ri) {
    const uint32_t r = reads[ri];
    if (!build_pairs(s, g, j, r, pj, roots, nroot)) return -1;
    // ---- the defs reached: kinds, minimum lengths
    for (uint32_t i = 0; i < g.n; ++i) {
      const uint32_t d = g.x[i];
      if (!defines(s, d, r)) continue;
      uint32_t a = 0;
      while (a < n_acc && acc[a].def != d) ++a;
      if (a == n_acc) {
        if (n_acc >= acc_cap) return -1;
        acc[a] = RowAcc{d, 0xFFFFFFFFu, 0xFFFFFFFFu, 0u, 0, 0};
        ++n_acc;
      }
      uint8_t kind = kinds[ri];
      if (r >= 512u && ((s.rbar[d] >> (r - 512u)) & 1u)) {   // WAR
        for (int tt = 0; tt < 4; ++tt)
          for (int uu = 0; uu < 4; ++uu) {
            const uint16_t w = s.dst[4u * j + tt];
            if (w != kSlNone && w != 255u && w == s.src[4u * d + uu]) kind |= 8u;
          }
      }
      acc[a].kind |= kind;
      acc[a].regs |= (uint16_t)(1u << ri);
      acc[a].mn = min(acc[a].mn, g.dist[i]);
    }
    // ---- pairs by descending address (counting sort over the function)
    for (uint32_t t = 0; t <= nf; ++t) g.cnt[t] = 0;
    for (uint32_t i = 0; i < g.n; ++i) ++g.cnt[f1 - 1u - g.x[i] + 1u];
    for (uint32_t t = 0; t < nf; ++t) g.cnt[t + 1] += g.cnt[t];
    for (uint32_t i = 0; i < g.n; ++i) g.order[g.cnt[f1 - 1u - g.x[i]]++] = i;
    // ---- layers of back-edge crossings: cur = layer L lengths, nxt = layer L+1 (0 = no state)
    for (uint32_t i = 0; i < g.n; ++i) { g.cur[i] = 0; g.nxt[i] = 0; g.seen[i] = 0; }
    for (int q = 0; q < nroot; ++q) {
      const uint32_t c = hfind(g, roots[q], 0u);
      if (roots[q] >= j) g.nxt[c] = 1u; else g.cur[c] = 1u;
    }
    for (uint32_t L = 0;; ++L) {
      bool any = false, fresh = false;
      for (uint32_t t = 0; t < g.n; ++t) {
        const uint32_t u = g.order[t], v = g.cur[u];
        if (!v) continue;
        any = true;
        if (!g.seen[u]) { g.seen[u] = 1; fresh = true; }
        const uint32_t x = g.x[u];
        if (defines(s, x, r)) {
          uint32_t a = 0;
          while (acc[a].def != x) ++a;
          if (L < acc[a].kstar) { acc[a].kstar = L; acc[a].mx = v; }
          else if (L == acc[a].kstar && v > acc[a].mx) acc[a].mx = v;
        }
        const uint32_t Pout = out_mask(s, x, g.P[u], r, pj, stop);
        if (stop) continue;
        const int nk = prev_of(s, x, kids);
        for (int q = 0; q < nk; ++q) {
          const uint32_t w = hfind(g, kids[q], Pout);
          uint32_t *lay = kids[q] >= x ? g.nxt : g.cur;   // a back edge starts layer L+1
          if (v + 1u > lay[w]) lay[w] = v + 1u;
        }
      }
      if (any ? !fresh : L > 0) break;   // layer 0 is empty only when every root is behind a back edge
      uint32_t *t = g.cur; g.cur = g.nxt; g.nxt = t;
      for (uint32_t i = 0; i < g.n; ++i) g.nxt[i] = 0;
    }
  }
  // ---- rule 2, per def: the smallest unpredicated k (not the def, not j) reading every
  //      linking register that every path of each of them passes
  for (uint32_t a = 0; a < n_acc; ++a) {
    const uint32_t i = acc[a].def, regs = acc[a].regs;
    const int r0 = __ffs(regs) - 1;
    if (!build_pairs(s, g, j, reads[r0], pj, roots, nroot)) return -1;
    int cur_reg = r0;
    for (uint32_t t = 0; t < nf; ++t) g.cnt[t] = 0;
    for (uint32_t u = 0; u < g.n; ++u) g.cnt[g.x[u] - f0] = 1;   // instructions the search meets
    uint32_t n_cand = 0;
    for (uint32_t k = f0; k < f1; ++k) {
      if (!g.cnt[k - f0] || k == j || k == i || (s.guard[k] & 7u) != 7u) continue;
      bool all = true;
      for (int ri = 0; ri < nr && all; ++ri)
        if ((regs >> ri) & 1u) all = reads_reg(s, k, reads[ri]);
      if (all) g.cand[n_cand++] = k;
    }
    int32_t dom = -1;
    for (uint32_t c = 0; c < n_cand && dom < 0; ++c) {
      const uint32_t k = g.cand[c];
      bool sep = true;
      for (int ri = 0; ri < nr && sep; ++ri) {
        if (!((regs >> ri) & 1u)) continue;
        if (cur_reg != ri) {
          if (!build_pairs(s, g, j, reads[ri], pj, roots, nroot)) return -1;
          cur_reg = ri;
        }
        sep = !reaches_without(s, g, reads[ri], pj, roots, nroot, k, i);
      }
      if (sep) dom = (int32_t)k;
    }
    acc[a].kstar = (uint32_t)dom;   // reused: the rule-2 result
  }
  for (uint32_t a = 1; a < n_acc; ++a)
    for (uint32_t b = a; b > 0 && acc[b - 1].def > acc[b].def; --b) {
      const RowAcc t = acc[b]; acc[b] = acc[b - 1]; acc[b - 1] = t;
    }
  if (o_def)
    for (uint32_t a = 0; a < n_acc; ++a) {
      o_def[a] = acc[a].def; o_kind[a] = acc[a].kind; o_min[a] = acc[a].mn; o_max[a] = acc[a].mx;
      o_dom[a] = (int32_t)acc[a].kstar;
    }
  return (int)n_acc;
}

// pass 1 (row_ptr == nullptr): counts[j]; pass 2: edges at row_ptr[j]
__global__ void __launch_bounds__(kSlThreads) k_slice(SliceIn s, uint8_t *scratch, size_t per_thread, uint32_t cap,
                                                      uint32_t hcap, uint32_t nfmax, uint32_t *counts,
                                                      const uint32_t *row_ptr, uint32_t *e_def, uint8_t *e_kind,
                                                      uint32_t *e_min, uint32_t *e_max, int32_t *e_dom, int *error) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint8_t *base = scratch + (size_t)tid * per_thread;
  SliceScratch g;
  uint32_t *w = reinterpret_cast<uint32_t *>(base);
  g.cap = cap;
  g.hcap = hcap;
  g.nfmax = nfmax;
  g.x = w; w += cap; g.P = w; w += cap; g.dist = w; w += cap; g.hslot = w; w += cap; g.order = w; w += cap;
  g.cur = w; w += cap; g.nxt = w; w += cap; g.stamp = w; w += cap; g.queue = w; w += cap;
  g.cnt = w; w += nfmax + 1; g.cand = w; w += nfmax;
  g.hx = w; w += hcap; g.hp = w; w += hcap; g.hv = w; w += hcap;
  RowAcc *acc = reinterpret_cast<RowAcc *>(w);
  g.seen = reinterpret_cast<uint8_t *>(acc + cap);
  for (uint32_t h = 0; h < hcap; ++h) g.hv[h] = kSlEmpty;
  for (uint32_t i = 0; i < cap; ++i) g.stamp[i] = 0;
  g.n = 0;
  g.gen = 0;
  for (uint32_t j = tid; j < s.n; j += gridDim.x * blockDim.x) {
    const uint32_t f = s.func_of[j], f0 = s.func_begin[f], f1 = s.func_begin[f + 1];
    int c;
    if (!row_ptr) {
      c = slice_row(s, g, acc, cap, j, f0, f1, nullptr, nullptr, nullptr, nullptr, nullptr);
      if (c >= 0) counts[j] = (uint32_t)c;
    } else {
      const uint32_t o = row_ptr[j];
      c = slice_row(s, g, acc, cap, j, f0, f1, e_def + o, e_kind + o, e_min + o, e_max + o, e_dom + o);
      if (c >= 0 && (uint32_t)c != row_ptr[j + 1] - o) c = -1;
    }
    if (c < 0) atomicExch(error, 1);
  }
}

}  // namespace

size_t slice_scratch_per_thread(uint32_t cap, uint32_t hcap, uint32_t nfmax) {
  return (size_t)cap * (9 * 4 + sizeof(RowAcc) + 1) + (size_t)hcap * 12 + ((size_t)nfmax * 2 + 1) * 4 + 64;
}

cudaError_t launch_slice(const gpa_sass_desc *h, uint32_t *h_row_ptr, uint64_t cap_edges, uint32_t *h_def,
                         uint8_t *h_kind, uint32_t *h_min, uint32_t *h_max, int32_t *h_dom, uint64_t *n_edges,
                         int n_sms, cudaStream_t st, int *status) {
  const uint32_t n = h->n_instr, NB = h->n_blocks;
  *status = 0;
  // host-side CFG helpers: block of each instruction, predecessor CSR (ascending source block)
  std::vector<uint32_t> blk_of(std::max<uint32_t>(n, 1)), pred_ptr(NB + 1, 0), pred(std::max<uint32_t>(h->succ_ptr[NB], 1));
  for (uint32_t b = 0; b < NB; ++b)
    for (uint32_t j = h->block_begin[b]; j < h->block_begin[b + 1]; ++j) blk_of[j] = b;
  for (uint32_t b = 0; b < NB; ++b)
    for (uint32_t e = h->succ_ptr[b]; e < h->succ_ptr[b + 1]; ++e) pred_ptr[h->succ[e] + 1]++;
  for (uint32_t b = 0; b < NB; ++b) pred_ptr[b + 1] += pred_ptr[b];
  {
    std::vector<uint32_t> fill(NB, 0);
    for (uint32_t b = 0; b < NB; ++b)
      for (uint32_t e = h->succ_ptr[b]; e < h->succ_ptr[b + 1]; ++e) {
        const uint32_t t = h->succ[e];
        pred[pred_ptr[t] + fill[t]++] = b;
      }
  }
  uint32_t maxf = 1;
  for (uint32_t f = 0; f < h->n_funcs; ++f) maxf = std::max(maxf, h->func_begin[f + 1] - h->func_begin[f]);
  const uint32_t cap = 4u * maxf + 256u;   // (x, P) pairs per search (Q39)
  uint32_t hcap = 1;
  while (hcap < 2u * cap) hcap <<= 1;
  const size_t per_thread = (slice_scratch_per_thread(cap, hcap, maxf) + 255) & ~(size_t)255;
  std::vector<uint32_t> func_of(std::max<uint32_t>(n, 1));
  for (uint32_t f = 0; f < h->n_funcs; ++f)
    for (uint32_t j = h->func_begin[f]; j < h->func_begin[f + 1]; ++j) func_of[j] = f;
  // device copies (every allocation is released on every path)
  std::vector<void *> owned;
  cudaError_t e = cudaSuccess;
  auto alloc = [&](size_t bytes) -> void * {
    void *d = nullptr;
    if (e == cudaSuccess) e = cudaMallocAsync(&d, std::max<size_t>(bytes, 16), st);
    if (d) owned.push_back(d);
    return d;
  };
  auto up = [&](const void *src, size_t bytes) -> void * {
    void *d = alloc(bytes);
    if (e == cudaSuccess && bytes) e = cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, st);
    return d;
  };
  SliceIn s{n, NB, (const uint32_t *)up(h->block_begin, (NB + 1) * 4), (const uint32_t *)up(blk_of.data(), (size_t)n * 4),
            (const uint32_t *)up(pred_ptr.data(), (NB + 1) * 4), (const uint32_t *)up(pred.data(), (size_t)pred_ptr[NB] * 4),
            (const uint32_t *)up(h->func_begin, (size_t)(h->n_funcs + 1) * 4), (const uint32_t *)up(func_of.data(), (size_t)n * 4),
            (const uint8_t *)up(h->guard, n), (const uint8_t *)up(h->wbar, n), (const uint8_t *)up(h->rbar, n),
            (const uint8_t *)up(h->wait, n), (const uint16_t *)up(h->dst, (size_t)n * 8),
            (const uint16_t *)up(h->src, (size_t)n * 8)};
  // threads: one per use up to what the GPU holds, bounded by the scratch budget (a quarter of the
  // free device memory, at most GPA_SLICE_SCRATCH_MB, default 4 GB: measured best of 1-16 GB, the
  // mapping of a larger pool allocation costs more than the extra concurrency saves)
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = 2ull << 30;
  uint64_t budget = std::min<uint64_t>(free_b / 4, 4ull << 30);
  if (const char *env = getenv("GPA_SLICE_SCRATCH_MB")) budget = std::min<uint64_t>(budget, strtoull(env, nullptr, 10) << 20);
  budget = std::max<uint64_t>(budget, 64ull << 20);
  uint64_t threads = std::min<uint64_t>((uint64_t)std::max(n_sms, 1) * 8 * kSlThreads, ((uint64_t)n + kSlThreads - 1) / kSlThreads * kSlThreads);
  threads = std::min<uint64_t>(threads, std::max<uint64_t>(kSlThreads, (budget / per_thread) / kSlThreads * kSlThreads));
  threads = std::max<uint64_t>(threads, kSlThreads);
  void *d_scr = alloc(threads * per_thread), *d_cnt = alloc((size_t)std::max<uint32_t>(n, 1) * 4), *d_err = alloc(4);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_err, 0, 4, st);
  const uint32_t grid = (uint32_t)(threads / kSlThreads);
  std::vector<uint32_t> cnt(std::max<uint32_t>(n, 1));
  int err = 0;
  if (e == cudaSuccess) {
    k_slice<<<grid, kSlThreads, 0, st>>>(s, (uint8_t *)d_scr, per_thread, cap, hcap, maxf, (uint32_t *)d_cnt, nullptr, nullptr,
                                         nullptr, nullptr, nullptr, nullptr, (int *)d_err);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(cnt.data(), d_cnt, (size_t)n * 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&err, d_err, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  uint64_t E = 0;
  if (e == cudaSuccess) {
    h_row_ptr[0] = 0;
    for (uint32_t j = 0; j < n; ++j) {
      E += cnt[j];
      h_row_ptr[j + 1] = (uint32_t)E;
    }
    *n_edges = E;
    if (err) *status = 1;                    // state budget exceeded
    else if (E > cap_edges) *status = 2;     // caller's edge arrays too small
  }
  if (e == cudaSuccess && !*status && E) {
    void *d_rp = up(h_row_ptr, ((size_t)n + 1) * 4);
    void *d_def = alloc(E * 4), *d_kind = alloc(E), *d_min = alloc(E * 4), *d_max = alloc(E * 4), *d_dom = alloc(E * 4);
    if (e == cudaSuccess) {
      k_slice<<<grid, kSlThreads, 0, st>>>(s, (uint8_t *)d_scr, per_thread, cap, hcap, maxf, (uint32_t *)d_cnt,
                                           (const uint32_t *)d_rp, (uint32_t *)d_def, (uint8_t *)d_kind, (uint32_t *)d_min,
                                           (uint32_t *)d_max, (int32_t *)d_dom, (int *)d_err);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_def, d_def, E * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_kind, d_kind, E, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_min, d_min, E * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_max, d_max, E * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_dom, d_dom, E * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&err, d_err, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess && err) *status = 1;
  }
  for (void *ptr : owned) cudaFreeAsync(ptr, st);
  const cudaError_t e2 = cudaStreamSynchronize(st);
  return e != cudaSuccess ? e : e2;
}

}  // namespace gpa

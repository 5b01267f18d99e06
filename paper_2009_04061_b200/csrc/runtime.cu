// runtime.cu -- host side of the C ABI (include/gpa.h): validation, create-time transposes and
// permutations, workspace layout, call-order state, launch sequencing, host-ingest staging.
// Every hot-path step runs in the sm_100a kernels of ingest.cu / blame.cu / rollup.cu /
// estimate.cu (fused.cu: the same bodies as one cooperative kernel); nothing here computes blame.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "gpa_internal.cuh"

using namespace gpa;

namespace {

thread_local char g_err[512] = "";

gpa_status fail(gpa_status st, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}

gpa_status cuda_fail(cudaError_t e, const char *where) {
  return fail(GPA_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CUDA_TRY(expr)                                   \
  do {                                                   \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr);  \
  } while (0)

// ------------------------------------------------------------------------------ validation
gpa_status validate(const gpa_program_desc *d, std::vector<int32_t> *loop_func_out) {
  if (!d) return fail(GPA_ERR_INVALID_ARGUMENT, "desc is NULL");
  const uint32_t n = d->n_instr;
  if (n == 0) return fail(GPA_ERR_INVALID_PROGRAM, "n_instr must be >= 1");
  if (d->n_reasons < 4 || d->n_reasons > (uint32_t)kReasonsMax)
    return fail(GPA_ERR_INVALID_PROGRAM, "n_reasons %u not in [4, 16]", d->n_reasons);
  if (d->n_funcs == 0 || d->n_kernels == 0 || d->n_lines == 0)
    return fail(GPA_ERR_INVALID_PROGRAM, "n_funcs, n_kernels and n_lines must be >= 1");
  if (!d->opclass || !d->iflags || !d->latency || !d->line_id || !d->loop_id || !d->func_begin ||
      !d->kernel_func_begin || !d->row_ptr)
    return fail(GPA_ERR_INVALID_ARGUMENT, "a required desc array is NULL");
  if (d->n_loops && !d->loop_parent) return fail(GPA_ERR_INVALID_ARGUMENT, "loop_parent is NULL");
  const uint32_t E = d->row_ptr[n];
  if (E && (!d->edge_def || !d->edge_kind || !d->edge_min_len || !d->edge_max_len || !d->edge_dom_k))
    return fail(GPA_ERR_INVALID_ARGUMENT, "an edge array is NULL");
  for (uint32_t i = 0; i < n; ++i) {
    if (d->opclass[i] >= OC_COUNT) return fail(GPA_ERR_INVALID_PROGRAM, "opclass[%u] = %u >= 11", i, d->opclass[i]);
    if (d->line_id[i] >= d->n_lines) return fail(GPA_ERR_INVALID_PROGRAM, "line_id[%u] out of range", i);
    if (d->loop_id[i] < -1 || d->loop_id[i] >= (int32_t)d->n_loops)
      return fail(GPA_ERR_INVALID_PROGRAM, "loop_id[%u] out of range", i);
  }
  // functions and kernels: contiguous, strictly increasing, covering
  if (d->func_begin[0] != 0 || d->func_begin[d->n_funcs] != n)
    return fail(GPA_ERR_INVALID_PROGRAM, "func_begin must start at 0 and end at n_instr");
  for (uint32_t f = 0; f < d->n_funcs; ++f)
    if (d->func_begin[f + 1] <= d->func_begin[f])
      return fail(GPA_ERR_INVALID_PROGRAM, "function %u is empty or ranges are not increasing", f);
  if (d->kernel_func_begin[0] != 0 || d->kernel_func_begin[d->n_kernels] != d->n_funcs)
    return fail(GPA_ERR_INVALID_PROGRAM, "kernel_func_begin must start at 0 and end at n_funcs");
  for (uint32_t k = 0; k < d->n_kernels; ++k)
    if (d->kernel_func_begin[k + 1] <= d->kernel_func_begin[k])
      return fail(GPA_ERR_INVALID_PROGRAM, "kernel %u has no function", k);
  // loop forest acyclic
  for (uint32_t l = 0; l < d->n_loops; ++l) {
    int32_t x = (int32_t)l;
    uint32_t steps = 0;
    while (x >= 0) {
      if (x >= (int32_t)d->n_loops) return fail(GPA_ERR_INVALID_PROGRAM, "loop_parent[%d] out of range", x);
      x = d->loop_parent[x];
      if (++steps > d->n_loops) return fail(GPA_ERR_INVALID_PROGRAM, "loop forest has a cycle through loop %u", l);
    }
  }
  // func of each instruction; loops inside one function (P:289 intra-function structure)
  std::vector<uint32_t> func_of(n);
  for (uint32_t f = 0; f < d->n_funcs; ++f)
    for (uint32_t i = d->func_begin[f]; i < d->func_begin[f + 1]; ++i) func_of[i] = f;
  std::vector<int32_t> loop_func(d->n_loops, -1);
  for (uint32_t i = 0; i < n; ++i)
    for (int32_t x = d->loop_id[i]; x >= 0; x = d->loop_parent[x]) {
      if (loop_func[x] < 0) loop_func[x] = (int32_t)func_of[i];
      else if (loop_func[x] != (int32_t)func_of[i])
        return fail(GPA_ERR_INVALID_PROGRAM, "loop %d spans functions %d and %u", x, loop_func[x], func_of[i]);
    }
  // CSR
  if (d->row_ptr[0] != 0) return fail(GPA_ERR_INVALID_PROGRAM, "row_ptr[0] != 0");
  std::vector<uint32_t> last_row(n, 0xffffffffu);
  for (uint32_t j = 0; j < n; ++j) {
    if (d->row_ptr[j + 1] < d->row_ptr[j]) return fail(GPA_ERR_INVALID_PROGRAM, "row_ptr not monotone at %u", j);
    for (uint32_t e = d->row_ptr[j]; e < d->row_ptr[j + 1]; ++e) {
      uint32_t i = d->edge_def[e];
      if (i >= n) return fail(GPA_ERR_INVALID_PROGRAM, "edge %u: def %u >= n_instr", e, i);
      if (func_of[i] != func_of[j])
        return fail(GPA_ERR_INVALID_PROGRAM, "edge %u: def %u and use %u in different functions (P:289)", e, i, j);
      if (last_row[i] == j) return fail(GPA_ERR_INVALID_PROGRAM, "duplicate edge (%u -> %u) (Q10)", i, j);
      last_row[i] = j;
      if (d->edge_kind[e] == 0 || d->edge_kind[e] > 15) return fail(GPA_ERR_INVALID_PROGRAM, "edge %u: bad kind", e);
      if (d->edge_min_len[e] < 1 || d->edge_max_len[e] < d->edge_min_len[e])
        return fail(GPA_ERR_INVALID_PROGRAM, "edge %u: need 1 <= min_len <= max_len", e);
      if (d->edge_dom_k[e] < -1 || d->edge_dom_k[e] >= (int32_t)n)
        return fail(GPA_ERR_INVALID_PROGRAM, "edge %u: dom_k out of range", e);
    }
  }
  if (loop_func_out) *loop_func_out = std::move(loop_func);
  return GPA_OK;
}

// ------------------------------------------------------------------------------ layout
struct Layout {
  size_t off = 0;
  size_t take(size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  }
};

constexpr uint32_t kPatWs = 16;   // patterns the workspace is sized for
constexpr uint32_t kLoopPatWs = 4;// of which may use loop scopes (models 2 and 4)

struct HostPlan {
  // create-time arrays (host)
  std::vector<uint32_t> edge_use, def_ptr, def_perm;
  std::vector<int32_t> edge_lca, loop_func;
  std::vector<uint32_t> tile_run_ptr, run_be, run_dst, seg1_perm, seg1_begin, seg1_end, seg1_id, seg2_perm,
      seg2_begin, seg2_end;
  uint32_t n_partials = 0;
  std::vector<uint32_t> loop_items, loop_item_ptr, pre_perm, pre_begin, pre_end, kloop_ptr, kloops;
  uint32_t n_rows = 0;
};

gpa_status build_plan(const gpa_program_desc *d, HostPlan &h) {
  const uint32_t n = d->n_instr, E = d->row_ptr[n], L = d->n_loops;
  std::vector<int32_t> lf;
  gpa_status st = validate(d, &lf);
  if (st != GPA_OK) return st;
  h.loop_func = lf;
  // edge -> use; def-major stable transpose
  h.edge_use.resize(E);
  for (uint32_t j = 0; j < n; ++j)
    for (uint32_t e = d->row_ptr[j]; e < d->row_ptr[j + 1]; ++e) h.edge_use[e] = j;
  h.def_ptr.assign(n + 1, 0);
  for (uint32_t e = 0; e < E; ++e) h.def_ptr[d->edge_def[e] + 1]++;
  for (uint32_t i = 0; i < n; ++i) h.def_ptr[i + 1] += h.def_ptr[i];
  h.def_perm.resize(E);
  {
    std::vector<uint32_t> cur(h.def_ptr.begin(), h.def_ptr.end() - 1);
    for (uint32_t e = 0; e < E; ++e) h.def_perm[cur[d->edge_def[e]]++] = e;
  }
  // loop depths and lca per edge
  std::vector<int32_t> depth(L, -1);
  for (uint32_t l = 0; l < L; ++l) {
    int32_t dd = 0;
    for (int32_t x = d->loop_parent[l]; x >= 0; x = d->loop_parent[x]) ++dd;
    depth[l] = dd;
  }
  auto lca = [&](int32_t a, int32_t b) -> int32_t {
    if (a < 0 || b < 0) return -1;
    while (depth[a] > depth[b]) a = d->loop_parent[a];
    while (depth[b] > depth[a]) b = d->loop_parent[b];
    while (a != b) {
      a = d->loop_parent[a];
      b = d->loop_parent[b];
      if (a < 0 || b < 0) return -1;
    }
    return a;
  };
  h.edge_lca.resize(E);
  for (uint32_t e = 0; e < E; ++e) h.edge_lca[e] = lca(d->loop_id[d->edge_def[e]], d->loop_id[h.edge_use[e]]);

  // ---- rollup runs: tiles of 32 instructions; per tile the maximal runs of equal line, equal
  //      innermost loop (loop members) and equal function, in program order (segment ids: lines,
  //      then loops, then functions -- the stage-1 row order)
  const uint32_t n_seg1 = d->n_lines + L + d->n_funcs;
  {
    const uint32_t n_tiles = (n + 31) / 32;
    std::vector<uint32_t> func_of(n);
    for (uint32_t f = 0; f < d->n_funcs; ++f)
      for (uint32_t i = d->func_begin[f]; i < d->func_begin[f + 1]; ++i) func_of[i] = f;
    auto seg_of = [&](int kind, uint32_t i) -> int64_t {
      if (kind == 0) return d->line_id[i];
      if (kind == 1) return d->loop_id[i] >= 0 ? (int64_t)d->n_lines + d->loop_id[i] : -1;
      return (int64_t)d->n_lines + L + func_of[i];
    };
    std::vector<uint32_t> run_seg;
    std::vector<uint32_t> runs_of(n_seg1, 0);
    h.tile_run_ptr.assign(n_tiles + 1, 0);
    for (uint32_t t = 0; t < n_tiles; ++t) {
      const uint32_t i0 = 32 * t, i1 = std::min(n, i0 + 32);
      for (int kind = 0; kind < 3; ++kind)
        for (uint32_t i = i0; i < i1;) {
          const int64_t sg = seg_of(kind, i);
          uint32_t k = i + 1;
          while (k < i1 && seg_of(kind, k) == sg) ++k;
          if (sg >= 0) {
            h.run_be.push_back((i - i0) | ((k - i0) << 8));
            run_seg.push_back((uint32_t)sg);
            runs_of[sg]++;
          }
          i = k;
        }
      h.tile_run_ptr[t + 1] = (uint32_t)h.run_be.size();
    }
    // destinations: a segment's only run writes its row; runs of multi-run segments write partials
    std::vector<std::vector<uint32_t>> parts(n_seg1);
    h.run_dst.resize(run_seg.size());
    for (size_t r = 0; r < run_seg.size(); ++r) {
      const uint32_t sg = run_seg[r];
      if (runs_of[sg] == 1) {
        h.run_dst[r] = sg;
      } else {
        parts[sg].push_back(h.n_partials);
        h.run_dst[r] = kPartialBit | h.n_partials++;
      }
    }
    for (uint32_t sg = 0; sg < n_seg1; ++sg) {
      if (runs_of[sg] == 1) continue;       // 0 runs (an all-nested loop): stage 1 writes zeros
      h.seg1_id.push_back(sg);
      h.seg1_begin.push_back((uint32_t)h.seg1_perm.size());
      h.seg1_perm.insert(h.seg1_perm.end(), parts[sg].begin(), parts[sg].end());
      h.seg1_end.push_back((uint32_t)h.seg1_perm.size());
    }
  }
  // ---- loop preorder (children visited in increasing id), subtree ranges
  std::vector<std::vector<uint32_t>> kids(L);
  std::vector<uint32_t> roots;
  for (uint32_t l = 0; l < L; ++l) {
    if (d->loop_parent[l] < 0) roots.push_back(l);
    else kids[d->loop_parent[l]].push_back(l);
  }
  h.pre_perm.clear();
  h.pre_begin.assign(L, 0);
  h.pre_end.assign(L, 0);
  {
    std::vector<std::pair<uint32_t, bool>> stack;
    for (auto it = roots.rbegin(); it != roots.rend(); ++it) stack.push_back({*it, false});
    while (!stack.empty()) {
      auto [l, done] = stack.back();
      stack.pop_back();
      if (done) {
        h.pre_end[l] = (uint32_t)h.pre_perm.size();
        continue;
      }
      h.pre_begin[l] = (uint32_t)h.pre_perm.size();
      h.pre_perm.push_back(l);
      stack.push_back({l, true});
      for (auto it = kids[l].rbegin(); it != kids[l].rend(); ++it) stack.push_back({*it, false});
    }
  }
  // ---- stage 2: loops inclusive (over loop-excl rows in preorder), kernels (over function rows)
  for (uint32_t p = 0; p < L; ++p) h.seg2_perm.push_back(d->n_lines + h.pre_perm[p]);
  for (uint32_t f = 0; f < d->n_funcs; ++f) h.seg2_perm.push_back(d->n_lines + L + f);
  for (uint32_t l = 0; l < L; ++l) {
    h.seg2_begin.push_back(h.pre_begin[l]);
    h.seg2_end.push_back(h.pre_end[l]);
  }
  for (uint32_t k = 0; k < d->n_kernels; ++k) {
    h.seg2_begin.push_back(L + d->kernel_func_begin[k]);
    h.seg2_end.push_back(L + d->kernel_func_begin[k + 1]);
  }
  h.n_rows = n_seg1 + L + d->n_kernels;
  // ---- estimate: loop-scoped items (edges by lca, in-loop instructions by loop), kernel -> loops
  h.loop_item_ptr.assign(L + 1, 0);
  for (uint32_t e = 0; e < E; ++e)
    if (h.edge_lca[e] >= 0) h.loop_item_ptr[h.edge_lca[e] + 1]++;
  for (uint32_t i = 0; i < n; ++i)
    if (d->loop_id[i] >= 0) h.loop_item_ptr[d->loop_id[i] + 1]++;
  for (uint32_t l = 0; l < L; ++l) h.loop_item_ptr[l + 1] += h.loop_item_ptr[l];
  h.loop_items.resize(h.loop_item_ptr[L]);
  {
    std::vector<uint32_t> cur(h.loop_item_ptr.begin(), h.loop_item_ptr.end() - 1);
    for (uint32_t e = 0; e < E; ++e)
      if (h.edge_lca[e] >= 0) h.loop_items[cur[h.edge_lca[e]]++] = e;
    for (uint32_t i = 0; i < n; ++i)
      if (d->loop_id[i] >= 0) h.loop_items[cur[d->loop_id[i]]++] = E + i;
  }
  std::vector<uint32_t> kernel_of_func(d->n_funcs);
  for (uint32_t k = 0; k < d->n_kernels; ++k)
    for (uint32_t f = d->kernel_func_begin[k]; f < d->kernel_func_begin[k + 1]; ++f) kernel_of_func[f] = k;
  h.kloop_ptr.assign(d->n_kernels + 1, 0);
  for (uint32_t l = 0; l < L; ++l)
    if (h.loop_func[l] >= 0) h.kloop_ptr[kernel_of_func[h.loop_func[l]] + 1]++;
  for (uint32_t k = 0; k < d->n_kernels; ++k) h.kloop_ptr[k + 1] += h.kloop_ptr[k];
  h.kloops.resize(h.kloop_ptr[d->n_kernels]);
  {
    std::vector<uint32_t> cur(h.kloop_ptr.begin(), h.kloop_ptr.end() - 1);
    for (uint32_t l = 0; l < L; ++l)
      if (h.loop_func[l] >= 0) h.kloops[cur[kernel_of_func[h.loop_func[l]]]++] = l;
  }
  return GPA_OK;
}

struct Offsets {
  size_t dinfo, opclass, iflags, latency, line_id, loop_id, func_begin, kfb, kgb, row_ptr, edge_def, edge_min,
      edge_max, edge_use, edge_dom, edge_lca, edge_kind, def_ptr, def_perm;
  size_t tile_run_ptr, run_be, run_dst, seg1_perm, seg1_begin, seg1_end, seg1_id, seg2_perm, seg2_begin, seg2_end,
      part_v, part_al, rows_v, rows_al;
  size_t pats, mval, mrow, loop_items, loop_item_ptr, pre_perm, pre_begin, pre_end, kloop_ptr, kloops,
      loop_func, lM_excl, lM_incl, fM, kM, est, hot, n_hot, rank, cov, occ;
  size_t C, stats, AL, cand, selfm, share, B, partials, part_x, part_sync, part_zero;
  bool part_reserved = false;
  size_t total;
};

Offsets layout(const gpa_program_desc *d, const HostPlan &h) {
  const size_t n = d->n_instr, E = d->row_ptr[d->n_instr], L = d->n_loops, nf = d->n_funcs,
               nk = d->n_kernels, R = d->n_reasons, ncol = R + 6;
  Layout a;
  Offsets o;
  // outputs first (large, hot)
  // the count table and the stats are one contiguous block, so a multi-GPU step sums both with
  // a single collective (Program.reduce_view)
  o.C = a.take(n * 2 * R * 8 + 4 * 8);
  o.stats = o.C + n * 2 * R * 8;
  o.AL = a.take(n * 2 * 8);
  o.cand = a.take(E);
  o.selfm = a.take(n);
  o.share = a.take(E * 3 * 8);
  o.B = a.take(n * 8 * 8);
  o.partials = (n * 2 * R * 4 <= kSmemTableMax) ? a.take((size_t)kMaxIngestCtas * n * 2 * R * 4) : a.take(0);
  {
    const bool part = n * 2 * R * 4 > kSmemTableMax && n * 2 * R < ((size_t)kPartMaxCtas << 15);  // see part_feasible (15-bit local bins)
    const size_t pairs = (size_t)kPartBufs * kPartMaxCtas * kPartMaxCtas;
    o.part_x = a.take(part ? pairs * kPartCap * 2 : 0);   // 2-byte keys
    o.part_sync = a.take(part ? 2 * kPartBufs * 4 : 0);   // producer + consumer counters per buffer
    o.part_zero = a.take(part ? kPartZeroBytes : 0);       // zeros: source of the staging-buffer clears
    o.part_reserved = part;
  }
  o.dinfo = a.take(n * sizeof(DefInfo));
  o.opclass = a.take(n);
  o.iflags = a.take(n);
  o.latency = a.take(n * 4);
  o.line_id = a.take(n * 4);
  o.loop_id = a.take(n * 4);
  o.func_begin = a.take((nf + 1) * 4);
  o.kfb = a.take((nk + 1) * 4);
  o.kgb = a.take(nk * 4);
  o.row_ptr = a.take((n + 1) * 4);
  o.edge_def = a.take(E * 4);
  o.edge_min = a.take(E * 4);
  o.edge_max = a.take(E * 4);
  o.edge_use = a.take(E * 4);
  o.edge_dom = a.take(E * 4);
  o.edge_lca = a.take(E * 4);
  o.edge_kind = a.take(E);
  o.def_ptr = a.take((n + 1) * 4);
  o.def_perm = a.take(E * 4);
  o.tile_run_ptr = a.take(h.tile_run_ptr.size() * 4);
  o.run_be = a.take(h.run_be.size() * 4);
  o.run_dst = a.take(h.run_dst.size() * 4);
  o.seg1_perm = a.take(h.seg1_perm.size() * 4);
  o.seg1_begin = a.take(h.seg1_begin.size() * 4);
  o.seg1_end = a.take(h.seg1_end.size() * 4);
  o.seg1_id = a.take(h.seg1_id.size() * 4);
  o.seg2_perm = a.take(h.seg2_perm.size() * 4);
  o.seg2_begin = a.take(h.seg2_begin.size() * 4);
  o.seg2_end = a.take(h.seg2_end.size() * 4);
  o.part_v = a.take((size_t)h.n_partials * 2 * ncol * 8);
  o.part_al = a.take((size_t)h.n_partials * 2 * 8);
  o.rows_v = a.take((size_t)h.n_rows * 2 * ncol * 8);
  o.rows_al = a.take((size_t)h.n_rows * 2 * 8);
  o.pats = a.take(kPatWs * sizeof(gpa_pattern));
  o.mval = a.take((size_t)kLoopPatWs * (E + n) * 8);
  o.mrow = a.take((size_t)kPatWs * n * 8);
  o.loop_items = a.take(h.loop_items.size() * 4);
  o.loop_item_ptr = a.take((L + 1) * 4);
  o.pre_perm = a.take(L * 4);
  o.pre_begin = a.take(L * 4);
  o.pre_end = a.take(L * 4);
  o.kloop_ptr = a.take((nk + 1) * 4);
  o.kloops = a.take(L * 4);
  o.loop_func = a.take(L * 4);
  o.lM_excl = a.take(kPatWs * L * 8);
  o.lM_incl = a.take(kPatWs * L * 8);
  o.fM = a.take(kPatWs * nf * 8);
  o.kM = a.take(kPatWs * nk * 8);
  o.est = a.take(kPatWs * nk * sizeof(gpa_estimate_out));
  o.hot = a.take((size_t)kPatWs * nk * kTopKMax * sizeof(gpa_hotspot));
  o.n_hot = a.take((size_t)kPatWs * nk * 4);
  o.rank = a.take((size_t)kPatWs * nk * 4);
  o.cov = a.take((size_t)nk * sizeof(gpa_coverage));
  o.occ = a.take((size_t)nk * sizeof(KernOcc));
  o.total = a.off;
  return o;
}

template <typename T>
gpa_status upload(uint8_t *ws, size_t off, const T *src, size_t count, cudaStream_t s) {
  if (count == 0) return GPA_OK;
  CUDA_TRY(cudaMemcpyAsync(ws + off, src, count * sizeof(T), cudaMemcpyHostToDevice, s));
  return GPA_OK;
}

#define UP(off, ptr, cnt)                                                 \
  do {                                                                    \
    gpa_status _s = upload(ws, (off), (ptr), (size_t)(cnt), s);           \
    if (_s != GPA_OK) return _s;                                          \
  } while (0)

gpa_status check_prog(gpa_program *p) {
  if (!p) return fail(GPA_ERR_INVALID_ARGUMENT, "program is NULL");
  return GPA_OK;
}

}  // namespace

extern "C" {

const char *gpa_last_error(void) { return g_err; }
const char *gpa_version(void) { return "gpa-b200 0.1 (sm_100a)"; }

gpa_status gpa_validate_program(const gpa_program_desc *desc) { return validate(desc, nullptr); }

gpa_status gpa_workspace_size(const gpa_program_desc *desc, size_t *bytes) {
  if (!bytes) return fail(GPA_ERR_INVALID_ARGUMENT, "bytes is NULL");
  HostPlan h;
  gpa_status st = build_plan(desc, h);
  if (st != GPA_OK) return st;
  *bytes = layout(desc, h).total;
  return GPA_OK;
}

gpa_status gpa_program_create(const gpa_program_desc *d, void *d_workspace, size_t bytes,
                              void *stream, gpa_program **out) {
  if (!out || !d_workspace) return fail(GPA_ERR_INVALID_ARGUMENT, "out / workspace is NULL");
  *out = nullptr;
  if (((uintptr_t)d_workspace & 255u) != 0) return fail(GPA_ERR_WORKSPACE, "workspace not 256-byte aligned");
  HostPlan h;
  gpa_status st = build_plan(d, h);
  if (st != GPA_OK) return st;
  Offsets o = layout(d, h);
  if (bytes < o.total) return fail(GPA_ERR_WORKSPACE, "workspace %zu bytes < required %zu", bytes, o.total);
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t *ws = (uint8_t *)d_workspace;
  const uint32_t n = d->n_instr, E = d->row_ptr[n];
  {
    std::vector<DefInfo> di(n);
    for (uint32_t i = 0; i < n; ++i)
      di[i] = DefInfo{d->latency[i], d->loop_id[i], (uint32_t)d->opclass[i] | (uint32_t)d->iflags[i] << 8, 0u};
    UP(o.dinfo, di.data(), n);
  }
  UP(o.opclass, d->opclass, n);
  UP(o.iflags, d->iflags, n);
  UP(o.latency, d->latency, n);
  UP(o.line_id, d->line_id, n);
  UP(o.loop_id, d->loop_id, n);
  UP(o.func_begin, d->func_begin, d->n_funcs + 1);
  UP(o.kfb, d->kernel_func_begin, d->n_kernels + 1);
  std::vector<uint32_t> kgb(d->n_kernels, 0xffffffffu);
  if (d->kernel_grid_blocks) std::copy(d->kernel_grid_blocks, d->kernel_grid_blocks + d->n_kernels, kgb.begin());
  UP(o.kgb, kgb.data(), kgb.size());
  UP(o.row_ptr, d->row_ptr, n + 1);
  UP(o.edge_def, d->edge_def, E);
  UP(o.edge_min, d->edge_min_len, E);
  UP(o.edge_max, d->edge_max_len, E);
  UP(o.edge_use, h.edge_use.data(), E);
  UP(o.edge_dom, d->edge_dom_k, E);
  UP(o.edge_lca, h.edge_lca.data(), E);
  UP(o.edge_kind, d->edge_kind, E);
  UP(o.def_ptr, h.def_ptr.data(), n + 1);
  UP(o.def_perm, h.def_perm.data(), E);
  UP(o.tile_run_ptr, h.tile_run_ptr.data(), h.tile_run_ptr.size());
  UP(o.run_be, h.run_be.data(), h.run_be.size());
  UP(o.run_dst, h.run_dst.data(), h.run_dst.size());
  UP(o.seg1_perm, h.seg1_perm.data(), h.seg1_perm.size());
  UP(o.seg1_begin, h.seg1_begin.data(), h.seg1_begin.size());
  UP(o.seg1_end, h.seg1_end.data(), h.seg1_end.size());
  UP(o.seg1_id, h.seg1_id.data(), h.seg1_id.size());
  UP(o.seg2_perm, h.seg2_perm.data(), h.seg2_perm.size());
  UP(o.seg2_begin, h.seg2_begin.data(), h.seg2_begin.size());
  UP(o.seg2_end, h.seg2_end.data(), h.seg2_end.size());
  UP(o.loop_items, h.loop_items.data(), h.loop_items.size());
  UP(o.loop_item_ptr, h.loop_item_ptr.data(), h.loop_item_ptr.size());
  UP(o.pre_perm, h.pre_perm.data(), h.pre_perm.size());
  UP(o.pre_begin, h.pre_begin.data(), h.pre_begin.size());
  UP(o.pre_end, h.pre_end.data(), h.pre_end.size());
  UP(o.kloop_ptr, h.kloop_ptr.data(), h.kloop_ptr.size());
  UP(o.kloops, h.kloops.data(), h.kloops.size());
  UP(o.loop_func, h.loop_func.data(), h.loop_func.size());
  CUDA_TRY(cudaMemsetAsync(ws + o.C, 0, o.partials - o.C, s));   // outputs zeroed
  if (o.part_reserved) CUDA_TRY(cudaMemsetAsync(ws + o.part_zero, 0, kPartZeroBytes, s));
  CUDA_TRY(cudaStreamSynchronize(s));

  int device = 0, n_sms = 0, optin = 0;   // queried before the handle exists: a failure leaks nothing
  CUDA_TRY(cudaGetDevice(&device));
  CUDA_TRY(cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, device));
  CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  gpa_program *p = new gpa_program();
  p->device = device;
  p->n_sms = n_sms;
  p->smem_optin = (size_t)optin;
  p->ws = ws;
  p->ws_bytes = bytes;
  DevProgram &dp = p->d;
  dp.n = n; dp.E = E; dp.R = d->n_reasons; dp.ncol = d->n_reasons + 6;
  dp.al_pre = n >= kPdlMaxInstr ? 1u : 0u;   // A_i, L_i by their own pass only for large programs
  dp.n_lines = d->n_lines; dp.n_loops = d->n_loops; dp.n_funcs = d->n_funcs; dp.n_kernels = d->n_kernels;
#define DP(field, type, off) dp.field = (type)(ws + o.off)
  DP(dinfo, const DefInfo *, dinfo);
  DP(opclass, const uint8_t *, opclass); DP(iflags, const uint8_t *, iflags);
  DP(latency, const uint32_t *, latency); DP(line_id, const uint32_t *, line_id);
  DP(loop_id, const int32_t *, loop_id); DP(func_begin, const uint32_t *, func_begin);
  DP(kernel_func_begin, const uint32_t *, kfb); DP(kernel_grid_blocks, const uint32_t *, kgb);
  DP(row_ptr, const uint32_t *, row_ptr); DP(edge_def, const uint32_t *, edge_def);
  DP(edge_min, const uint32_t *, edge_min); DP(edge_max, const uint32_t *, edge_max);
  DP(edge_use, const uint32_t *, edge_use); DP(edge_dom, const int32_t *, edge_dom);
  DP(edge_lca, const int32_t *, edge_lca); DP(edge_kind, const uint8_t *, edge_kind);
  DP(def_ptr, const uint32_t *, def_ptr); DP(def_perm, const uint32_t *, def_perm);
  DP(C, uint64_t *, C); DP(stats, uint64_t *, stats); DP(AL, uint64_t *, AL);
  DP(cand, uint8_t *, cand); DP(selfm, uint8_t *, selfm); DP(share, double *, share);
  DP(B, double *, B); DP(partials, uint32_t *, partials);
  DP(part_x, uint32_t *, part_x); DP(part_sync, unsigned int *, part_sync);
  DP(part_zero, const uint16_t *, part_zero);
#undef DP
  RollupPlan &rp = p->rp;
  rp.tile_run_ptr = (const uint32_t *)(ws + o.tile_run_ptr);
  rp.run_be = (const uint32_t *)(ws + o.run_be);
  rp.run_dst = (const uint32_t *)(ws + o.run_dst);
  rp.n_tiles = (uint32_t)h.tile_run_ptr.size() - 1;
  rp.seg1_perm = (const uint32_t *)(ws + o.seg1_perm);
  rp.part_v = (double *)(ws + o.part_v);
  rp.part_al = (uint64_t *)(ws + o.part_al);
  rp.seg1_begin = (const uint32_t *)(ws + o.seg1_begin);
  rp.seg1_end = (const uint32_t *)(ws + o.seg1_end);
  rp.n_seg1 = (uint32_t)h.seg1_begin.size();   // segments with 0 or >= 2 runs
  rp.seg1_id = (const uint32_t *)(ws + o.seg1_id);
  rp.n_rows1 = d->n_lines + d->n_loops + d->n_funcs;
  rp.seg2_perm = (const uint32_t *)(ws + o.seg2_perm);
  rp.seg2_begin = (const uint32_t *)(ws + o.seg2_begin);
  rp.seg2_end = (const uint32_t *)(ws + o.seg2_end);
  rp.n_seg2 = (uint32_t)h.seg2_begin.size();
  rp.rows_v = (double *)(ws + o.rows_v);
  rp.rows_al = (uint64_t *)(ws + o.rows_al);
  EstimatePlan &ep = p->ep;
  ep.pats = (const gpa_pattern *)(ws + o.pats);
  p->pats_dev = (gpa_pattern *)(ws + o.pats);
  ep.mval = (double *)(ws + o.mval);
  ep.mrow = (double *)(ws + o.mrow);
  ep.loop_items = (const uint32_t *)(ws + o.loop_items);
  ep.loop_item_ptr = (const uint32_t *)(ws + o.loop_item_ptr);
  ep.pre_perm = (const uint32_t *)(ws + o.pre_perm);
  ep.pre_begin = (const uint32_t *)(ws + o.pre_begin);
  ep.pre_end = (const uint32_t *)(ws + o.pre_end);
  ep.kloop_ptr = (const uint32_t *)(ws + o.kloop_ptr);
  ep.kloops = (const uint32_t *)(ws + o.kloops);
  ep.loop_func = (const int32_t *)(ws + o.loop_func);
  ep.lM_excl = (double *)(ws + o.lM_excl);
  ep.lM_incl = (double *)(ws + o.lM_incl);
  ep.fM = (double *)(ws + o.fM);
  ep.kM = (double *)(ws + o.kM);
  const size_t ncol = dp.ncol, rowv = 2 * ncol * 8, rowal = 16;
  const size_t r_line = 0, r_lex = d->n_lines, r_func = r_lex + d->n_loops,
               r_lin = r_func + d->n_funcs, r_kern = r_lin + d->n_loops;
  ep.loop_incl_al = rp.rows_al + 2 * r_lin;
  ep.func_al = rp.rows_al + 2 * r_func;
  ep.kern_al = rp.rows_al + 2 * r_kern;
  ep.out = (gpa_estimate_out *)(ws + o.est);
  ep.occ = (const KernOcc *)(ws + o.occ);
  p->occ_dev = (KernOcc *)(ws + o.occ);
  p->grid_host.assign(d->kernel_grid_blocks ? d->kernel_grid_blocks : nullptr,
                      d->kernel_grid_blocks ? d->kernel_grid_blocks + d->n_kernels : nullptr);
  p->ap.hot = (gpa_hotspot *)(ws + o.hot);
  p->ap.n_hot = (uint32_t *)(ws + o.n_hot);
  p->ap.rank = (uint32_t *)(ws + o.rank);
  p->ap.cov = (gpa_coverage *)(ws + o.cov);

  auto setv = [&](int v, size_t off, size_t by) { p->view_off[v] = off; p->view_bytes[v] = by; };
  setv(GPA_VIEW_COUNTS, o.C, (size_t)n * 2 * dp.R * 8);
  setv(GPA_VIEW_STATS, o.stats, 32);
  setv(GPA_VIEW_INSTR_AL, o.AL, (size_t)n * 16);
  setv(GPA_VIEW_CAND, o.cand, E);
  setv(GPA_VIEW_SELF, o.selfm, n);
  setv(GPA_VIEW_SHARE, o.share, (size_t)E * 24);
  setv(GPA_VIEW_INSTR_BLAME, o.B, (size_t)n * 64);
  setv(GPA_VIEW_LINE, o.rows_v + r_line * rowv, d->n_lines * rowv);
  setv(GPA_VIEW_LINE_AL, o.rows_al + r_line * rowal, d->n_lines * rowal);
  setv(GPA_VIEW_LOOP_EXCL, o.rows_v + r_lex * rowv, d->n_loops * rowv);
  setv(GPA_VIEW_LOOP_EXCL_AL, o.rows_al + r_lex * rowal, d->n_loops * rowal);
  setv(GPA_VIEW_LOOP_INCL, o.rows_v + r_lin * rowv, d->n_loops * rowv);
  setv(GPA_VIEW_LOOP_INCL_AL, o.rows_al + r_lin * rowal, d->n_loops * rowal);
  setv(GPA_VIEW_FUNC, o.rows_v + r_func * rowv, d->n_funcs * rowv);
  setv(GPA_VIEW_FUNC_AL, o.rows_al + r_func * rowal, d->n_funcs * rowal);
  setv(GPA_VIEW_KERNEL, o.rows_v + r_kern * rowv, d->n_kernels * rowv);
  setv(GPA_VIEW_KERNEL_AL, o.rows_al + r_kern * rowal, d->n_kernels * rowal);
  setv(GPA_VIEW_ESTIMATES, o.est, 0);

  // ingest variant: CTA-private shared-memory table when it fits, else the partitioned
  // (bucket-exchange) kernel when its constraints hold, else L2 atomics
  p->variant = VAR_SMEM;
  p->part_ok = o.part_reserved && part_feasible(dp, p->n_sms, p->smem_optin);
  if (ingest_smem_bytes(dp) > std::min(p->smem_optin, kSmemTableMax)) p->variant = p->part_ok ? VAR_PART : VAR_L2;
  // segment ingest: a shared-memory table sized for the largest kernel that fits
  {
    uint32_t max_np = 0;
    for (uint32_t k = 0; k < d->n_kernels; ++k)
      max_np = std::max(max_np, d->func_begin[d->kernel_func_begin[k + 1]] - d->func_begin[d->kernel_func_begin[k]]);
#ifndef GPA_SEG_SMEM_MAX
#define GPA_SEG_SMEM_MAX (72 * 1024)   // 3 CTAs of 512 threads per SM; kernels > 1024 instrs (R = 9) take L2 atomics
#endif
    const uint64_t cap = std::min<uint64_t>(std::min<uint64_t>(p->smem_optin, kSmemTableMax), GPA_SEG_SMEM_MAX) / 4;
    const uint64_t want = (uint64_t)max_np * 2 * d->n_reasons;
    p->seg_tab_bins = (uint32_t)std::min(want, cap);
  }
  *out = p;
  return GPA_OK;
}

gpa_status gpa_program_destroy(gpa_program *p) {
  if (!p) return GPA_OK;
  if (p->analyze_exec) cudaGraphExecDestroy(p->analyze_exec);
  if (p->capture_stream) cudaStreamDestroy(p->capture_stream);
  if (p->side_stream) cudaStreamDestroy(p->side_stream);
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  if (p->ev_join) cudaEventDestroy(p->ev_join);
  if (p->staging) cudaFree(p->staging);
  if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
  for (int i = 0; i < 2; ++i) {
    if (p->ev_copied[i]) cudaEventDestroy(p->ev_copied[i]);
    if (p->ev_done[i]) cudaEventDestroy(p->ev_done[i]);
  }
  delete p;
  return GPA_OK;
}

gpa_status gpa_reset_counts(gpa_program *p, void *stream) {
  gpa_status st = check_prog(p);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  // the stats words follow the count table in the workspace (layout: one block), so one memset
  // clears both (one launch fewer per step: it matters for small programs)
  CUDA_TRY(cudaMemsetAsync(p->d.C, 0, (size_t)p->d.n * 2 * p->d.R * 8 + 32, s));
  p->state = ST_COUNTS | (p->state & ST_PATTERNS);
  return GPA_OK;
}

gpa_status gpa_ingest_samples(gpa_program *p, const gpa_sample *d_samples, uint64_t n, void *stream) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (n == 0) {
    p->state = (p->state | ST_COUNTS) & ~(ST_BLAMED | ST_AGGREGATED | ST_ESTIMATED | ST_ADVISED);
    return GPA_OK;
  }
  if (!d_samples) return fail(GPA_ERR_INVALID_ARGUMENT, "d_samples is NULL");
  if (((uintptr_t)d_samples & 7u) != 0) return fail(GPA_ERR_INVALID_ARGUMENT, "d_samples not 8-byte aligned");
  cudaError_t e = launch_ingest(p->d, p->variant, d_samples, n, p->n_sms, p->smem_optin, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "ingest launch");
  p->launches += (p->variant == VAR_L2) ? 1 : 2;
  p->state = (p->state | ST_COUNTS) & ~(ST_BLAMED | ST_AGGREGATED | ST_ESTIMATED | ST_ADVISED);
  return GPA_OK;
}

gpa_status gpa_ingest_segments(gpa_program *p, const gpa_sample *d_samples, uint64_t n, const uint64_t *d_seg_begin,
                               const uint32_t *d_seg_kernel, uint32_t n_seg, uint32_t pc_base, void *stream) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (n_seg == 0 || n == 0) {
    p->state = (p->state | ST_COUNTS) & ~(ST_BLAMED | ST_AGGREGATED | ST_ESTIMATED | ST_ADVISED);
    return GPA_OK;
  }
  if (!d_samples || !d_seg_begin || !d_seg_kernel) return fail(GPA_ERR_INVALID_ARGUMENT, "NULL samples or segment table");
  if (((uintptr_t)d_samples & 7u) != 0) return fail(GPA_ERR_INVALID_ARGUMENT, "d_samples not 8-byte aligned");
  if (((uintptr_t)d_seg_begin & 7u) != 0 || ((uintptr_t)d_seg_kernel & 3u) != 0)
    return fail(GPA_ERR_INVALID_ARGUMENT, "segment table misaligned");
  cudaError_t e = launch_ingest_segments(p->d, d_samples, n, d_seg_begin, d_seg_kernel, n_seg, pc_base, p->seg_tab_bins,
                                         p->n_sms, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "segment ingest launch");
  p->launches += 1;
  p->state = (p->state | ST_COUNTS) & ~(ST_BLAMED | ST_AGGREGATED | ST_ESTIMATED | ST_ADVISED);
  return GPA_OK;
}

gpa_status gpa_ingest_samples_host(gpa_program *p, const gpa_sample *h, uint64_t n, void *stream) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (n && !h) return fail(GPA_ERR_INVALID_ARGUMENT, "h_samples is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t chunk = 4ull << 20;   // records per staging buffer (32 MB)
  if (!p->staging) {
    p->staging_bytes = chunk * 8;
    CUDA_TRY(cudaMalloc(&p->staging, 2 * p->staging_bytes));
    CUDA_TRY(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CUDA_TRY(cudaEventCreateWithFlags(&p->ev_copied[i], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&p->ev_done[i], cudaEventDisableTiming));
      CUDA_TRY(cudaEventRecord(p->ev_done[i], s));
    }
  }
  for (uint64_t k0 = 0, c = 0; k0 < n; k0 += chunk, ++c) {
    const uint64_t m = std::min(chunk, n - k0);
    const int b = (int)(c & 1);
    uint8_t *buf = (uint8_t *)p->staging + b * p->staging_bytes;
    CUDA_TRY(cudaStreamWaitEvent(p->copy_stream, p->ev_done[b], 0));
    CUDA_TRY(cudaMemcpyAsync(buf, h + k0, m * 8, cudaMemcpyHostToDevice, p->copy_stream));
    CUDA_TRY(cudaEventRecord(p->ev_copied[b], p->copy_stream));
    CUDA_TRY(cudaStreamWaitEvent(s, p->ev_copied[b], 0));
    st = gpa_ingest_samples(p, (const gpa_sample *)buf, m, stream);
    if (st) return st;
    CUDA_TRY(cudaEventRecord(p->ev_done[b], s));
  }
  if (n == 0) p->state = (p->state | ST_COUNTS) & ~(ST_BLAMED | ST_AGGREGATED | ST_ESTIMATED | ST_ADVISED);
  CUDA_TRY(cudaStreamSynchronize(s));
  return GPA_OK;
}

gpa_status gpa_blame(gpa_program *p, void *stream) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (!(p->state & ST_COUNTS)) return fail(GPA_ERR_BAD_STATE, "gpa_blame before gpa_reset_counts/gpa_ingest_samples");
  cudaError_t e = launch_blame(p->d, p->n_sms, (cudaStream_t)stream, &p->launches);
  if (e != cudaSuccess) return cuda_fail(e, "blame launch");
  p->state |= ST_BLAMED;
  p->state &= ~(ST_AGGREGATED | ST_ESTIMATED | ST_ADVISED);
  return GPA_OK;
}

gpa_status gpa_aggregate(gpa_program *p, void *stream) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (!(p->state & ST_BLAMED)) return fail(GPA_ERR_BAD_STATE, "gpa_aggregate before gpa_blame");
  cudaError_t e = launch_rollup(p->d, p->rp, p->n_sms, (cudaStream_t)stream, &p->launches);
  if (e != cudaSuccess) return cuda_fail(e, "rollup launch");
  p->state |= ST_AGGREGATED;
  p->state &= ~(ST_ESTIMATED | ST_ADVISED);
  return GPA_OK;
}

gpa_status gpa_set_patterns(gpa_program *p, const gpa_pattern *pats, uint32_t n_pat, void *stream) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (n_pat == 0 || n_pat > kPatWs || !pats)
    return fail(GPA_ERR_INVALID_ARGUMENT, "need 1..%u patterns", kPatWs);
  uint32_t loop_pats = 0;
  for (uint32_t q = 0; q < n_pat; ++q) {
    const gpa_pattern &x = pats[q];
    if (x.model > 5) return fail(GPA_ERR_INVALID_ARGUMENT, "pattern %u: model %u > 5", q, x.model);
    if (x.sample_class > 1) return fail(GPA_ERR_INVALID_ARGUMENT, "pattern %u: sample_class > 1", q);
    if (x.model == 2 || x.model == 4) ++loop_pats;
    if (x.model == 5 && (!(x.W > 0) || !(x.W_new > 0) || !(x.f >= 0)))
      return fail(GPA_ERR_DOMAIN, "pattern %u: Eq. 10 needs W > 0, W_new > 0, f >= 0", q);
    if (!(x.ratio >= 0)) return fail(GPA_ERR_DOMAIN, "pattern %u: ratio must be >= 0", q);
  }
  if (loop_pats > kLoopPatWs) return fail(GPA_ERR_INVALID_ARGUMENT, "at most %u loop-scoped patterns", kLoopPatWs);
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemcpyAsync(p->pats_dev, pats, n_pat * sizeof(gpa_pattern), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  p->ep.n_pat = n_pat;
  // the analyze graph bakes the pattern plan (n_pat, loop_slot) into its
  // kernel parameters: any new pattern set invalidates it
  if (p->analyze_exec) {
    cudaGraphExecDestroy(p->analyze_exec);
    p->analyze_exec = nullptr;
  }
  for (uint32_t q = 0, slot = 0; q < (uint32_t)kPatternsMax; ++q)
    p->ep.loop_slot[q] = (q < n_pat && (pats[q].model == 2 || pats[q].model == 4)) ? (int8_t)slot++ : (int8_t)-1;
  p->view_bytes[GPA_VIEW_ESTIMATES] = (size_t)p->d.n_kernels * n_pat * sizeof(gpa_estimate_out);
  p->state |= ST_PATTERNS;
  p->state &= ~(ST_ESTIMATED | ST_ADVISED);
  return GPA_OK;
}

gpa_status gpa_estimate(gpa_program *p, void *stream) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (!(p->state & ST_AGGREGATED)) return fail(GPA_ERR_BAD_STATE, "gpa_estimate before gpa_aggregate");
  if (!(p->state & ST_PATTERNS)) return fail(GPA_ERR_BAD_STATE, "gpa_estimate before gpa_set_patterns");
  cudaError_t e = launch_estimate(p->d, p->ep, p->n_sms, (cudaStream_t)stream, &p->launches);
  if (e != cudaSuccess) return cuda_fail(e, "estimate launch");
  p->state = (p->state | ST_ESTIMATED) & ~ST_ADVISED;
  return GPA_OK;
}

static gpa_status analyze_graph(gpa_program *p, uint32_t npat, void *stream);

gpa_status gpa_analyze(gpa_program *p, void *stream) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (!(p->state & ST_COUNTS)) return fail(GPA_ERR_BAD_STATE, "gpa_analyze before gpa_reset_counts/gpa_ingest_samples");
  const uint32_t npat = (p->state & ST_PATTERNS) ? p->ep.n_pat : 0;
  if (p->analyze_mode == GPA_ANALYZE_FUSED) {
    if (!fused_feasible(npat)) return fail(GPA_ERR_INVALID_ARGUMENT, "fused analysis needs <= 16 patterns (%u set)", npat);
    EstimatePlan ep = p->ep;
    ep.n_pat = npat;
    const cudaError_t e = launch_analyze_fused(p->d, p->rp, ep, p->n_sms, kFusedMaxCtas, (cudaStream_t)stream,
                                               &p->launches);
    if (e != cudaSuccess) return cuda_fail(e, "fused analysis launch");
  } else {
    const gpa_status gs = analyze_graph(p, npat, stream);
    if (gs) return gs;
  }
  p->state |= ST_BLAMED | ST_AGGREGATED;
  p->state = npat ? (p->state | ST_ESTIMATED) & ~ST_ADVISED : p->state & ~(ST_ESTIMATED | ST_ADVISED);
  return GPA_OK;
}

gpa_status gpa_set_analyze_mode(gpa_program *p, int mode) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (mode < GPA_ANALYZE_AUTO || mode > GPA_ANALYZE_FUSED) return fail(GPA_ERR_INVALID_ARGUMENT, "analyze mode %d unknown", mode);
  p->analyze_mode = mode;
  return GPA_OK;
}

// the multi-kernel analysis, captured once as a CUDA graph and replayed
static gpa_status analyze_graph(gpa_program *p, uint32_t npat, void *stream) {
  if (!p->analyze_exec || p->analyze_npat != npat) {
    if (p->analyze_exec) {
      cudaGraphExecDestroy(p->analyze_exec);
      p->analyze_exec = nullptr;
    }
    if (!p->capture_stream) CUDA_TRY(cudaStreamCreateWithFlags(&p->capture_stream, cudaStreamNonBlocking));
    if (!p->side_stream) CUDA_TRY(cudaStreamCreateWithFlags(&p->side_stream, cudaStreamNonBlocking));
    if (!p->ev_fork) CUDA_TRY(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
    if (!p->ev_join) CUDA_TRY(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
    cudaGraph_t g = nullptr;
    uint64_t n = 0;
    // two branches after the blame rows: def reduction -> rollup, and the estimate sums (which read
    // only cand / share / selfm and C); they join before Eqs. 2-5 / 10, which need the rollup's A sums
    CUDA_TRY(cudaStreamBeginCapture(p->capture_stream, cudaStreamCaptureModeThreadLocal));
#ifndef GPA_EST_FORK
#define GPA_EST_FORK 1
#endif
    cudaStream_t cs = p->capture_stream, ss = GPA_EST_FORK ? p->side_stream : p->capture_stream;
    cudaError_t e = launch_blame_rows(p->d, p->n_sms, cs, &n);
    if (e == cudaSuccess && npat) {
      e = cudaEventRecord(p->ev_fork, cs);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(ss, p->ev_fork, 0);
      if (e == cudaSuccess) e = launch_estimate_sums(p->d, p->ep, p->n_sms, ss, &n);
      if (e == cudaSuccess) e = cudaEventRecord(p->ev_join, ss);
    }
#ifndef GPA_DEF_ROLL
#define GPA_DEF_ROLL 1
#endif
    // the def reduction fused into the rollup tiles (one dependent level fewer: config 3's analysis
    // 63 -> 61 us, config 2's 34 -> 33 us), or its own kernel (from 2^20 instructions on: config 4
    // measured 0.5 % slower fused)
#ifndef GPA_DEF_ROLL_MAX_N
#define GPA_DEF_ROLL_MAX_N kPdlMaxInstr
#endif
    const bool dr = GPA_DEF_ROLL && p->d.n < (uint32_t)(GPA_DEF_ROLL_MAX_N) && p->rp.n_tiles == (p->d.n + 31) / 32;
    if (e == cudaSuccess && !dr) e = launch_def_reduce(p->d, p->n_sms, cs, &n);
    if (e == cudaSuccess)
      e = launch_rollup(p->d, p->rp, p->n_sms, cs, &n, dr);
    if (e == cudaSuccess && npat) {
      e = cudaStreamWaitEvent(cs, p->ev_join, 0);
      if (e == cudaSuccess) e = launch_estimate_final(p->d, p->ep, p->n_sms, cs, &n);
    }
    cudaError_t e2 = cudaStreamEndCapture(p->capture_stream, &g);
    if (e != cudaSuccess) return cuda_fail(e, "analyze capture");
    if (e2 != cudaSuccess) return cuda_fail(e2, "analyze end capture");
    e = cudaGraphInstantiate(&p->analyze_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(e, "analyze instantiate");
    p->analyze_npat = npat;
    p->analyze_launches = n;
  }
  CUDA_TRY(cudaGraphLaunch(p->analyze_exec, (cudaStream_t)stream));
  p->launches += p->analyze_launches;
  return GPA_OK;
}

static gpa_status validate_sass(const gpa_sass_desc *h) {
  const uint32_t n = h->n_instr, NB = h->n_blocks, NF = h->n_funcs;
  if (n == 0 || NB == 0 || NF == 0) return fail(GPA_ERR_INVALID_PROGRAM, "empty SASS program");
  if (h->block_begin[0] != 0 || h->block_begin[NB] != n || h->func_begin[0] != 0 || h->func_begin[NF] != n)
    return fail(GPA_ERR_INVALID_PROGRAM, "block / function ranges must cover [0, n_instr)");
  std::vector<uint32_t> bfunc(NB);
  for (uint32_t b = 0, f = 0; b < NB; ++b) {
    if (h->block_begin[b + 1] <= h->block_begin[b]) return fail(GPA_ERR_INVALID_PROGRAM, "empty or unordered block %u", b);
    while (f < NF && h->func_begin[f + 1] <= h->block_begin[b]) ++f;
    if (f >= NF || h->block_begin[b + 1] > h->func_begin[f + 1]) return fail(GPA_ERR_INVALID_PROGRAM, "block %u crosses a function", b);
    bfunc[b] = f;
  }
  for (uint32_t f = 0; f < NF; ++f)
    if (h->func_begin[f + 1] <= h->func_begin[f]) return fail(GPA_ERR_INVALID_PROGRAM, "empty function %u", f);
  if (h->succ_ptr[0] != 0) return fail(GPA_ERR_INVALID_PROGRAM, "succ_ptr[0] != 0");
  for (uint32_t b = 0; b < NB; ++b) {
    if (h->succ_ptr[b + 1] < h->succ_ptr[b]) return fail(GPA_ERR_INVALID_PROGRAM, "succ_ptr not monotone");
    for (uint32_t e = h->succ_ptr[b]; e < h->succ_ptr[b + 1]; ++e)
      if (h->succ[e] >= NB || bfunc[h->succ[e]] != bfunc[b])
        return fail(GPA_ERR_INVALID_PROGRAM, "block %u: successor outside its function", b);
  }
  for (uint32_t i = 0; i < n; ++i) {
    if (h->guard[i] > 15 || h->wbar[i] > 63 || h->rbar[i] > 63 || h->wait[i] > 63)
      return fail(GPA_ERR_INVALID_PROGRAM, "instruction %u: guard / barrier field out of range", i);
    for (int t = 0; t < 4; ++t) {
      const uint16_t d = h->dst[4u * i + t], sr = h->src[4u * i + t];
      if ((d != 0xFFFF && d > 262) || (sr != 0xFFFF && sr > 262) || (d > 255 && d < 256) || (sr > 255 && sr < 256))
        return fail(GPA_ERR_INVALID_PROGRAM, "instruction %u: operand out of range", i);
    }
  }
  return GPA_OK;
}

gpa_status gpa_slice(const gpa_sass_desc *h, uint64_t cap_edges, uint32_t *h_row_ptr, uint32_t *h_def, uint8_t *h_kind,
                     uint32_t *h_min, uint32_t *h_max, int32_t *h_dom, uint64_t *n_edges, void *stream) {
  if (!h || !h_row_ptr || !n_edges || !h->func_begin || !h->block_begin || !h->succ_ptr || !h->guard || !h->dst ||
      !h->src || !h->wbar || !h->rbar || !h->wait || (h->succ_ptr && h->n_blocks && h->succ_ptr[h->n_blocks] && !h->succ))
    return fail(GPA_ERR_INVALID_ARGUMENT, "NULL SASS array or output");
  if (cap_edges && (!h_def || !h_kind || !h_min || !h_max || !h_dom))
    return fail(GPA_ERR_INVALID_ARGUMENT, "NULL edge output array");
  gpa_status vst = validate_sass(h);
  if (vst) return vst;
  int dev = 0, n_sms = 148;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, dev));
  int status = 0;
  cudaError_t e = launch_slice(h, h_row_ptr, cap_edges, h_def, h_kind, h_min, h_max, h_dom, n_edges, n_sms,
                               (cudaStream_t)stream, &status);
  if (e != cudaSuccess) return cuda_fail(e, "slice");
  if (status == 1) return fail(GPA_ERR_OVERFLOW, "slicing: a search exceeded its state budget");
  if (status == 2) return fail(GPA_ERR_OVERFLOW, "slicing: %llu edges > cap_edges %llu", (unsigned long long)*n_edges,
                               (unsigned long long)cap_edges);
  return GPA_OK;
}

gpa_status gpa_simulate(const gpa_sass_desc *h, const uint8_t *h_cls, const uint32_t *h_lat, uint32_t func,
                        const gpa_simcfg *cfg, uint32_t n_sm, uint64_t cap, gpa_sample *d_records, int32_t *d_truth,
                        uint64_t *h_counts, void *stream) {
  if (!h || !h_cls || !h_lat || !cfg || !d_records || !h_counts || !h->func_begin || !h->block_begin || !h->succ_ptr ||
      !h->guard || !h->dst || !h->src || !h->wbar || !h->rbar || !h->wait)
    return fail(GPA_ERR_INVALID_ARGUMENT, "NULL argument");
  gpa_status vst = validate_sass(h);
  if (vst) return vst;
  if (func >= h->n_funcs) return fail(GPA_ERR_INVALID_ARGUMENT, "func %u >= n_funcs", func);
  if (!cfg->schedulers || !cfg->warps_per_scheduler || !cfg->period || !cfg->trip_count || !n_sm || !cap)
    return fail(GPA_ERR_INVALID_ARGUMENT, "schedulers, warps, period, trip_count, n_sm and cap must be > 0");
  if ((uint64_t)cfg->schedulers * cfg->warps_per_scheduler > 64)
    return fail(GPA_ERR_INVALID_ARGUMENT, "at most 64 warps per simulated SM");
  cudaError_t e = launch_simulate(h, h_cls, h_lat, func, *cfg, n_sm, cap, d_records, d_truth, h_counts,
                                  (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "simulate");
  for (uint32_t i = 0; i < n_sm; ++i)
    if (h_counts[i] == ~0ull) return fail(GPA_ERR_OVERFLOW, "SM %u exceeded cap_per_sm or max_cycles", i);
  return GPA_OK;
}

// Occupancy of every kernel (DESIGN.md §3.2 Q34): the usual calculator -- blocks per SM are the
// tightest of the warp, block-slot, register (allocation-unit rounded) and shared-memory limits.
gpa_status gpa_set_launches(gpa_program *p, const gpa_launch *h_launch, const gpa_arch *arch, void *stream) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (!h_launch || !arch) return fail(GPA_ERR_INVALID_ARGUMENT, "NULL launches or arch");
  if (!arch->sm_count || !arch->warp_size || !arch->schedulers_per_sm || !arch->reg_alloc_unit)
    return fail(GPA_ERR_INVALID_ARGUMENT, "arch needs sm_count, warp_size, schedulers_per_sm, reg_alloc_unit > 0");
  const uint32_t nk = p->d.n_kernels;
  std::vector<KernOcc> occ(nk);
  for (uint32_t k = 0; k < nk; ++k) {
    KernOcc &o = occ[k];
    o = KernOcc{0.0, 0.0, 0.0, 0u, 0u};
    const gpa_launch &l = h_launch[k];
    const uint32_t grid = p->grid_host.empty() ? 0u : p->grid_host[k];
    if (!l.threads_per_block || !grid || grid == 0xffffffffu) continue;
    const uint64_t warps_per_block = (l.threads_per_block + arch->warp_size - 1) / arch->warp_size;
    const uint64_t unit = arch->reg_alloc_unit;
    const uint64_t regs_per_warp = l.regs_per_thread ? ((uint64_t)l.regs_per_thread * arch->warp_size + unit - 1) / unit * unit : 0;
    const uint64_t by_warps = arch->max_warps_per_sm / warps_per_block;
    const uint64_t by_slots = arch->max_blocks_per_sm;
    const uint64_t by_regs = regs_per_warp ? arch->regs_per_sm / (regs_per_warp * warps_per_block) : UINT64_MAX;
    const uint64_t by_smem = l.smem_per_block ? arch->smem_per_sm / l.smem_per_block : UINT64_MAX;
    const uint64_t blocks = std::min(std::min(by_warps, by_slots), std::min(by_regs, by_smem));
    if (blocks == 0) continue;   // cannot launch
    const bool slots_bind = by_slots == blocks && by_warps > blocks;   // ties go to the warp limit
    const uint64_t resident = std::min<uint64_t>(blocks, (grid + arch->sm_count - 1) / arch->sm_count);
    o.W = (double)(resident * warps_per_block) / arch->schedulers_per_sm;
    if (grid < arch->sm_count) {
      o.match_block = 1;
      o.W_new_block = o.W * grid / arch->sm_count;
    }
    if (slots_bind && resident == blocks) {
      uint64_t warps = arch->max_warps_per_sm;
      if (regs_per_warp) warps = std::min<uint64_t>(warps, arch->regs_per_sm / regs_per_warp);
      o.W_new_thread = (double)warps / arch->schedulers_per_sm;
      o.match_thread = o.W_new_thread > o.W;
    }
  }
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemcpyAsync(p->occ_dev, occ.data(), nk * sizeof(KernOcc), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  p->state &= ~(ST_ESTIMATED | ST_ADVISED);
  return GPA_OK;
}

gpa_status gpa_advise(gpa_program *p, uint32_t top_k, void *stream) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (top_k < 1 || top_k > GPA_TOP_K_MAX) return fail(GPA_ERR_INVALID_ARGUMENT, "top_k %u not in [1, %u]", top_k, GPA_TOP_K_MAX);
  if (!(p->state & ST_ESTIMATED)) return fail(GPA_ERR_BAD_STATE, "gpa_advise before gpa_estimate / gpa_analyze with patterns");
  p->ap.top_k = top_k;
  cudaError_t e = launch_advice(p->d, p->ep, p->ap, (cudaStream_t)stream, &p->launches);
  if (e != cudaSuccess) return cuda_fail(e, "advice launch");
  p->state |= ST_ADVISED;
  return GPA_OK;
}

gpa_status gpa_read_advice(gpa_program *p, gpa_hotspot *h_hot, uint32_t *h_n_hot, uint32_t *h_rank, gpa_coverage *h_cov,
                           void *stream) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (!(p->state & ST_ADVISED)) return fail(GPA_ERR_BAD_STATE, "gpa_read_advice before gpa_advise");
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t nk = p->d.n_kernels, nq = p->ep.n_pat, K = p->ap.top_k;
  if (h_hot)   // device rows hold kTopKMax entries; the caller's hold top_k
    CUDA_TRY(cudaMemcpy2DAsync(h_hot, K * sizeof(gpa_hotspot), p->ap.hot, kTopKMax * sizeof(gpa_hotspot),
                               K * sizeof(gpa_hotspot), nk * nq, cudaMemcpyDeviceToHost, s));
  if (h_n_hot) CUDA_TRY(cudaMemcpyAsync(h_n_hot, p->ap.n_hot, nk * nq * 4, cudaMemcpyDeviceToHost, s));
  if (h_rank) CUDA_TRY(cudaMemcpyAsync(h_rank, p->ap.rank, nk * nq * 4, cudaMemcpyDeviceToHost, s));
  if (h_cov) CUDA_TRY(cudaMemcpyAsync(h_cov, p->ap.cov, nk * sizeof(gpa_coverage), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return GPA_OK;
}

gpa_status gpa_read_estimates(gpa_program *p, gpa_estimate_out *h_out, void *stream) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (!h_out) return fail(GPA_ERR_INVALID_ARGUMENT, "h_out is NULL");
  if (!(p->state & ST_PATTERNS)) return fail(GPA_ERR_BAD_STATE, "no patterns set");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemcpyAsync(h_out, p->ep.out, p->view_bytes[GPA_VIEW_ESTIMATES], cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return GPA_OK;
}

gpa_status gpa_get_stats(gpa_program *p, uint64_t out[4], void *stream) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (!out) return fail(GPA_ERR_INVALID_ARGUMENT, "out is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemcpyAsync(out, p->d.stats, 32, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return GPA_OK;
}

gpa_status gpa_view(gpa_program *p, int view, uint64_t *offset, uint64_t *bytes) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (view < 0 || view >= GPA_VIEW_COUNT_ || !offset || !bytes)
    return fail(GPA_ERR_INVALID_ARGUMENT, "bad view id or NULL output");
  *offset = p->view_off[view];
  *bytes = p->view_bytes[view];
  return GPA_OK;
}

gpa_status gpa_instr_vector(gpa_program *p, double *d_out, void *stream) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (!d_out) return fail(GPA_ERR_INVALID_ARGUMENT, "d_out is NULL");
  if (!(p->state & ST_BLAMED)) return fail(GPA_ERR_BAD_STATE, "gpa_instr_vector before gpa_blame");
  cudaError_t e = launch_vrows(p->d, d_out, p->n_sms, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "instr vector launch");
  return GPA_OK;
}

gpa_status gpa_program_info(gpa_program *p, uint64_t info[8]) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (!info) return fail(GPA_ERR_INVALID_ARGUMENT, "info is NULL");
  const DevProgram &d = p->d;
  uint64_t v[8] = {d.n, d.E, d.R, d.ncol, d.n_lines, d.n_loops, d.n_funcs, d.n_kernels};
  memcpy(info, v, sizeof(v));
  return GPA_OK;
}

gpa_status gpa_ingest_variant(gpa_program *p, int *variant) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (!variant) return fail(GPA_ERR_INVALID_ARGUMENT, "variant is NULL");
  *variant = p->variant;
  return GPA_OK;
}

gpa_status gpa_set_ingest_variant(gpa_program *p, int variant) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (variant < 0 || variant > VAR_L2) return fail(GPA_ERR_INVALID_ARGUMENT, "variant %d unknown", variant);
  if (variant == VAR_SMEM && ingest_smem_bytes(p->d) > std::min(p->smem_optin, kSmemTableMax))
    return fail(GPA_ERR_INVALID_ARGUMENT, "count table does not fit shared memory");
  if (variant == VAR_PART && !p->part_ok)
    return fail(GPA_ERR_INVALID_ARGUMENT, "partitioned ingest not applicable to this program");
  p->variant = variant;
  return GPA_OK;
}

gpa_status gpa_launch_count(gpa_program *p, uint64_t *launches) {
  gpa_status st = check_prog(p);
  if (st) return st;
  if (!launches) return fail(GPA_ERR_INVALID_ARGUMENT, "launches is NULL");
  *launches = p->launches;
  return GPA_OK;
}

}  // extern "C"

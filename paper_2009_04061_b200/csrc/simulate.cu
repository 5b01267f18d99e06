// simulate.cu -- a GPU workload generator for the path: the PC-sampling
// model of P:125-142 run as one thread per simulated SM (DESIGN.md §3.2 Q40-Q44).
//
// Each simulated SM runs schedulers x warps_per_scheduler warps of one SASS function with an
// in-order scoreboard (register ready times, write / read barrier clear times), loose round-robin
// issue (one instruction per scheduler per cycle), and every `period` cycles takes a sample from
// the schedulers in turn: an active sample if that scheduler issued, a latency sample otherwise,
// with the sampled warp's stall reason (memory / execution / synchronization dependency on the
// producer it waits for, or not-selected).  The records go straight into a device buffer that
// gpa_ingest_samples / gpa_ingest_segments consume; a ground-truth sidecar names the producer of
// every dependency stall.  SMs are independent: a launch simulates thousands of them.
#include <algorithm>
#include <vector>

#include "gpa_internal.cuh"

namespace gpa {
namespace {

constexpr uint32_t kSimRegs = 263;   // R0-R254, RZ, P0-P6
constexpr uint32_t kSimThreads = 64;
constexpr uint32_t kNotSel = 7;

struct SimIn {
  uint32_t n, n_blocks, f0;
  const uint32_t *block_begin, *blk_of, *succ_ptr, *succ;
  const uint8_t *guard, *wbar, *rbar, *wait, *cls;
  const uint16_t *dst, *src;
  const uint32_t *lat;
};

struct SimWarp {
  uint32_t pc, done, loop_count, last_pc, predv;
  int64_t last_issue;
};

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ bool mem_class(uint8_t c) { return c == 0 || c == 1 || c == 3 || c == 4; }

// readiness of warp x's next instruction at cycle t; else the reason and producer
__device__ bool sim_ready(const SimIn &s, const SimWarp &x, const int64_t *ready, const int32_t *prod,
                          const int64_t *bclear, const int32_t *bprod, int64_t t, uint32_t &why, int32_t &who) {
  const uint32_t j = x.pc;
  int64_t worst = -1;
  int32_t p = -1;
  for (uint32_t b = 0; b < 6; ++b)
    if (((s.wait[j] >> b) & 1u) && bclear[b] > t && bclear[b] > worst) { worst = bclear[b]; p = bprod[b]; }
  for (int t2 = 0; t2 < 4; ++t2) {
    const uint16_t r = s.src[4u * j + t2];
    if (r == 0xFFFFu || r == 255u) continue;
    if (ready[r] > t && ready[r] > worst) { worst = ready[r]; p = prod[r]; }
  }
  if ((s.guard[j] & 7u) != 7u) {
    const uint32_t r = 256u + (s.guard[j] & 7u);
    if (ready[r] > t && ready[r] > worst) { worst = ready[r]; p = prod[r]; }
  }
  if (worst < 0) return true;
  who = p;
  why = p < 0 ? R_EXEC : (s.cls[p] == 9 ? R_SYNC : mem_class(s.cls[p]) ? R_MEM : R_EXEC);
  return false;
}

__global__ void __launch_bounds__(kSimThreads) k_simulate(SimIn s, gpa_simcfg cfg, uint32_t n_sm, uint64_t cap,
                                                          uint8_t *scratch, size_t per_sm, gpa_sample *out,
                                                          int32_t *truth, uint64_t *counts) {
  const uint32_t sm = blockIdx.x * blockDim.x + threadIdx.x;
  if (sm >= n_sm) return;
  const uint32_t S = cfg.schedulers, WP = cfg.warps_per_scheduler, W = S * WP;
  uint8_t *base = scratch + (size_t)sm * per_sm;
  SimWarp *w = reinterpret_cast<SimWarp *>(base);
  int64_t *ready = reinterpret_cast<int64_t *>(w + W);       // [W][kSimRegs]
  int64_t *bclear = ready + (size_t)W * kSimRegs;            // [W][6]
  int32_t *prod = reinterpret_cast<int32_t *>(bclear + (size_t)W * 6);   // [W][kSimRegs]
  int32_t *bprod = prod + (size_t)W * kSimRegs;              // [W][6]
  uint32_t *rr = reinterpret_cast<uint32_t *>(bprod + (size_t)W * 6);    // [S]
  uint32_t *srr = rr + S;                                    // [S]
  int32_t *issued = reinterpret_cast<int32_t *>(srr + S);    // [S]
  for (uint32_t k = 0; k < W; ++k) {
    SimWarp &x = w[k];
    x.pc = s.f0; x.done = 0; x.loop_count = 0; x.last_pc = 0; x.last_issue = -1; x.predv = 0;
    for (uint32_t r = 0; r < kSimRegs; ++r) { ready[(size_t)k * kSimRegs + r] = 0; prod[(size_t)k * kSimRegs + r] = -1; }
    for (uint32_t r = 0; r < 6; ++r) { bclear[k * 6 + r] = 0; bprod[k * 6 + r] = -1; }
    for (uint32_t q = 0; q < 7; ++q)
      x.predv |= (uint32_t)(mix64(cfg.seed ^ ((uint64_t)(sm * W + k) << 8) ^ q) & 1u) << q;
  }
  for (uint32_t i = 0; i < S; ++i) { rr[i] = 0; srr[i] = 0; }
  uint32_t live = W;
  uint64_t n_rec = 0;
  gpa_sample *o = out + (uint64_t)sm * cap;
  int32_t *tr = truth ? truth + (uint64_t)sm * cap : nullptr;
  int64_t c = 0;
  bool fail = false;
  for (; live > 0 && !fail; ++c) {
    if (c >= (int64_t)cfg.max_cycles) { fail = true; break; }
    for (uint32_t sc = 0; sc < S; ++sc) {
      issued[sc] = -1;
      for (uint32_t i = 0; i < WP; ++i) {
        const uint32_t lw = (rr[sc] + i) % WP, wi = lw * S + sc;
        SimWarp &x = w[wi];
        int64_t *rd = ready + (size_t)wi * kSimRegs;
        int32_t *pd = prod + (size_t)wi * kSimRegs;
        uint32_t why;
        int32_t who;
        if (x.done || x.last_issue == c || !sim_ready(s, x, rd, pd, bclear + wi * 6, bprod + wi * 6, c, why, who)) continue;
        const uint32_t j = x.pc, g = s.guard[j];
        const bool on = (g & 7u) == 7u || ((((x.predv >> (g & 7u)) & 1u) != 0) != ((g & 8u) != 0));
        if (on) {
          for (int t2 = 0; t2 < 4; ++t2) {
            const uint16_t d = s.dst[4u * j + t2];
            if (d == 0xFFFFu || d == 255u) continue;
            rd[d] = c + s.lat[j];
            pd[d] = (int32_t)j;
          }
          for (uint32_t t2 = 0; t2 < 6; ++t2) {
            if ((s.wbar[j] >> t2) & 1u) { bclear[wi * 6 + t2] = c + s.lat[j]; bprod[wi * 6 + t2] = (int32_t)j; }
            else if ((s.rbar[j] >> t2) & 1u) { bclear[wi * 6 + t2] = c + cfg.rbar_latency; bprod[wi * 6 + t2] = (int32_t)j; }
          }
        }
        x.last_issue = c;
        x.last_pc = j;
        issued[sc] = (int32_t)wi;
        rr[sc] = (lw + 1u) % WP;
        if (j + 1 < s.block_begin[s.blk_of[j] + 1]) {
          x.pc = j + 1;
        } else {   // control policy: self-loops run trip_count times, two-way branches by warp parity
          const uint32_t bb = s.blk_of[j], e0 = s.succ_ptr[bb], e1 = s.succ_ptr[bb + 1];
          uint32_t self = 0, other = 0xFFFFFFFFu, n_other = 0, first_other = 0xFFFFFFFFu;
          for (uint32_t e = e0; e < e1; ++e) {
            if (s.succ[e] == bb) self = 1;
            else { if (first_other == 0xFFFFFFFFu) first_other = s.succ[e]; ++n_other; }
          }
          if (self && x.loop_count + 1 < cfg.trip_count) {
            ++x.loop_count;
            other = bb;
          } else {
            x.loop_count = 0;
            if (n_other == 1 || (self && n_other >= 1)) other = first_other;
            else if (n_other >= 2) {
              const uint32_t pick = wi % 2u;
              uint32_t cnt = 0;
              for (uint32_t e = e0; e < e1; ++e)
                if (s.succ[e] != bb) { if (cnt == pick) { other = s.succ[e]; break; } ++cnt; }
            }
          }
          if (other == 0xFFFFFFFFu) { x.done = 1; --live; }
          else x.pc = s.block_begin[other];
        }
        break;
      }
    }
    if (c > 0 && c % cfg.period == 0) {
      const uint32_t sc2 = (uint32_t)((c / cfg.period - 1) % S);
      for (uint32_t i = 0; i < WP; ++i) {
        const uint32_t lw = (srr[sc2] + i) % WP, wi = lw * S + sc2;
        const SimWarp &x = w[wi];
        if (x.done && issued[sc2] != (int32_t)wi) continue;
        srr[sc2] = (lw + 1u) % WP;
        const uint32_t cls = issued[sc2] >= 0 ? 0u : 1u;
        uint32_t pc, reason, why = 0;
        int32_t who = -1;
        if (issued[sc2] == (int32_t)wi) {
          pc = x.last_pc;
          reason = R_NONE;
        } else {
          pc = x.pc;
          reason = sim_ready(s, x, ready + (size_t)wi * kSimRegs, prod + (size_t)wi * kSimRegs, bclear + wi * 6,
                             bprod + wi * 6, c, why, who)
                       ? kNotSel
                       : why;
        }
        if (n_rec >= cap) { fail = true; break; }
        gpa_sample r;
        r.pc = pc;
        r.count = 1;
        r.reason = (uint8_t)reason;
        r.flags = (uint8_t)cls;
        o[n_rec] = r;
        if (tr) tr[n_rec] = (reason == R_MEM || reason == R_EXEC || reason == R_SYNC) ? who : -1;
        ++n_rec;
        break;
      }
    }
  }
  counts[sm] = fail ? ~0ull : n_rec;
}

}  // namespace

cudaError_t launch_simulate(const gpa_sass_desc *h, const uint8_t *h_cls, const uint32_t *h_lat, uint32_t func,
                            const gpa_simcfg &cfg, uint32_t n_sm, uint64_t cap, gpa_sample *d_out, int32_t *d_truth,
                            uint64_t *h_counts, cudaStream_t st) {
  const uint32_t n = h->n_instr, NB = h->n_blocks;
  std::vector<uint32_t> blk_of(n);
  for (uint32_t b = 0; b < NB; ++b)
    for (uint32_t j = h->block_begin[b]; j < h->block_begin[b + 1]; ++j) blk_of[j] = b;
  std::vector<void *> owned;
  cudaError_t e = cudaSuccess;
  auto up = [&](const void *src, size_t bytes) -> void * {
    void *d = nullptr;
    if (e == cudaSuccess) e = cudaMallocAsync(&d, std::max<size_t>(bytes, 16), st);
    if (e == cudaSuccess && bytes) e = cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, st);
    owned.push_back(d);
    return d;
  };
  SimIn s;
  s.n = n;
  s.n_blocks = NB;
  s.f0 = h->func_begin[func];
  s.block_begin = (const uint32_t *)up(h->block_begin, (NB + 1) * 4);
  s.blk_of = (const uint32_t *)up(blk_of.data(), (size_t)n * 4);
  s.succ_ptr = (const uint32_t *)up(h->succ_ptr, (NB + 1) * 4);
  s.succ = (const uint32_t *)up(h->succ, (size_t)h->succ_ptr[NB] * 4);
  s.guard = (const uint8_t *)up(h->guard, n);
  s.wbar = (const uint8_t *)up(h->wbar, n);
  s.rbar = (const uint8_t *)up(h->rbar, n);
  s.wait = (const uint8_t *)up(h->wait, n);
  s.cls = (const uint8_t *)up(h_cls, n);
  s.dst = (const uint16_t *)up(h->dst, (size_t)n * 8);
  s.src = (const uint16_t *)up(h->src, (size_t)n * 8);
  s.lat = (const uint32_t *)up(h_lat, (size_t)n * 4);
  const uint32_t W = cfg.schedulers * cfg.warps_per_scheduler;
  const size_t per_sm = (((size_t)W * sizeof(SimWarp) + 7) & ~(size_t)7) + (size_t)W * kSimRegs * 12 + (size_t)W * 6 * 12 +
                        (size_t)cfg.schedulers * 12 + 64;
  void *d_scr = nullptr, *d_cnt = nullptr;
  if (e == cudaSuccess) e = cudaMallocAsync(&d_scr, ((per_sm + 255) & ~(size_t)255) * n_sm, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&d_cnt, (size_t)n_sm * 8, st);
  if (e == cudaSuccess) {
    k_simulate<<<(n_sm + kSimThreads - 1) / kSimThreads, kSimThreads, 0, st>>>(
        s, cfg, n_sm, cap, (uint8_t *)d_scr, (per_sm + 255) & ~(size_t)255, d_out, d_truth, (uint64_t *)d_cnt);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(h_counts, d_cnt, (size_t)n_sm * 8, cudaMemcpyDeviceToHost, st);
  for (void *p : owned) if (p) cudaFreeAsync(p, st);
  if (d_scr) cudaFreeAsync(d_scr, st);
  if (d_cnt) cudaFreeAsync(d_cnt, st);
  cudaError_t e2 = cudaStreamSynchronize(st);
  return e != cudaSuccess ? e : e2;
}

}  // namespace gpa

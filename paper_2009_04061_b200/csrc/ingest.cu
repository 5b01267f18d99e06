// ingest.cu -- row a1: PC-sample records -> C[pc][class][reason].
//
// Variant S (k_ingest_smem): the whole count table fits one CTA's shared memory (n*2R*4 B
//   <= 227 KB, e.g. config 2).  A persistent grid of one 1024-thread CTA per SM streams the
//   records with 16-byte non-allocating loads (4 outstanding per thread), validates each
//   record and adds its count to a CTA-private u32 table with shared-memory atomics; u32
//   wrap-around is detected from the atomic's return value and carried into the u64 table.
//   CTA tables are written out coalesced and summed per bin by k_ingest_reduce (no global
//   atomics on the hot path, deterministic).
// Variant P (k_ingest_part): tables larger than one SM's shared memory (config 3: 50k PCs x 18
//   bins = 3.6 MB).  The bin space is split into G = #SM contiguous buckets, one per CTA of a
//   persistent cooperative grid, each held in that CTA's shared memory.  Every CTA streams
//   64 KB chunks of records into a double-buffered shared-memory ring with TMA bulk copies
//   (cp.async.bulk + mbarrier), counting-sorts each chunk by bucket in shared memory, and
//   writes each bucket's run of 4-byte keys {local bin:16 | count:16} coalesced into an
//   L2-resident exchange buffer slot (dst, src).  One chunk later the owning CTA drains its
//   slots into its table with shared-memory atomics.  Producer/consumer hand-off uses monotonic
//   per-buffer global counters (split-phase: arrive after producing chunk k, wait before
//   consuming it one iteration later), with 3 exchange buffers in flight, so HBM sees each
//   record once and the keys never leave L2.  Keys beyond a slot's capacity (extreme skew)
//   fall back to L2 atomics, so the result is exact for any distribution.
// Variant L (k_ingest_l2): tables larger than shared memory; one RED.E.ADD.64 per record into
//   the L2-resident u64 table.
#include <algorithm>

#include "gpa_internal.cuh"

namespace gpa {
namespace {

constexpr int kIngestThreads = 1024;
constexpr int kUnroll = 4;

__device__ __forceinline__ uint4 ld_stream(const uint4 *p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ uint2 ld_stream8(const uint2 *p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}

struct IngestStats {
  unsigned long long valid, bad_records, bad_samples;
};

// Validity (Q12) and bin index (pc*2 + class)*R + reason.
__device__ __forceinline__ bool decode(uint32_t pc, uint32_t w, uint32_t n, uint32_t R,
                                       uint32_t &bin, uint32_t &cnt) {
  cnt = w & 0xffffu;
  const uint32_t reason = (w >> 16) & 0xffu, flags = w >> 24;
  const bool ok = pc < n && reason < R && flags <= 1u && !(flags == 1u && reason == R_NONE);
  bin = (pc * 2u + flags) * R + reason;
  return ok;
}

__device__ __forceinline__ void flush_stats(IngestStats st, uint64_t *stats) {
  __shared__ unsigned long long s[3];
  if (threadIdx.x < 3) s[threadIdx.x] = 0;
  __syncthreads();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    st.valid += __shfl_down_sync(0xffffffffu, st.valid, o);
    st.bad_records += __shfl_down_sync(0xffffffffu, st.bad_records, o);
    st.bad_samples += __shfl_down_sync(0xffffffffu, st.bad_samples, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&s[0], st.valid);
    atomicAdd(&s[1], st.bad_records);
    atomicAdd(&s[2], st.bad_samples);
  }
  __syncthreads();
  if (threadIdx.x < 3 && s[threadIdx.x]) atomicAdd((unsigned long long *)&stats[threadIdx.x], s[threadIdx.x]);
}

// Records are processed as 16-byte pairs; `head` (0/1 record before the first 16-byte
// boundary) and an odd tail are handled by thread 0 of CTA 0.
template <bool kSmem>
__global__ void __launch_bounds__(kIngestThreads, 1)
k_ingest(const uint2 *__restrict__ rec, uint64_t n_rec, uint32_t head, uint32_t n_instr, uint32_t R,
         uint32_t bins, uint64_t *__restrict__ C, uint32_t *__restrict__ partials,
         uint64_t *__restrict__ stats) {
  extern __shared__ uint32_t tab[];
  if (kSmem) {
    for (uint32_t b = threadIdx.x; b < bins; b += blockDim.x) tab[b] = 0;
    __syncthreads();
  }
  IngestStats st{0, 0, 0};
  auto add = [&](uint32_t pc, uint32_t w) {
    uint32_t bin, cnt;
    if (decode(pc, w, n_instr, R, bin, cnt)) {
      st.valid += cnt;
      if (kSmem) {
        const uint32_t old = atomicAdd(&tab[bin], cnt);
        if (old > 0xffffffffu - cnt) atomicAdd((unsigned long long *)&C[bin], 1ull << 32);  // u32 wrap
      } else {
        atomicAdd((unsigned long long *)&C[bin], (unsigned long long)cnt);
      }
    } else {
      st.bad_records += 1;
      st.bad_samples += cnt;
    }
  };
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (head) {
      uint2 v = ld_stream8(rec);
      add(v.x, v.y);
    }
    if ((n_rec - head) & 1ull) {
      uint2 v = ld_stream8(rec + n_rec - 1);
      add(v.x, v.y);
    }
  }
  const uint4 *r16 = reinterpret_cast<const uint4 *>(rec + head);
  const uint64_t n16 = (n_rec - head) >> 1;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (kUnroll - 1) * stride < n16; i += kUnroll * stride) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = ld_stream(r16 + i + u * stride);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      add(v[u].x, v[u].y);
      add(v[u].z, v[u].w);
    }
  }
  for (; i < n16; i += stride) {
    uint4 v = ld_stream(r16 + i);
    add(v.x, v.y);
    add(v.z, v.w);
  }
  flush_stats(st, stats);
  if (kSmem) {
    // __syncthreads() inside flush_stats ordered every table update before this read-out
    uint32_t *dst = partials + (uint64_t)blockIdx.x * bins;
    for (uint32_t b = threadIdx.x; b < bins; b += blockDim.x) dst[b] = tab[b];
  }
}

// Sum the per-CTA tables bin by bin (coalesced across threads) into the u64 table.
__global__ void k_ingest_reduce(const uint32_t *__restrict__ partials, uint32_t n_ctas,
                                uint32_t bins, uint64_t *__restrict__ C) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < bins; b += gridDim.x * blockDim.x) {
    uint64_t s = 0;
    for (uint32_t c = 0; c < n_ctas; ++c) s += partials[(uint64_t)c * bins + b];
    if (s) C[b] += s;
  }
}


// ----------------------------------------------------------------------------- variant P
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void spin_until(const unsigned int *ctr, unsigned int target) {
  while (true) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    if (v >= target) break;
    __nanosleep(32);
  }
}

struct PartArgs {
  const uint2 *rec;       // 16-byte aligned body
  uint64_t n_even;        // records in the body (even)
  uint32_t n_instr, R, bins, ppb, bpb;
  uint32_t mg;            // ceil(2^32 / G): pc / G = umulhi(pc, mg), exact for pc < 2^32 / G
  uint64_t *C, *stats;
  uint32_t *X;            // [kPartBufs][kPartMaxCtas dst][kPartMaxCtas src][kPartCap] keys, 0-padded
  unsigned int *sync;     // [kPartBufs] produced, [kPartBufs] consumed
};

constexpr int kProdThreads = kPartThreads / 2;    // warps 0-15: partition the record stream
constexpr int kConsThreads = kPartThreads / 2;    // warps 16-31: drain this CTA's bucket
constexpr int kProdRecs = kPartChunk / kProdThreads;   // records per producer thread per chunk
constexpr int kRing = 4;                           // TMA ring depth (chunks in flight per CTA)
constexpr int kConsVec = (kPartMaxCtas * kPartCap / 4 + kConsThreads - 1) / kConsThreads;  // uint4 per thread

__device__ __forceinline__ void named_bar(uint32_t id, uint32_t threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void tma_bulk_load_ef(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}

// shared -> global bulk copy (async proxy), tracked by this thread's bulk async-groups
__device__ __forceinline__ void tma_bulk_store(void *gdst, const void *ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_addr(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_le1() { asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__global__ void __launch_bounds__(kPartThreads, 1) k_ingest_part(PartArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  const uint32_t G = gridDim.x, me = blockIdx.x;
  const uint32_t slot_keys = G * kPartCap;                                       // one staging buffer
  uint2 *ring = reinterpret_cast<uint2 *>(sm);                                   // [kRing][chunk] records
  uint32_t *stag = reinterpret_cast<uint32_t *>(sm + kRing * kPartChunk * 8);  // [2][G][cap] keys
  uint32_t *cnt = stag + 2 * slot_keys;                                         // [kPartMaxCtas]
  uint64_t *bars = reinterpret_cast<uint64_t *>(cnt + kPartMaxCtas);            // [kRing]
  uint32_t *tab = reinterpret_cast<uint32_t *>(bars + kRing);                   // [bpb]
  (void)lane;
  for (uint32_t i = tid; i < a.bpb; i += kPartThreads) tab[i] = 0;
  for (uint32_t i = tid; i < 2 * slot_keys; i += kPartThreads) stag[i] = 0;
  for (uint32_t i = tid; i < kPartMaxCtas; i += kPartThreads) cnt[i] = 0;
  if (tid == 0) {
    for (int r = 0; r < kRing; ++r) mbar_init(&bars[r], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t per_chunk = (uint64_t)kPartChunk * G;
  const uint32_t n_chunks = (uint32_t)((a.n_even + per_chunk - 1) / per_chunk);
  auto slice_len = [&](uint32_t k, uint64_t &start) -> uint32_t {
    start = (uint64_t)k * per_chunk + (uint64_t)me * kPartChunk;
    return start >= a.n_even ? 0u
                             : (uint32_t)(a.n_even - start < (uint64_t)kPartChunk ? a.n_even - start : (uint64_t)kPartChunk);
  };
  IngestStats st{0, 0, 0};
  if (tid < kProdThreads) {
    // ======================= producers: TMA ring -> decode + slot-shaped scatter -> bulk stores
    const uint32_t ptid = tid;
    const uint64_t pol = evict_first_policy();
    const uint32_t n_instr = a.n_instr, R = a.R, twoR = 2 * a.R, mg = a.mg;
    auto issue = [&](uint32_t k) {
      uint64_t s0;
      const uint32_t len = slice_len(k, s0);
      if (len) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bars[k % kRing], len * 8);
        tma_bulk_load_ef(ring + (k % kRing) * kPartChunk, a.rec + s0, len * 8, &bars[k % kRing], pol);
      }
    };
    if (ptid == 0)
      for (uint32_t k = 0; k < kRing - 1 && k < n_chunks; ++k) issue(k);
    for (uint32_t k = 0; k < n_chunks; ++k) {
      uint64_t s0;
      const uint32_t len = slice_len(k, s0);
      const uint32_t buf = k % kPartBufs;
      uint32_t *sg = stag + (k & 1) * slot_keys;
      if (ptid == 0) {
        // ring slot (k+3)%4 held chunk k-1, decoded (and released by the barriers) last iteration
        if (k + kRing - 1 < n_chunks) issue(k + kRing - 1);
        // exchange buffer k%NBUF is free once every CTA drained chunk k-NBUF
        if (k >= (uint32_t)kPartBufs) spin_until(&a.sync[kPartBufs + buf], G * (k / kPartBufs));
      }
      if (len) mbar_wait(&bars[k % kRing], (k / kRing) & 1);
      named_bar(1, kProdThreads);
      // ---- decode: branchless validity, bucket = pc mod G (interleaved PCs balance the load),
      //      key = {local bin:16 | count:16}, local bin = (pc / G) * 2R + class * R + reason;
      //      the key goes straight to position cnt[b]++ of bucket b's zero-padded slot
      const uint4 *rs = reinterpret_cast<const uint4 *>(ring + (k % kRing) * kPartChunk);
      uint32_t valid = 0, badr = 0, bads = 0;
#pragma unroll
      for (int u = 0; u < kProdRecs / 2; ++u) {
        const uint32_t pair = u * kProdThreads + ptid;
        const bool in = 2 * pair < len;   // len is even: both records of the pair or neither
        const uint4 v = in ? rs[pair] : make_uint4(0xffffffffu, 0, 0xffffffffu, 0);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t pc = h ? v.z : v.x, w = h ? v.w : v.y;
          const uint32_t reason = (w >> 16) & 0xffu, flags = w >> 24, c = w & 0xffffu;
          const bool ok = pc < n_instr && reason < R && w < 0x2000000u && (w >> 16) != 0x100u;
          const uint32_t q = __umulhi(pc, mg), b = pc - q * G;
          const uint32_t local = q * twoR + flags * R + reason;
          if (ok) {
            const uint32_t pos = atomicAdd(&cnt[b], 1u);
            if (pos < (uint32_t)kPartCap) {
              sg[b * kPartCap + pos] = __byte_perm(local, w, 0x5410);
            } else {   // slot overflow (extreme skew): exact via L2 atomics
              atomicAdd((unsigned long long *)&a.C[((uint64_t)q * G + b) * twoR + flags * R + reason],
                        (unsigned long long)c);
            }
          }
          valid += ok ? c : 0u;
          badr += (in && !ok) ? 1u : 0u;
          bads += (in && !ok) ? c : 0u;
        }
      }
      st.valid += valid;
      st.bad_records += badr;
      st.bad_samples += bads;
      // every thread that wrote the staging buffer orders its generic-proxy writes before the
      // async-proxy bulk stores issued after the barrier
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      named_bar(1, kProdThreads);
      if (ptid < G) {   // one bulk store per destination: slot (dst = ptid, src = me) of buffer k%NBUF
        const uint64_t slot = ((uint64_t)buf * kPartMaxCtas + ptid) * kPartMaxCtas + me;
        tma_bulk_store(a.X + slot * kPartCap, sg + ptid * kPartCap, kPartCap * 4);
        bulk_commit();
        cnt[ptid] = 0;
        if (k > 0) {      // chunk k-1's stores are now complete (global writes and smem reads)
          bulk_wait_le1();
          fence_proxy_async_global();
        }
      }
      named_bar(1, kProdThreads);
      if (k > 0) {
        if (ptid == 0) {
          __threadfence();
          atomicAdd(&a.sync[(k - 1) % kPartBufs], 1u);   // this CTA produced chunk k-1
        }
        uint4 *old = reinterpret_cast<uint4 *>(stag + ((k - 1) & 1) * slot_keys);   // re-zero for chunk k+1
        for (uint32_t i = ptid; i < slot_keys / 4; i += kProdThreads) old[i] = make_uint4(0, 0, 0, 0);
      }
    }
    if (n_chunks) {
      if (ptid < G) {
        bulk_wait_all();
        fence_proxy_async_global();
      }
      named_bar(1, kProdThreads);
      if (ptid == 0) {
        __threadfence();
        atomicAdd(&a.sync[(n_chunks - 1) % kPartBufs], 1u);
      }
    }
  } else {
    // ======================= consumers: my bucket's slot row (contiguous, L2) -> table
    const uint32_t ctid = tid - kProdThreads;
    const uint32_t nvec = slot_keys / 4;
    auto wait_chunk = [&](uint32_t j) {
      if (ctid == 0) spin_until(&a.sync[j % kPartBufs], G * (j / kPartBufs + 1));
      named_bar(2, kConsThreads);
    };
    auto load_chunk = [&](uint32_t j, uint4 (&r)[kConsVec]) {
      const uint4 *row = reinterpret_cast<const uint4 *>(
          a.X + ((uint64_t)(j % kPartBufs) * kPartMaxCtas + me) * kPartMaxCtas * kPartCap);
#pragma unroll
      for (int u = 0; u < kConsVec; ++u) {
        const uint32_t idx = ctid + u * kConsThreads;
        r[u] = idx < nvec ? __ldcg(row + idx) : make_uint4(0, 0, 0, 0);
      }
    };
    auto add_key = [&](uint32_t kk) {
      const uint32_t c = kk >> 16;
      if (c) {
        const uint32_t lb = kk & 0xffffu;
        const uint32_t old = atomicAdd(&tab[lb], c);
        if (old > 0xffffffffu - c)
          atomicAdd((unsigned long long *)&a.C[((uint64_t)(lb / (2 * a.R)) * G + me) * (2 * a.R) + lb % (2 * a.R)],
                    1ull << 32);   // u32 wrap
      }
    };
    uint4 cur[kConsVec], nxt[kConsVec];
    if (n_chunks) {
      wait_chunk(0);
      load_chunk(0, cur);
    }
    for (uint32_t j = 0; j < n_chunks; ++j) {
      if (j + 1 < n_chunks) {
        wait_chunk(j + 1);
        load_chunk(j + 1, nxt);
      }
#pragma unroll
      for (int u = 0; u < kConsVec; ++u) {
        add_key(cur[u].x);
        add_key(cur[u].y);
        add_key(cur[u].z);
        add_key(cur[u].w);
      }
      named_bar(2, kConsThreads);
      if (ctid == 0) atomicAdd(&a.sync[kPartBufs + j % kPartBufs], 1u);   // this CTA drained chunk j
#pragma unroll
      for (int u = 0; u < kConsVec; ++u) cur[u] = nxt[u];
    }
  }
  __syncthreads();
  flush_stats(st, a.stats);
  const uint32_t twoR = 2 * a.R;
  for (uint32_t i = tid; i < a.bpb; i += kPartThreads) {
    const uint32_t bin = ((i / twoR) * G + me) * twoR + i % twoR;   // local (pc/G, class, reason) -> bin
    if (bin < a.bins && tab[i]) atomicAdd((unsigned long long *)&a.C[bin], (unsigned long long)tab[i]);
  }
}

// head record and odd tail of the body, outside the 16-byte-aligned even part
__global__ void k_ingest_edges(const uint2 *rec, uint64_t n_rec, uint32_t head, uint32_t n_instr, uint32_t R,
                               uint64_t *C, uint64_t *stats) {
  IngestStats st{0, 0, 0};
  const uint64_t idx[2] = {0, n_rec - 1};
  const bool use[2] = {head != 0, ((n_rec - head) & 1ull) != 0 && n_rec - 1 >= head};
  for (int t = 0; t < 2; ++t) {
    if (!use[t] || threadIdx.x != t) continue;
    const uint2 v = ld_stream8(rec + idx[t]);
    uint32_t bin, c;
    if (decode(v.x, v.y, n_instr, R, bin, c)) {
      st.valid += c;
      atomicAdd((unsigned long long *)&C[bin], (unsigned long long)c);
    } else {
      st.bad_records += 1;
      st.bad_samples += c;
    }
  }
  flush_stats(st, stats);
}

}  // namespace

size_t part_smem_bytes(uint32_t bpb, uint32_t G) {
  return (size_t)kRing * kPartChunk * 8 + (size_t)2 * G * kPartCap * 4 + kPartMaxCtas * 4 + kRing * 8 +
         (size_t)bpb * 4;
}

static uint32_t part_grid(int n_sms) { return (uint32_t)std::min(n_sms, kPartMaxCtas); }

// buckets: PCs pc = q*G + b go to CTA b (ppb = ceil(n/G) PCs, ppb * 2R bins); 16-bit local bins
static bool part_shape(const DevProgram &p, int n_sms, uint32_t &G, uint32_t &ppb, uint32_t &bpb) {
  if (n_sms < 1) return false;
  G = part_grid(n_sms);
  ppb = (p.n + G - 1) / G;
  bpb = ppb * 2 * p.R;
  return ppb < 4096 && bpb < 65536;
}

bool part_feasible(const DevProgram &p, int n_sms, size_t smem_optin) {
  uint32_t G, ppb, bpb;
  return part_shape(p, n_sms, G, ppb, bpb) && part_smem_bytes(bpb, G) + 256 <= smem_optin;
}

size_t ingest_smem_bytes(const DevProgram &p) { return (size_t)p.n * 2 * p.R * 4; }

cudaError_t launch_ingest(const DevProgram &p, int variant, const void *records, uint64_t n,
                          int n_sms, size_t smem_optin, cudaStream_t s) {
  const uint2 *rec = (const uint2 *)records;
  const uint32_t head = ((uintptr_t)rec & 15u) ? 1u : 0u;
  const uint32_t bins = p.n * 2 * p.R;
  // enough CTAs to keep HBM busy, one per SM at most; tiny streams use few CTAs
  const uint64_t per_cta = 1ull << 15;
  uint32_t grid = (uint32_t)std::min<uint64_t>((uint64_t)n_sms, std::max<uint64_t>(1, (n + per_cta - 1) / per_cta));
  if (variant == VAR_SMEM) {
    const size_t smem = ingest_smem_bytes(p);
    if (smem > smem_optin || smem > kSmemTableMax) return cudaErrorInvalidValue;
    grid = std::min<uint32_t>(grid, kMaxIngestCtas);
    cudaError_t e = cudaFuncSetAttribute(k_ingest<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_ingest<true><<<grid, kIngestThreads, smem, s>>>(rec, n, head, p.n, p.R, bins, p.C, p.partials, p.stats);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const uint32_t rgrid = std::max<uint32_t>(1, std::min<uint32_t>((bins + 255) / 256, 4 * n_sms));
    k_ingest_reduce<<<rgrid, 256, 0, s>>>(p.partials, grid, bins, p.C);
    return cudaGetLastError();
  }
  if (variant == VAR_L2) {
    if (n_sms > 0) grid = std::min<uint32_t>(grid * 4, 4 * n_sms);
    k_ingest<false><<<grid, kIngestThreads, 0, s>>>(rec, n, head, p.n, p.R, bins, p.C, nullptr, p.stats);
    return cudaGetLastError();
  }
  if (variant == VAR_PART) {
    if (!part_feasible(p, n_sms, smem_optin)) return cudaErrorInvalidValue;
    uint32_t G, ppb, bpb;
    part_shape(p, n_sms, G, ppb, bpb);
    PartArgs a;
    a.rec = rec + head;
    a.n_even = (n - head) & ~1ull;
    a.n_instr = p.n;
    a.R = p.R;
    a.bins = bins;
    a.ppb = ppb;
    a.bpb = bpb;
    a.mg = (uint32_t)(((1ull << 32) + G - 1) / G);
    a.C = p.C;
    a.stats = p.stats;
    a.X = p.part_x;
    a.sync = p.part_sync;
    const size_t smem = part_smem_bytes(a.bpb, G);
    cudaError_t e = cudaFuncSetAttribute(k_ingest_part, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(p.part_sync, 0, 2 * kPartBufs * sizeof(unsigned int), s);
    if (e != cudaSuccess) return e;
    if (head || ((n - head) & 1ull)) {
      k_ingest_edges<<<1, 32, 0, s>>>(rec, n, head, p.n, p.R, p.C, p.stats);
      e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    if (a.n_even == 0) return cudaSuccess;
    void *args[] = {&a};
    return cudaLaunchCooperativeKernel((const void *)k_ingest_part, dim3(G), dim3(kPartThreads), args, smem, s);
  }
  return cudaErrorNotSupported;
}

}  // namespace gpa

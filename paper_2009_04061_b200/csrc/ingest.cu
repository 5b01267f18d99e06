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
//   bins = 3.6 MB).  The bin space is split over the G = #SM CTAs of a persistent cooperative
//   grid by pc mod G, each CTA holding its bins in shared memory.  Per round every CTA streams
//   kPartChunk records (direct 16-byte loads), counting-sorts them by destination CTA into
//   zero-padded slots of 2-byte keys {local bin:13-15 | count:3-1} in shared memory, and writes its
//   whole row of slots into an L2-resident exchange buffer with one bulk store; each CTA then
//   fetches its column of every producer's row with one 2-D TMA tile load and adds the keys into
//   its table with shared-memory atomics.  Warp-specialised (decoders / control / publisher /
//   loader / processors) with mbarrier hand-offs inside the CTA and monotonic
//   per-buffer release/acquire counters between CTAs (16 exchange buffers in flight), so HBM
//   sees each record once and the keys stay in L2.  Counts > 7, slot overflow (extreme skew)
//   and malformed records go through L2 atomics / the stats, so the result is exact for any
//   distribution.  Tables of up to 2^15 bins per CTA (programs of ~250k instructions at R = 9)
//   stay on this path (15-bit local bins, counts > 1 via L2).
// Variant L (k_ingest_l2): tables larger than shared memory; one RED.E.ADD.64 per record into
//   the L2-resident u64 table.
#include <algorithm>
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "gpa_internal.cuh"

namespace gpa {
namespace {

constexpr int kIngestThreads = 1024;
#ifndef GPA_INGEST_UNROLL
#define GPA_INGEST_UNROLL 4
#endif
constexpr int kUnroll = GPA_INGEST_UNROLL;   // 16-byte loads in flight per thread (variants S and L)
#ifndef GPA_SMEM_U16
#define GPA_SMEM_U16 1
#endif
constexpr bool kSmemU16 = GPA_SMEM_U16;      // variant S: u16 counters in shared memory

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
  // kSmemU16: u16 counters, two bins per word (bins = n * 2R is even); else one u32 counter per bin
  const uint32_t words = kSmemU16 ? bins / 2 : bins;
  if (kSmem) {
    for (uint32_t b = threadIdx.x; b < words; b += blockDim.x) tab[b] = 0;
    __syncthreads();
  }
  IngestStats st{0, 0, 0};
  auto add = [&](uint32_t pc, uint32_t w) {
    uint32_t bin, cnt;
    if (decode(pc, w, n_instr, R, bin, cnt)) {
      st.valid += cnt;
      if (kSmem && kSmemU16) {
        // u16 counters (half the table: half the zeroing, flush and reduction traffic).  The
        // atomic's returned word decides, exactly and race-free, what a field overflow did, and the
        // difference goes to C through L2 atomics (rare): a low field wrapping past 0xffff carries
        // +1 into the high field (C[hi] -= 1; if that wraps the high field too, C[hi] += 65536),
        // a high field wrapping drops 65536 out of the word.
        const uint32_t sh = (bin & 1u) * 16u;
        const uint32_t old = atomicAdd(&tab[bin >> 1], cnt << sh);
        if (((old >> sh) & 0xffffu) + cnt > 0xffffu) {
          atomicAdd((unsigned long long *)&C[bin], 65536ull);
          if (!sh) atomicAdd((unsigned long long *)&C[bin + 1], (old >> 16) == 0xffffu ? 65535ull : ~0ull);
        }
      } else if (kSmem) {
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
  if (kSmem) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // k_ingest_reduce may launch
  flush_stats(st, stats);
  if (kSmem) {
    // __syncthreads() inside flush_stats ordered every table update before this read-out
    uint32_t *dst = partials + (uint64_t)blockIdx.x * words;
    for (uint32_t b = threadIdx.x; b < words; b += blockDim.x) dst[b] = tab[b];
  }
}

// Sum the per-CTA tables bin by bin (coalesced across threads) into the u64 table: blockIdx.y
// takes a group of kReduceGroup CTA tables (all loads of a thread independent and in flight
// together), and the group sums meet in C through u64 atomics (integer adds: exact in any order).
constexpr uint32_t kReduceGroup = 16;
__global__ void k_ingest_reduce(const uint32_t *__restrict__ partials, uint32_t n_ctas,
                                uint32_t bins, uint64_t *__restrict__ C) {
  pdl_wait();   // launched as a programmatic dependent of k_ingest: scheduled during its tail
  const uint32_t c0 = blockIdx.y * kReduceGroup;
  const uint32_t words = kSmemU16 ? bins / 2 : bins;   // a word = two u16 bins, or one u32 bin
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < words; b += gridDim.x * blockDim.x) {
    uint32_t v[kReduceGroup];
#pragma unroll
    for (uint32_t c = 0; c < kReduceGroup; ++c) v[c] = c0 + c < n_ctas ? partials[(uint64_t)(c0 + c) * words + b] : 0u;
    if (kSmemU16) {
      uint64_t lo = 0, hi = 0;
#pragma unroll
      for (uint32_t c = 0; c < kReduceGroup; ++c) {
        lo += v[c] & 0xffffu;
        hi += v[c] >> 16;
      }
      if (lo) atomicAdd((unsigned long long *)&C[2 * b], (unsigned long long)lo);
      if (hi) atomicAdd((unsigned long long *)&C[2 * b + 1], (unsigned long long)hi);
    } else {
      uint64_t s = 0;
#pragma unroll
      for (uint32_t c = 0; c < kReduceGroup; ++c) s += v[c];
      if (s) atomicAdd((unsigned long long *)&C[b], (unsigned long long)s);
    }
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
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity), "r"(1000000u)   // suspend-time hint (ns): park the warp instead of spinning
      : "memory");
}
#ifndef GPA_SPIN_RELAXED
#define GPA_SPIN_RELAXED 0
#endif
// wait until *ctr >= target (a counter other CTAs advance with red.release.gpu).  An ld.acquire.gpu
// per poll compiles to a load plus an L1 invalidation (CCTL.IVALL, 16 M per 10^9 records in round
// 1's ncu profile); polling with relaxed loads and one acquire fence after the wait
// (GPA_SPIN_RELAXED=1) measured slower on config 3 (2.22 -> 2.42 ms).
__device__ __forceinline__ void spin_until(const unsigned int *ctr, unsigned int target) {
  while (true) {
    unsigned int v;
#if GPA_SPIN_RELAXED
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
#else
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
#endif
    if (v >= target) break;
    __nanosleep(32);
  }
#if GPA_SPIN_RELAXED
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
}

#ifdef GPA_PART_TIMING
// phase timers (cycles, summed over CTAs) for tuning: read with tools/part_timing.py
__device__ unsigned long long g_part_timing[16];
#define PT_DECL unsigned long long _pt0 = 0, _pt1, _pta[16] = {0};
#define PT_START _pt0 = clock64()
#define PT_MARK(slot)    \
  do {                   \
    _pt1 = clock64();    \
    _pta[slot] += _pt1 - _pt0; \
    _pt0 = _pt1;         \
  } while (0)
#define PT_FLUSH                                                                       \
  do {                                                                                 \
    if ((threadIdx.x & 31) == 0)                                                       \
      for (int _i = 0; _i < 16; ++_i)                                                  \
        if (_pta[_i]) atomicAdd(&g_part_timing[_i], _pta[_i]);                         \
  } while (0)
#else
#define PT_DECL
#define PT_START do {} while (0)
#define PT_MARK(slot) do {} while (0)
#define PT_FLUSH do {} while (0)
#endif

struct PartArgs {
  const uint2 *rec;       // 16-byte aligned body
  uint64_t n_even;        // records in the body (even)
  uint32_t n_instr, R, bins, ppb, bpb;
  uint32_t mg;            // ceil(2^32 / G): pc / G = umulhi(pc, mg), exact for pc < 2^32 / G
  uint64_t *C, *stats;
  uint16_t *X;            // [kPartBufs][src < kPartMaxCtas][dst < G][kPartCap] 2-byte keys, zero-padded
  unsigned int *sync;     // [kPartBufs] produced, [kPartBufs] consumed
  const uint16_t *zero;   // kPartZeroBytes of zeros (staging clears by bulk copy, GPA_PART_TMA_ZERO)
};

// warp roles of the 1024-thread CTA
#ifndef GPA_PART_DECODE_WARPS
#define GPA_PART_DECODE_WARPS 20
#endif
constexpr int kDecodeWarps = GPA_PART_DECODE_WARPS;  // warps 0..D-1: decode + scatter records
constexpr int kCtrlWarp = kDecodeWarps;              // warp D: TMA issue, exchange stores, recycling
constexpr int kPubWarp = kDecodeWarps + 1;           // warp D+1: publication of stored chunks
constexpr int kConsWarps = kPartThreads / 32 - kDecodeWarps - 2;   // warps D+2..: drain this CTA's bucket
constexpr int kLoaderWarp = kPubWarp + 1;           //   warp 24: exchange -> inbox TMA loads
constexpr int kProcBase = (kLoaderWarp + 1) * 32;   //   warps 25-31: inbox -> table
constexpr int kProcThreads = (kConsWarps - 1) * 32;
constexpr int kDecodeThreads = kDecodeWarps * 32;
constexpr int kConsThreads = kConsWarps * 32;
constexpr int kConsBase = (kPubWarp + 1) * 32;
#ifndef GPA_PART_INBOX
#define GPA_PART_INBOX 2
#endif
constexpr int kInbox = GPA_PART_INBOX;                          // consumer inbox depth (exchange chunks)
#ifndef GPA_PART_STAGE
#define GPA_PART_STAGE 3
#endif
constexpr int kStage = GPA_PART_STAGE;                          // staging buffers (decode k+1 never waits for chunk k's store)
constexpr int kTrash = 32;                         // lane-distinct sink for dropped keys / padding
// key = local bin (LB bits) | count (16 - LB bits, at most 7): LB = 13 for tables below 8,192 bins
// per CTA (config 3), 14 / 15 for the larger tables of 100k-250k-instruction programs, whose
// records of count > 1 / > 3 take the rare (L2 atomic) branch
constexpr uint32_t kMinLocalBits = 13, kMaxLocalBits = 15;
constexpr uint32_t kMaxKeyCount = 7;
template <uint32_t LB> constexpr uint32_t key_max_count() { return (1u << (16 - LB)) - 1 < kMaxKeyCount ? (1u << (16 - LB)) - 1 : kMaxKeyCount; }
constexpr uint32_t kDummyCount = 1u << 30;        // dummy-bucket counter start (never < kPartCap)
// a chunk adds at most G * cap * 7 samples to any one table entry: a launch of at most
// flush_every(shape) chunks (the host splits longer streams) keeps every entry below 2^32 until the
// final flush
constexpr uint32_t kBarProc = 2;   // named barrier of the processor warps (0 is __syncthreads)
// Exchange shapes (records per CTA per chunk, slot capacity, staging / inbox ring depths, exchange
// buffers).  Base: the shape above (tuning macros GPA_PART_*).  Wide: bigger chunks with fuller
// slots (mean 60.5 keys of 80 instead of 43 of 56 at G = 148) and a 2-deep inbox, used when the
// CTA then stays within kWideSmemMax -- the shared-memory size above which the SM's L1 carve-out
// shrinks (config 3: 142 KB; 2.21 -> 2.15 ms); tables too large for it keep Base.
template <int CHUNK, int CAP, int STAGE, int INBOX, int BUFS, bool TMA_ZERO>
struct PartCfg {
  static constexpr int kChunk = CHUNK, kCap = CAP, kStage = STAGE, kInbox = INBOX, kBufs = BUFS;
  // staging buffers cleared by a bulk copy from a zero block (no LSU wavefronts) instead of
  // shared-memory stores: measured faster for Base's large-table (PeleC-scale) CTAs, slower for Wide
  static constexpr bool kTmaZero = TMA_ZERO;
  static_assert(CHUNK % (2 * kDecodeThreads) == 0, "whole record pairs per decode thread");
  static_assert((CAP * 2) % 16 == 0, "slots must be whole 16-byte units for bulk copies");
  static_assert(STAGE >= 2 && INBOX >= 2, "the ring hand-offs need two buffers (one deadlocks)");
  static_assert(BUFS <= kPartBufs && CAP * BUFS <= kPartCap * kPartBufs, "exchange fits the reserved buffers");
  static_assert((size_t)kPartMaxCtas * CAP * 2 <= kPartZeroBytes, "the zero block covers a staging buffer");
};
#ifndef GPA_PARTW_CHUNK
#define GPA_PARTW_CHUNK 8960
#endif
#ifndef GPA_PARTW_CAP
#define GPA_PARTW_CAP 80
#endif
#ifndef GPA_PARTW_STAGE
#define GPA_PARTW_STAGE 3
#endif
#ifndef GPA_PARTW_INBOX
#define GPA_PARTW_INBOX 2
#endif
#ifndef GPA_PARTW_BUFS
#define GPA_PARTW_BUFS 8
#endif
#ifndef GPA_PARTW_MAX_SMEM
#define GPA_PARTW_MAX_SMEM (164 * 1024)
#endif
#ifndef GPA_PART_TMA_ZERO
#define GPA_PART_TMA_ZERO 1      // Base shape
#endif
#ifndef GPA_PARTW_TMA_ZERO
#define GPA_PARTW_TMA_ZERO 0     // Wide shape
#endif
using PartBase = PartCfg<kPartChunk, kPartCap, kStage, kInbox, kPartBufs, GPA_PART_TMA_ZERO>;
using PartWide = PartCfg<GPA_PARTW_CHUNK, GPA_PARTW_CAP, GPA_PARTW_STAGE, GPA_PARTW_INBOX, GPA_PARTW_BUFS,
                         GPA_PARTW_TMA_ZERO>;
constexpr size_t kWideSmemMax = GPA_PARTW_MAX_SMEM;
struct PartShape {
  uint32_t chunk, cap, stage, inbox, bufs;
};
template <class Cfg>
constexpr PartShape shape_of() {
  return PartShape{(uint32_t)Cfg::kChunk, (uint32_t)Cfg::kCap, (uint32_t)Cfg::kStage, (uint32_t)Cfg::kInbox,
                   (uint32_t)Cfg::kBufs};
}
// chunks per launch that keep every u32 table entry wrap-free until the kernel's final flush
inline uint32_t flush_every(const PartShape &c) {
  return (uint32_t)(0xffffffffull / ((uint64_t)kPartMaxCtas * c.cap * kMaxKeyCount));
}
static_assert(kConsBase + kConsThreads == kPartThreads, "warp roles cover the CTA");

__device__ __forceinline__ void named_bar(uint32_t id, uint32_t threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void red_release_add(unsigned int *p, unsigned int v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}


// shared -> global bulk copy (async proxy), tracked by this thread's bulk async-groups
// (evict-last: the exchange rows are read back by the consumers and the buffers are reused, so
// they should not be pushed out of L2 by the record stream; measured 1.6x fewer DRAM writes)
__device__ __forceinline__ void tma_bulk_store(void *gdst, const void *ssrc, uint32_t bytes) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
               "r"(smem_addr(ssrc)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// 2-D TMA tile load: box {cap keys, G rows} at (x, y) of tensor map *tm -> smem, mbarrier tx
__device__ __forceinline__ void tma_tile_load_2d(void *dst, const CUtensorMap *tm, uint32_t x, uint32_t y,
                                                 uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_addr(dst)),
      "l"(tm), "r"(x), "r"(y), "r"(smem_addr(bar))
      : "memory");
}

template <uint32_t LB, class Cfg>
__global__ void __launch_bounds__(kPartThreads, 1) k_ingest_part(PartArgs a, const __grid_constant__ CUtensorMap xmap) {
  // the exchange shape of this instantiation (shadows the Base constants of the same names)
  constexpr int kPartChunk = Cfg::kChunk, kPartCap = Cfg::kCap, kStage = Cfg::kStage, kInbox = Cfg::kInbox,
                kPartBufs = Cfg::kBufs;
  constexpr uint32_t kLocalBits = LB, kKeyMaxCount = key_max_count<LB>();
  constexpr int CHUNK = kPartChunk;
  constexpr int kDecodeRecs = CHUNK / kDecodeThreads;   // records per decode thread per chunk
#ifndef GPA_PART_BATCH
#define GPA_PART_BATCH 1
#endif
  constexpr int kDecodeBatch = GPA_PART_BATCH;
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t G = gridDim.x, me = blockIdx.x;
  const uint32_t slot_keys = G * kPartCap;                                       // keys per staging / inbox buffer
  const uint32_t ibuf_keys = ((slot_keys * 2 + 127) & ~127u) / 2;             // 128-B aligned buffers (TMA)
  uint16_t *inbox = reinterpret_cast<uint16_t *>(sm);                            // [kInbox][G src][cap]
  uint16_t *stag = inbox + kInbox * ibuf_keys;                                  // [kStage][G dst][cap]
  uint32_t *trash = reinterpret_cast<uint32_t *>(stag + kStage * ibuf_keys);    // [kTrash]
  uint32_t *cnt = trash + kTrash;                                                // [kStage][kPartMaxCtas + 8]
  uint64_t *buf_ready = reinterpret_cast<uint64_t *>(cnt + kStage * (kPartMaxCtas + 8));   // [kStage] publisher -> decoders
  uint64_t *decoded = buf_ready + kStage;                                        // [kStage]  decoders -> control
  uint64_t *inbox_full = decoded + kStage;                                       // [kInbox]  TMA -> consumers
  uint64_t *inbox_free = inbox_full + kInbox;                                    // [kInbox]  consumers -> loader
  uint64_t *stored = inbox_free + kInbox;   // [kPartBufs] control -> publisher (control runs at most
                                            // kPartBufs-1 chunks ahead: see the cons-counter wait)
  uint32_t *tab = reinterpret_cast<uint32_t *>(stored + kPartBufs);              // [bpb + kTrash]
  for (uint32_t i = tid; i < a.bpb + kTrash; i += kPartThreads) tab[i] = 0;
  for (uint32_t i = tid; i < kStage * ibuf_keys / 2; i += kPartThreads) reinterpret_cast<uint32_t *>(stag)[i] = 0;
  // bucket G is the dummy bucket of invalid / large-count records: its counter starts past the
  // slot capacity, so its records always take the rare branch
  for (uint32_t i = tid; i < kStage * (kPartMaxCtas + 8); i += kPartThreads)
    cnt[i] = i % (kPartMaxCtas + 8) == G ? kDummyCount : 0u;
  if (tid == 0) {
    for (int r = 0; r < kStage; ++r) {
      mbar_init(&buf_ready[r], 1);
      mbar_init(&decoded[r], kDecodeWarps);
    }
    for (int r = 0; r < kInbox; ++r) {
      mbar_init(&inbox_full[r], 1);
      mbar_init(&inbox_free[r], 1);
    }
    for (int r = 0; r < kPartBufs; ++r) mbar_init(&stored[r], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t per_chunk = (uint64_t)CHUNK * G;
  const uint32_t n_chunks = (uint32_t)((a.n_even + per_chunk - 1) / per_chunk);
  auto slice_len = [&](uint32_t k, uint64_t &start) -> uint32_t {
    start = (uint64_t)k * per_chunk + (uint64_t)me * CHUNK;
    return start >= a.n_even ? 0u
                             : (uint32_t)(a.n_even - start < (uint64_t)CHUNK ? a.n_even - start : (uint64_t)CHUNK);
  };
  // row (buf, src) of the exchange: G slots of kPartCap keys, one per destination; a producer
  // writes its row with one bulk store, a consumer reads its column (x = dst * cap) with one
  // 2-D TMA tile load (tensor map xmap: rows = kPartBufs * kPartMaxCtas, cols = G * cap)
  auto xrow = [&](uint32_t buf, uint32_t src) -> uint16_t * {
    return a.X + ((uint64_t)buf * kPartMaxCtas + src) * G * kPartCap;
  };
  const uint32_t twoR = 2 * a.R;
  IngestStats st{0, 0, 0};
#ifndef GPA_PART_MAXNREG   // registers per decoder thread / per other thread (20*72 + 12*40 = 32*60 <= 32*64)
#define GPA_PART_MAXNREG 72
#define GPA_PART_LOWNREG 40
#endif
#if GPA_PART_MAXNREG > 0
  // register split by warp role (setmaxnreg): the decoder warpgroups (warps 0-19) take the
  // registers the control / publisher / loader / processor warpgroups (warps 20-31) do not need,
  // so the decode keeps its addresses and keys in registers (measured 2.30 -> 2.26 ms on config 3)
  static_assert(kDecodeWarps % 4 == 0, "decoders fill whole warpgroups");
  static_assert(kDecodeWarps * GPA_PART_MAXNREG + (32 - kDecodeWarps) * GPA_PART_LOWNREG <= 32 * 64,
                "register split exceeds the CTA's register file");
  if (warp < kDecodeWarps) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(GPA_PART_MAXNREG));
  else asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(GPA_PART_LOWNREG));
#endif
  if (warp < kDecodeWarps) {
    // ======================= decoders: wait only on data (ring_full) and on a clean staging
    //                         buffer (buf_ready); decode + scatter; signal decoded
    const uint32_t dtid = tid;
    const uint32_t n_instr = a.n_instr, R = a.R, mg = a.mg, nG = 0u - G;
    const uint32_t trash_addr = smem_addr(trash + lane);
    auto load_chunk = [&](const uint4 *rs, uint32_t len, uint4 (&v)[kDecodeRecs / 2]) {
      const bool full = len == (uint32_t)CHUNK;
#pragma unroll
      for (int u = 0; u < kDecodeRecs / 2; ++u) {
        const uint32_t pair = u * kDecodeThreads + dtid;   // len is even: both records of a pair or neither
        v[u] = (full || 2 * pair < len) ? ld_stream(rs + pair) : make_uint4(0xffffffffu, 0, 0xffffffffu, 0);
      }
    };
    PT_DECL
    for (uint32_t k = 0; k < n_chunks; ++k) {
      uint64_t s0;
      const uint32_t len = slice_len(k, s0);
      const uint32_t sb = k % kStage;
      const uint32_t sg_addr = smem_addr(stag + sb * ibuf_keys), cnt_addr = smem_addr(cnt + sb * (kPartMaxCtas + 8));
      const uint4 *rs = reinterpret_cast<const uint4 *>(a.rec + s0);
      const bool full = len == (uint32_t)CHUNK;
      PT_START;
      uint4 vv[kDecodeRecs / 2];   // 16-byte streaming loads, in flight while waiting for the buffer
      load_chunk(rs, len, vv);
      mbar_wait(&buf_ready[sb], (k / kStage) & 1);
      PT_MARK(0);
      // ---- branch-free decode: bucket = pc mod G (interleaved PCs balance the load), key = local
      //      bin (pc / G) * 2R + class * R + reason | count << 13, stored at position cnt[b]++ of
      //      bucket b's zero-padded slot (invalid and padding records count in the dummy bucket G
      //      and land in a trash word; counts > 7 and slot overflow go through L2 atomics)
      uint32_t csum = 0, bads = 0, badr = 0;
      // records are processed in batches of kDecodeBatch pairs: all slot allocations (atomics) of a
      // batch are issued before its key stores, so their latencies overlap.  Validity (Q12): t =
      // flags:reason is valid iff t < R (ACT) or 0x101 <= t < 0x100 + R (LAT with a reason); then
      // class * R + reason = t - (t >> 8) * (256 - R).  Invalid records and counts > 7 go to the
      // dummy bucket G, whose counter never hands out a slot, so one compare (pos < cap) selects
      // the rare branch for them and for slot overflow; the branch re-derives which case it is.
#pragma unroll
      for (int u0 = 0; u0 < kDecodeRecs / 2; u0 += kDecodeBatch) {
        constexpr int kB = 2 * kDecodeBatch;
        uint32_t pos[kB], slot[kB];
        uint32_t key[kB];
#pragma unroll
        for (int i = 0; i < kB; ++i) {
          const int u = u0 + i / 2, h = i & 1;
          if (u >= kDecodeRecs / 2) break;
          const uint4 v = vv[u];
          const uint32_t pc = h ? v.z : v.x, w = h ? v.w : v.y;
          const uint32_t t = w >> 16, c = w & 0xffffu;
          const uint32_t tl = t - (t >> 8) * (256u - R);
          const bool fast = pc < n_instr && (t < R || t - 0x101u < R - 1u) && c <= kKeyMaxCount;
          const uint32_t q = __umulhi(pc, mg), b = q * nG + pc;
          const uint32_t be = fast ? b : G;
          key[i] = c * (1u << kLocalBits) + q * twoR + tl;
          slot[i] = sg_addr + be * (kPartCap * 2);
#ifndef GPA_ABLATE_DEC_ATOM
          asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(pos[i]) : "r"(cnt_addr + be * 4) : "memory");
#else
          pos[i] = (dtid + i) % 40u + (cnt_addr == 0xFFFFFFFFu ? be : 0u);
#endif
          csum += c;        // padding records have count 0
        }
#pragma unroll
        for (int i = 0; i < kB; ++i) {
          const int u = u0 + i / 2, h = i & 1;
          if (u >= kDecodeRecs / 2) break;
          const bool keep = pos[i] < (uint32_t)kPartCap;
          const uint32_t dst = keep ? slot[i] + pos[i] * 2 : trash_addr;
#ifndef GPA_ABLATE_DEC_STS
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(dst), "h"((unsigned short)key[i]) : "memory");
#else
          if (dst == 0xFFFFFFFFu) asm volatile("st.shared.u16 [%0], %1;" ::"r"(dst), "h"((unsigned short)key[i]) : "memory");
#endif
          if (!keep) {       // rare: an invalid record, a count > 7 or slot overflow (skew)
            const uint4 v = vv[u];
            const uint32_t pc = h ? v.z : v.x, w = h ? v.w : v.y;
            const uint32_t t = w >> 16, c = w & 0xffffu;
            if (pc < n_instr && (t < R || t - 0x101u < R - 1u)) {
              const uint32_t tl = t - (t >> 8) * (256u - R);
              atomicAdd((unsigned long long *)&a.C[(uint64_t)pc * twoR + tl], (unsigned long long)c);
            } else {
              bads += c;
              badr += (full || 2 * (u * kDecodeThreads + dtid) < len) ? 1u : 0u;   // padding is not a record
            }
          }
        }
      }
      st.valid += csum - bads;
      st.bad_samples += bads;
      st.bad_records += badr;
      // generic-proxy staging writes must be ordered before the control warp's bulk store
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&decoded[sb]);          // staging buffer handed over
      PT_MARK(2);
    }
    PT_FLUSH;
  } else if (warp == kCtrlWarp) {
    // ======================= control: one bulk store of the CTA's row per chunk, completed
    //                         stores handed to the publisher

    PT_DECL
    for (uint32_t k = 0; k < n_chunks; ++k) {
      const uint32_t sb = k % kStage, buf = k % kPartBufs;
      PT_START;
      mbar_wait(&decoded[sb], (k / kStage) & 1);        // all decoders finished chunk k
      PT_MARK(3);
      if (lane == 0) {
        // exchange buffer k%NBUF is free once every CTA drained chunk k-NBUF
        if (k >= (uint32_t)kPartBufs) spin_until(&a.sync[kPartBufs + buf], G * (k / kPartBufs));
        PT_MARK(4);
        tma_bulk_store(xrow(buf, me), stag + sb * ibuf_keys, slot_keys * 2);   // my row, all G slots
        bulk_commit();
        if (k > 0) {   // chunk k-1's store is complete: hand it to the publisher warp
          asm volatile("cp.async.bulk.wait_group 1;" ::: "memory");
          fence_proxy_async_global();
          mbar_arrive(&stored[(k - 1) % kPartBufs]);
          PT_MARK(5);
        }
      }
      __syncwarp();
    }
    PT_FLUSH;
    if (n_chunks && lane == 0) {
      bulk_wait_all();
      fence_proxy_async_global();
      mbar_arrive(&stored[(n_chunks - 1) % kPartBufs]);
    }
  } else if (warp == kPubWarp) {
    // ======================= publisher: release each stored chunk to the other CTAs, then clear
    //                         its staging buffer and counters for chunk k+kStage
    PT_DECL
    for (uint32_t r = 0; r < (uint32_t)kStage && r < n_chunks; ++r) {   // the staging buffers start clean
      if (lane == 0) mbar_arrive(&buf_ready[r]);
    }
    for (uint32_t k = 0; k < n_chunks; ++k) {
      PT_START;
      mbar_wait(&stored[k % kPartBufs], (k / kPartBufs) & 1);   // chunk k's store has completed
      PT_MARK(14);
      if (lane == 0) {
        fence_proxy_async_global();
        red_release_add(&a.sync[k % kPartBufs], 1u);   // this CTA produced chunk k
      }
      PT_MARK(15);
      if (k + kStage < n_chunks) {
        const uint32_t ob = k % kStage;
        for (uint32_t i = lane; i <= G; i += 32) cnt[ob * (kPartMaxCtas + 8) + i] = i == G ? kDummyCount : 0u;
        if constexpr (Cfg::kTmaZero) {
          // the staging buffer cleared by a bulk copy from a zero block (async proxy, no LSU
          // wavefronts); buf_ready completes when its bytes have landed
          __syncwarp();
          if (lane == 0) {
            mbar_expect_tx(&buf_ready[ob], slot_keys * 2);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr(stag + ob * ibuf_keys)),
                "l"(a.zero), "r"(slot_keys * 2), "r"(smem_addr(&buf_ready[ob]))
                : "memory");
          }
        } else {
          uint4 *z = reinterpret_cast<uint4 *>(stag + ob * ibuf_keys);
          for (uint32_t i = lane; i < slot_keys / 8; i += 32) z[i] = make_uint4(0, 0, 0, 0);
          __syncwarp();
          if (lane == 0) mbar_arrive(&buf_ready[ob]);
        }
      }
      PT_MARK(7);
    }
    PT_FLUSH;
  } else {
    // ======================= consumers: warp kLoaderWarp fetches my column of each exchange
    //                         buffer into the kInbox-deep smem inbox (one 2-D TMA tile load per
    //                         chunk, as soon as every producer published it and the slot is free);
    //                         the other warps only wait on their data and add keys to the table
    if (warp == kLoaderWarp) {
      // loads run kInbox chunks ahead; the loader alone polls the TMA completion and releases the
      // processor warps through a named barrier
      auto load = [&](uint32_t j) {
        spin_until(&a.sync[j % kPartBufs], G * (j / kPartBufs + 1));   // every producer published j
        fence_proxy_async_global();
        mbar_expect_tx(&inbox_full[j % kInbox], slot_keys * 2);
        tma_tile_load_2d(inbox + (j % kInbox) * ibuf_keys, &xmap, me * kPartCap, (j % kPartBufs) * kPartMaxCtas,
                         &inbox_full[j % kInbox]);
      };
      PT_DECL
      if (lane == 0)
        for (uint32_t j = 0; j < (uint32_t)kInbox && j < n_chunks; ++j) load(j);
      for (uint32_t j = 0; j < n_chunks; ++j) {
        PT_START;
        if (lane == 0) mbar_wait(&inbox_full[j % kInbox], (j / kInbox) & 1);
        __syncwarp();
        PT_MARK(12);
        if (j >= 1 && j - 1 + kInbox < n_chunks) {   // slot of chunk j-1 (processed already) -> chunk j-1+kInbox
          if (lane == 0) {
            mbar_wait(&inbox_free[(j - 1) % kInbox], ((j - 1) / kInbox) & 1);
            load(j - 1 + kInbox);
          }
          __syncwarp();
        }
        PT_MARK(13);
      }
      PT_FLUSH;
    } else {
      const uint32_t ctid = tid - kProcBase;
      const uint32_t tab_addr = smem_addr(tab), dummy_addr = smem_addr(tab + a.bpb + (ctid & 31));
      PT_DECL
      for (uint32_t j = 0; j < n_chunks; ++j) {
        PT_START;
        mbar_wait(&inbox_full[j % kInbox], (j / kInbox) & 1);
        PT_MARK(9);
        const uint4 *in4 = reinterpret_cast<const uint4 *>(inbox + (j % kInbox) * ibuf_keys);
#ifndef GPA_PART_PROC_ACTIVE
#define GPA_PART_PROC_ACTIVE 8
#endif
        // 8 of the 9 processor warps add keys (the ninth only joins the inbox barrier): the
        // processors have slack, and fewer of them queueing shared-memory updates shortens the
        // decoders' slot-allocation round trips (9 -> 8 warps: 2.26 -> 2.22 ms; 7: 2.23; 5: 2.38)
        constexpr uint32_t kProcActive = 32 * (GPA_PART_PROC_ACTIVE);   // threads that add keys
        static_assert(GPA_PART_PROC_ACTIVE <= kConsWarps - 1, "active processors exist");
        for (uint32_t v = ctid; v < (ctid < kProcActive ? slot_keys / 8 : 0u); v += kProcActive) {
          const uint4 kv = in4[v];
          const uint32_t w4[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const uint32_t key = (w4[e >> 1] >> ((e & 1) * 16)) & 0xffffu;
            const uint32_t c = key >> kLocalBits;
            // padding keys (c = 0) add 0 to a lane-distinct dummy word: cheaper on the shared-memory
            // pipe than a predicated (branching) update, measured
#ifdef GPA_PROC_PRED
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t@p red.shared.add.u32 [%0], %1;\n\t}" ::"r"(
                             tab_addr + (key & ((1u << kLocalBits) - 1)) * 4),
                         "r"(c)
                         : "memory");
            continue;
#endif
#ifdef GPA_PROC_SAMEADDR
            const uint32_t addr = tab_addr + (key & ((1u << kLocalBits) - 1)) * 4;   // padding: +0 to bin 0
#else
            const uint32_t addr = c ? tab_addr + (key & ((1u << kLocalBits) - 1)) * 4 : dummy_addr;
#endif
#ifndef GPA_ABLATE_PROC_RED
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(c) : "memory");
#else
            if (addr == 0xFFFFFFFFu) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(c) : "memory");
#endif
          }
        }
        PT_MARK(10);
        named_bar(kBarProc, kProcThreads);   // inbox slot j%kInbox fully read
        PT_MARK(11);
        if (ctid == 0) {
          mbar_arrive(&inbox_free[j % kInbox]);
          red_release_add(&a.sync[kPartBufs + j % kPartBufs], 1u);   // this CTA drained chunk j
        }
      }
      PT_FLUSH;
    }
  }
  __syncthreads();
  flush_stats(st, a.stats);
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

// ----------------------------------------------------------------------------- variant K
// Streams grouped by kernel launch (gpa_ingest_segments): segment s = records
// [seg_begin[s], seg_begin[s+1]) of kernel seg_kernel[s].  The record index space is cut into
// tiles of kSegTile records, tiles are dealt to the CTAs round-robin, and every (tile, segment)
// piece is counted in a shared-memory table covering only that kernel's PCs (config 4: <= 2048
// instructions x 2R bins), which is then added to C with one coalesced u64 atomic per nonzero
// bin.  Records whose pc lies outside the segment's kernel, segments of unknown kernels
// (seg_kernel >= n_kernels) and kernels too large for the table take L2 atomics: exact for any
// input.  A piece holds at most kSegTile records of count <= 65535, so u32 bins cannot wrap.
#ifndef GPA_SEG_TILE
#define GPA_SEG_TILE 32768
#endif
constexpr uint32_t kSegTile = GPA_SEG_TILE;
#ifndef GPA_SEG_THREADS
#define GPA_SEG_THREADS 512
#endif
constexpr uint32_t kSegThreads = GPA_SEG_THREADS;
#ifndef GPA_SEG_UNROLL
#define GPA_SEG_UNROLL 4
#endif
constexpr int kSegUnroll = GPA_SEG_UNROLL;   // 16-byte record loads in flight per thread

__global__ void __launch_bounds__(kSegThreads)
k_ingest_seg(const uint2 *__restrict__ rec, uint64_t n_rec, const uint64_t *__restrict__ seg_begin,
             const uint32_t *__restrict__ seg_kernel, uint32_t n_seg, uint32_t pc_base,
             const uint32_t *__restrict__ func_begin, const uint32_t *__restrict__ kernel_func_begin,
             uint32_t n_kernels, uint32_t n_instr, uint32_t R, uint32_t max_tab_bins,
             uint64_t *__restrict__ C, uint64_t *__restrict__ stats) {
  extern __shared__ uint32_t tab[];
  const uint32_t twoR = 2 * R;
  auto clampr = [&](uint64_t x) { return x < n_rec ? x : n_rec; };
  const uint64_t r0 = clampr(seg_begin[0]), r1 = clampr(seg_begin[n_seg]);
  const uint64_t n_tiles = r1 > r0 ? (r1 - r0 + kSegTile - 1) / kSegTile : 0;
  IngestStats st{0, 0, 0};
  for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const uint64_t t0 = r0 + t * kSegTile, t1 = t0 + kSegTile < r1 ? t0 + kSegTile : r1;
    // first segment overlapping the tile: the last s with seg_begin[s] <= t0
    uint32_t lo = 0, hi = n_seg;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (clampr(seg_begin[mid]) <= t0) lo = mid; else hi = mid;
    }
    for (uint32_t s = lo; s < n_seg; ++s) {
      const uint64_t b = clampr(seg_begin[s]) > t0 ? clampr(seg_begin[s]) : t0;
      const uint64_t e = clampr(seg_begin[s + 1]) < t1 ? clampr(seg_begin[s + 1]) : t1;
      if (clampr(seg_begin[s]) >= t1) break;
      if (b >= e) continue;
      const uint32_t k = seg_kernel[s];
      uint32_t p0 = 0, np = 0;
      if (k < n_kernels) {
        p0 = func_begin[kernel_func_begin[k]];
        np = func_begin[kernel_func_begin[k + 1]] - p0;
      }
      const bool use_tab = np > 0 && np * twoR <= max_tab_bins;
      const uint32_t nb = use_tab ? np * twoR : 0;
      __syncthreads();                                   // previous piece's flush read the table
      for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) tab[i] = 0;
      __syncthreads();
      auto add = [&](uint32_t pc, uint32_t w) {
        uint32_t bin, cnt;
        if (decode(pc - pc_base, w, n_instr, R, bin, cnt)) {
          st.valid += cnt;
          const uint32_t lb = bin - p0 * twoR;           // wraps past nb when pc < p0
          if (lb < nb) atomicAdd(&tab[lb], cnt);
          else atomicAdd((unsigned long long *)&C[bin], (unsigned long long)cnt);
        } else {
          st.bad_records += 1;
          st.bad_samples += cnt;
        }
      };
      // 16-byte pairs over the aligned body of [b, e); a head / odd tail record by thread 0
      const uint64_t hb = ((uintptr_t)(rec + b) & 15u) ? 1 : 0;
      const uint64_t body = (e - b - hb) >> 1;
      const uint4 *r16 = reinterpret_cast<const uint4 *>(rec + b + hb);
      uint64_t i = threadIdx.x;
      for (; i + (kSegUnroll - 1) * blockDim.x < body; i += kSegUnroll * blockDim.x) {   // loads in flight
        uint4 v[kSegUnroll];
#pragma unroll
        for (int u = 0; u < kSegUnroll; ++u) v[u] = ld_stream(r16 + i + u * blockDim.x);
#pragma unroll
        for (int u = 0; u < kSegUnroll; ++u) {
          add(v[u].x, v[u].y);
          add(v[u].z, v[u].w);
        }
      }
      for (; i < body; i += blockDim.x) {
        const uint4 v = ld_stream(r16 + i);
        add(v.x, v.y);
        add(v.z, v.w);
      }
      if (threadIdx.x == 0) {
        if (hb) { const uint2 v = ld_stream8(rec + b); add(v.x, v.y); }
        if ((e - b - hb) & 1) { const uint2 v = ld_stream8(rec + e - 1); add(v.x, v.y); }
      }
      __syncthreads();
      uint64_t *dst = C + (uint64_t)p0 * twoR;
      for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x)
        if (tab[i]) atomicAdd((unsigned long long *)&dst[i], (unsigned long long)tab[i]);
    }
  }
  flush_stats(st, stats);
}

}  // namespace

// 2-D view of the exchange buffers for the consumers' column loads: element = 2-byte key,
// cols = G * cap (one row = a producer's G slots), rows = kPartBufs * kPartMaxCtas, box = {cap, G}
static cudaError_t make_exchange_map(CUtensorMap *tm, void *X, uint32_t G, const PartShape &c) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
    encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  const cuuint64_t dims[2] = {(cuuint64_t)G * c.cap, (cuuint64_t)c.bufs * kPartMaxCtas};
  const cuuint64_t strides[1] = {(cuuint64_t)G * c.cap * 2};
  const cuuint32_t box[2] = {c.cap, G};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, X, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

#ifdef GPA_PART_TIMING
extern "C" int gpa_debug_read_timing(unsigned long long *out) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(out, g_part_timing, sizeof(g_part_timing));
}
#endif

static size_t part_smem_bytes(uint32_t bpb, uint32_t G, const PartShape &c) {
  const size_t ibuf = ((size_t)G * c.cap * 2 + 127) & ~(size_t)127;
  return (c.inbox + c.stage) * ibuf + kTrash * 4 + c.stage * (kPartMaxCtas + 8) * 4 +
         (2 * c.stage + c.bufs + 2 * c.inbox) * 8 + (size_t)(bpb + kTrash) * 4;
}
size_t part_smem_bytes(uint32_t bpb, uint32_t G) { return part_smem_bytes(bpb, G, shape_of<PartBase>()); }

static uint32_t part_grid(int n_sms) { return (uint32_t)std::min(n_sms, kPartMaxCtas); }

// buckets: PCs pc = q*G + b go to CTA b (ppb = ceil(n/G) PCs, ppb * 2R bins); 16-bit local bins
static bool part_shape(const DevProgram &p, int n_sms, uint32_t &G, uint32_t &ppb, uint32_t &bpb) {
  if (n_sms < 1) return false;
  G = part_grid(n_sms);
  ppb = (p.n + G - 1) / G;
  bpb = ppb * 2 * p.R;
  return bpb < (1u << kMaxLocalBits) && G <= 256;   // 2-byte keys: <= 15-bit local bins; TMA box <= 256
}

bool part_feasible(const DevProgram &p, int n_sms, size_t smem_optin) {   // Base is the smaller shape
  uint32_t G, ppb, bpb;
  return part_shape(p, n_sms, G, ppb, bpb) && part_smem_bytes(bpb, G, shape_of<PartBase>()) + 256 <= smem_optin;
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
    if (ingest_smem_bytes(p) > smem_optin || ingest_smem_bytes(p) > kSmemTableMax) return cudaErrorInvalidValue;
    const size_t smem = kSmemU16 ? ingest_smem_bytes(p) / 2 : ingest_smem_bytes(p);
    grid = std::min<uint32_t>(grid, kMaxIngestCtas);
    cudaError_t e = cudaFuncSetAttribute(k_ingest<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_ingest<true><<<grid, kIngestThreads, smem, s>>>(rec, n, head, p.n, p.R, bins, p.C, p.partials, p.stats);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const uint32_t groups = (grid + kReduceGroup - 1) / kReduceGroup;
    const uint32_t words = kSmemU16 ? bins / 2 : bins;
    const uint32_t rgrid = std::max<uint32_t>(1, std::min<uint32_t>((words + 255) / 256, 4 * n_sms));
    return launch_pdl(p.n, k_ingest_reduce, dim3(rgrid, groups), dim3(256), 0, s, (const uint32_t *)p.partials, grid,
                      bins, p.C);
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
    a.X = reinterpret_cast<uint16_t *>(p.part_x);
    a.sync = p.part_sync;
    a.zero = p.part_zero;
#ifndef GPA_PART_FORCE_LB
#define GPA_PART_FORCE_LB 0   // tuning probe: force the local-bin width
#endif
    const uint32_t lbits = GPA_PART_FORCE_LB ? GPA_PART_FORCE_LB
                                             : std::max<uint32_t>(kMinLocalBits, 32u - __builtin_clz(bpb));   // bpb < 2^lbits
#ifndef GPA_PART_WIDE
#define GPA_PART_WIDE 1
#endif
    // the Wide exchange shape when the CTA stays within kWideSmemMax with it, else Base
    const PartShape wide_c = shape_of<PartWide>(), base_c = shape_of<PartBase>();
    const size_t smem_w = part_smem_bytes(a.bpb, G, wide_c);
    const bool use_wide = GPA_PART_WIDE && smem_w <= kWideSmemMax && smem_w + 256 <= smem_optin;
    const PartShape &c = use_wide ? wide_c : base_c;
    const void *kern =
        use_wide ? (lbits == 13 ? (const void *)k_ingest_part<13, PartWide>
                                : lbits == 14 ? (const void *)k_ingest_part<14, PartWide> : (const void *)k_ingest_part<15, PartWide>)
                 : (lbits == 13 ? (const void *)k_ingest_part<13, PartBase>
                                : lbits == 14 ? (const void *)k_ingest_part<14, PartBase> : (const void *)k_ingest_part<15, PartBase>);
    const size_t smem = part_smem_bytes(a.bpb, G, c);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(p.part_sync, 0, 2 * c.bufs * sizeof(unsigned int), s);
    if (e != cudaSuccess) return e;
    if (head || ((n - head) & 1ull)) {
      k_ingest_edges<<<1, 32, 0, s>>>(rec, n, head, p.n, p.R, p.C, p.stats);
      e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    if (a.n_even == 0) return cudaSuccess;
    CUtensorMap xmap;
    e = make_exchange_map(&xmap, p.part_x, G, c);
    if (e != cudaSuccess) return e;
    // a launch runs at most flush_every(c) chunks, so no u32 table entry can wrap before the
    // kernel's final flush into the u64 table (> 6.5e10 records: several launches)
    // (GPA_PART_LAUNCH_CHUNKS lowers the limit: a test hook that exercises the split on small streams)
    uint64_t launch_chunks = flush_every(c);
    if (const char *env = getenv("GPA_PART_LAUNCH_CHUNKS")) {
      const unsigned long long v = strtoull(env, nullptr, 10);
      if (v > 0 && v < launch_chunks) launch_chunks = v;
    }
    const uint64_t body = a.n_even, max_launch = launch_chunks * G * c.chunk;
    const uint2 *base = a.rec;
    for (uint64_t off = 0; off < body; off += max_launch) {
      a.rec = base + off;
      a.n_even = std::min<uint64_t>(max_launch, body - off);
      if (off > 0) {
        e = cudaMemsetAsync(p.part_sync, 0, 2 * c.bufs * sizeof(unsigned int), s);
        if (e != cudaSuccess) return e;
      }
      void *args[] = {&a, &xmap};
      e = cudaLaunchCooperativeKernel(kern, dim3(G), dim3(kPartThreads), args, smem, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  return cudaErrorNotSupported;
}

cudaError_t launch_ingest_segments(const DevProgram &p, const void *records, uint64_t n, const uint64_t *seg_begin,
                                   const uint32_t *seg_kernel, uint32_t n_seg, uint32_t pc_base, uint32_t max_tab_bins,
                                   int n_sms, cudaStream_t s) {
#ifndef GPA_SEG_SMEM_PAD
#define GPA_SEG_SMEM_PAD 0   // tuning probe: extra dynamic shared memory per CTA (fewer CTAs per SM)
#endif
  const size_t smem = (size_t)max_tab_bins * 4 + GPA_SEG_SMEM_PAD;
  cudaError_t e = cudaFuncSetAttribute(k_ingest_seg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ingest_seg, kSegThreads, smem);
  const uint32_t grid = (uint32_t)std::max(1, n_sms * std::max(1, per_sm));
  k_ingest_seg<<<grid, kSegThreads, smem, s>>>((const uint2 *)records, n, seg_begin, seg_kernel, n_seg, pc_base,
                                               p.func_begin, p.kernel_func_begin, p.n_kernels, p.n, p.R,
                                               max_tab_bins, p.C, p.stats);
  return cudaGetLastError();
}

}  // namespace gpa

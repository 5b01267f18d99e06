// ingest.cu -- row a1: PC-sample records -> C[pc][class][reason].
//
// Variant S (k_ingest_smem): the whole count table fits one CTA's shared memory (n*2R*4 B
//   <= 227 KB, e.g. config 2).  A persistent grid of one 1024-thread CTA per SM streams the
//   records with 16-byte non-allocating loads (4 outstanding per thread), validates each
//   record and adds its count to a CTA-private u32 table with shared-memory atomics; u32
//   wrap-around is detected from the atomic's return value and carried into the u64 table.
//   CTA tables are written out coalesced and summed per bin by k_ingest_reduce (no global
//   atomics on the hot path, deterministic).
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

}  // namespace

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
  return cudaErrorNotSupported;
}

}  // namespace gpa

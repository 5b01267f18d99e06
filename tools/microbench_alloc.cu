// Exploratory microbenchmark (NOT the product path): cost of the producer-side slot allocation +
// key store of a partitioned histogram, per 32 records (one warp instruction's worth), one
// 1024-thread CTA per SM, random buckets:
//   A  (current)  G=148 buckets: atom.shared.add(cnt[b], 1) per lane, st.u16 at slot b, pos
//   B  (match)    P=32 buckets: match.any -> leader atom(cnt[p], n) -> shfl base -> st.u16
//   C  (ballot)   P=32 buckets: 5 ballots give the peer mask, then as B
//   D  (match37)  P=37 buckets, as B
// Reports cycles per warp-iteration per SM (all 32 warps busy).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mba tools/microbench_alloc.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int MODE, int NB, int CAP>
__global__ void __launch_bounds__(1024, 1) k_alloc(int iters, unsigned long long *cyc, uint32_t *sink) {
  extern __shared__ uint32_t sm[];
  uint32_t *cnt = sm;                                   // [NB] (+pad)
  uint16_t *slot = reinterpret_cast<uint16_t *>(sm + 64);   // [NB][CAP]
  for (uint32_t i = threadIdx.x; i < 64 + NB * CAP / 2 + 64; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t cnt_addr = (uint32_t)__cvta_generic_to_shared(cnt);
  const uint32_t slot_addr = (uint32_t)__cvta_generic_to_shared(slot);
  uint32_t h = hash32(threadIdx.x * 7919u + blockIdx.x * 104729u);
  uint32_t acc = 0;
  const unsigned long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < iters; ++it) {
    h = h * 1664525u + 1013904223u;
    const uint32_t b = (uint32_t)(((uint64_t)(h >> 8) * NB) >> 24);
    const uint16_t key = (uint16_t)(h >> 3);
    uint32_t pos;
    if (MODE == 0) {
      asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(pos) : "r"(cnt_addr + b * 4) : "memory");
    } else {
      uint32_t peers;
      if (MODE == 2) {
        peers = 0xffffffffu;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const uint32_t bal = __ballot_sync(0xffffffffu, (b >> k) & 1u);
          peers &= ((b >> k) & 1u) ? bal : ~bal;
        }
      } else {
        peers = __match_any_sync(0xffffffffu, b);
      }
      const uint32_t leader = __ffs(peers) - 1;
      const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
      uint32_t base = 0;
      if (lane == leader)
        asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(base) : "r"(cnt_addr + b * 4), "r"((uint32_t)__popc(peers)) : "memory");
      base = __shfl_sync(0xffffffffu, base, leader);
      pos = base + rank;
    }
    const uint32_t p = pos % CAP;
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(slot_addr + (b * CAP + p) * 2), "h"(key) : "memory");
    acc += pos;
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cyc, t1 - t0);
  if (acc == 0xdeadbeef) sink[0] = acc;
}

template <int MODE, int NB, int CAP>
void run(const char *name, int n_sms) {
  unsigned long long *cyc;
  uint32_t *sink;
  CK(cudaMalloc(&cyc, 8));
  CK(cudaMalloc(&sink, 4));
  const int iters = 4096;
  const size_t smem = (64 + NB * CAP / 2 + 64) * 4;
  CK(cudaFuncSetAttribute(k_alloc<MODE, NB, CAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaMemset(cyc, 0, 8));
    k_alloc<MODE, NB, CAP><<<n_sms, 1024, smem>>>(iters, cyc, sink);
    CK(cudaDeviceSynchronize());
  }
  unsigned long long c;
  CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
  const double per_sm = (double)c / n_sms;   // loop cycles of one CTA (all 32 warps ran iters iterations)
  printf("%-10s NB=%3d cap=%3d  %.2f cycles per warp-iteration per SM\n", name, NB, CAP, per_sm / iters / 32.0);
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  int n_sms;
  CK(cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, 0));
  run<0, 148, 56>("A-atom148", n_sms);
  run<1, 32, 240>("B-match32", n_sms);
  run<2, 32, 240>("C-ballot32", n_sms);
  run<1, 37, 210>("D-match37", n_sms);
  run<0, 32, 240>("E-atom32", n_sms);
  return 0;
}

// Exploratory microbenchmark (NOT the product path): per-SM throughput of the shared-memory
// operations the partitioned ingest is built from, one CTA of 1024 threads per SM, table of
// `words` u32 in shared memory, random (hashed) addresses:
//   red     : red.shared.add.u32 (no return)              -- consumer table update
//   atom    : atom.shared.add.u32 (returns old)            -- producer slot allocation
//   sts16   : st.shared.u16                                -- producer key store
//   redhalf : red with half the lanes predicated off (branch) -- padding skip
//   red2    : red.shared.add.u32 to 2*lane-distinct banks (conflict-free)
//   redv2   : red.shared.add.v2? (not in PTX for u32) -> atom on u64 pairs
// Reports lane-operations per cycle per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbs tools/microbench_smem.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int OP>
__global__ void __launch_bounds__(1024, 1) k_op(uint32_t words, int iters, unsigned long long *cyc, uint32_t *sink) {
  extern __shared__ uint32_t tab[];
  for (uint32_t i = threadIdx.x; i < words + 64; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tab);
  uint32_t acc = 0;
  uint32_t h = hash32(threadIdx.x * 7919u + blockIdx.x * 104729u);
  const unsigned long long t0 = clock64();
#pragma unroll 8
  for (int it = 0; it < iters; ++it) {
    h = h * 1664525u + 1013904223u;
    const uint32_t idx = (uint32_t)(((uint64_t)(h >> 8) * words) >> 24);
    const uint32_t addr = base + idx * 4;
    if (OP == 0) {
      asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(1u) : "memory");
    } else if (OP == 1) {
      uint32_t r;
      asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(r) : "r"(addr) : "memory");
      acc += r;
    } else if (OP == 2) {
      asm volatile("st.shared.u16 [%0], %1;" ::"r"(base + idx * 2), "h"((unsigned short)h) : "memory");
    } else if (OP == 3) {
      if (h & 0x80000000u) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(1u) : "memory");
    } else if (OP == 4) {
      const uint32_t a2 = base + (((idx & ~31u) | (threadIdx.x & 31)) % words) * 4;   // conflict-free banks
      asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a2), "r"(1u) : "memory");
    } else if (OP == 5) {
      // dummy redirect for half of the lanes (the product's padding path)
      const uint32_t a2 = (h & 0x80000000u) ? addr : base + (words + (threadIdx.x & 31)) * 4;
      asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a2), "r"(1u) : "memory");
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cyc, t1 - t0);
  if (acc == 0xdeadbeef) sink[0] = acc;
}

template <int OP>
void run(const char *name, uint32_t words, int n_sms) {
  unsigned long long *cyc;
  uint32_t *sink;
  CK(cudaMalloc(&cyc, 8));
  CK(cudaMalloc(&sink, 4));
  const int iters = 4096;
  const size_t smem = (words + 64) * 4;
  CK(cudaFuncSetAttribute(k_op<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaMemset(cyc, 0, 8));
    k_op<OP><<<n_sms, 1024, smem>>>(words, iters, cyc, sink);
    CK(cudaDeviceSynchronize());
  }
  unsigned long long c;
  CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
  const double per_sm = (double)c / n_sms;
  const double lanes = 1024.0 * iters;
  printf("%-8s words=%6u  %.3f lane-ops/cycle/SM  (%.2f cycles per warp-instr)\n", name, words, lanes / per_sm,
         per_sm / (lanes / 32));
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  int n_sms;
  CK(cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, 0));
  for (uint32_t words : {6084u, 24000u, 49000u}) {
    run<0>("red", words, n_sms);
    run<1>("atom", words, n_sms);
    run<2>("sts16", words, n_sms);
    run<3>("redhalf", words, n_sms);
    run<4>("redcf", words, n_sms);
    run<5>("reddum", words, n_sms);
  }
  return 0;
}

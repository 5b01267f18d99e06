// Exploratory microbenchmark (NOT the product path): throughput of distributed-shared-memory
// reductions (red.shared::cluster.add.u32, no return) for a table split across a cluster,
// fed by a streaming read of 8-byte records.  Compare with atomicAdd through a generic pointer.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/mbd tools/microbench_dsmem.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void gen(uint2 *rec, size_t n, uint32_t n_pc) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t u = mix64(i * 0x632BE59BD9B4E019ull + 17);
    uint32_t pc = (uint32_t)(((u & 0xffffffffull) * n_pc) >> 32);
    uint32_t reason = (uint32_t)((u >> 40) % 9);
    uint32_t lat = (uint32_t)((u >> 50) & 1);
    if (lat && reason == 0) reason = 1;
    rec[i] = make_uint2(pc, 1u | (reason << 16) | (lat << 24));
  }
}
__device__ __forceinline__ uint4 ldcs(const uint4 *p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void red_cluster(uint32_t cta, uint32_t local_off_bytes, uint32_t base, uint32_t v) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(base + local_off_bytes), "r"(cta));
  asm volatile("red.shared::cluster.add.u32 [%0], %1;" ::"r"(remote), "r"(v) : "memory");
}

// bin b -> CTA b % CS, slot b / CS ; MODE 0: red.shared::cluster via mapa; MODE 1: local only (b % CS forced to self)
template <int CS, int MODE>
__global__ void k_dsmem(const uint4 *rec, size_t n16, uint32_t slot_bins, unsigned long long *table) {
  extern __shared__ uint32_t tab[];
  cg::cluster_group cluster = cg::this_cluster();
  for (uint32_t b = threadIdx.x; b < slot_bins; b += blockDim.x) tab[b] = 0;
  cluster.sync();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tab);
  const uint32_t me = cluster.block_rank();
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  constexpr int U = 4;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldcs(rec + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t b0 = v[u].x * 18u + ((v[u].y >> 24) & 1u) * 9u + ((v[u].y >> 16) & 0xffu);
      uint32_t b1 = v[u].z * 18u + ((v[u].w >> 24) & 1u) * 9u + ((v[u].w >> 16) & 0xffu);
      uint32_t c0 = MODE ? me : b0 % CS, c1 = MODE ? me : b1 % CS;
      red_cluster(c0, (b0 / CS) * 4, base, v[u].y & 0xffffu);
      red_cluster(c1, (b1 / CS) * 4, base, v[u].w & 0xffffu);
    }
  }
  cluster.sync();
  for (uint32_t b = threadIdx.x; b < slot_bins; b += blockDim.x)
    if (tab[b]) atomicAdd(&table[(size_t)b * CS + me], (unsigned long long)tab[b]);
}

template <int CS, int MODE>
void run(const uint2 *rec, size_t n, uint32_t bins, unsigned long long *table, int sms, int threads) {
  uint32_t slot = (bins + CS - 1) / CS;
  size_t sm = slot * 4;
  auto kern = k_dsmem<CS, MODE>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  if (CS > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = sm; cfg.attrs = at; cfg.numAttrs = 1;
  cfg.gridDim = dim3(CS);
  int ncl = 0;
  CK(cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg));
  cfg.gridDim = dim3(ncl * CS);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  CK(cudaLaunchKernelEx(&cfg, kern, (const uint4 *)rec, n / 2, slot, table));
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    CK(cudaLaunchKernelEx(&cfg, kern, (const uint4 *)rec, n / 2, slot, table));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf("CS=%2d mode=%d threads=%4d clusters=%3d smem=%6zu  %8.3f ms  %7.1f GB/s  %.3e rec/s\n", CS, MODE, threads, ncl,
         sm, best, n * 8.0 / best / 1e6, n / best * 1e3);
}

int main(int argc, char **argv) {
  size_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 500000000ull;
  int sms = 148;
  uint2 *rec; CK(cudaMalloc(&rec, n * 8));
  unsigned long long *table; CK(cudaMalloc(&table, 64ull << 20));
  for (uint32_t npc : {50000u, 2000u}) {
    gen<<<sms * 8, 512>>>(rec, n, npc); CK(cudaDeviceSynchronize());
    uint32_t bins = npc * 18;
    printf("--- n_pc=%u bins=%u\n", npc, bins);
    run<16, 0>(rec, n, bins, table, sms, 1024);
    run<16, 0>(rec, n, bins, table, sms, 512);
    run<16, 1>(rec, n, bins, table, sms, 1024);
    if (bins <= 8 * 56000) { run<8, 0>(rec, n, bins, table, sms, 1024); run<8, 1>(rec, n, bins, table, sms, 1024); }
    if (bins <= 4 * 56000) { run<4, 0>(rec, n, bins, table, sms, 1024); run<2, 0>(rec, n, bins, table, sms, 1024); }
  }
  return 0;
}

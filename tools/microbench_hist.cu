// Exploratory microbenchmark (NOT the product path): which histogram primitive can
// keep up with an HBM-rate stream of 8-byte PC-sample records on sm_100a?
//   read    : plain streaming read (roofline calibration)
//   smem    : CTA-private shared-memory table, ATOMS per record (fits config-2 tables)
//   red32/64: L2-resident global table, RED.E.ADD per record (config-3 tables)
//   dsmem   : table split over a thread-block cluster, remote red.shared::cluster
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o mb tools/microbench_hist.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void gen(uint2* rec, size_t n, uint32_t n_pc, uint32_t skew) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t u = mix64(i * 0x632BE59BD9B4E019ull + 17);
    uint32_t pc = (uint32_t)(((u & 0xffffffffull) * n_pc) >> 32);
    if (skew) pc = (uint32_t)((((u & 0xffffffffull) * ((u >> 32) & 0xffff)) >> 32) * n_pc >> 16);
    uint32_t reason = (uint32_t)((u >> 40) % 9);
    uint32_t lat = (uint32_t)((u >> 50) & 1);
    if (lat && reason == 0) reason = 1;
    rec[i] = make_uint2(pc, 1u | (reason << 16) | (lat << 24));
  }
}

__device__ __forceinline__ uint4 ldcs(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t binof(uint32_t pc, uint32_t w) {
  return pc * 18u + ((w >> 24) & 1u) * 9u + ((w >> 16) & 0xffu);
}

constexpr int U = 4;

__global__ void k_read(const uint4* rec, size_t n16, unsigned long long* out) {
  uint32_t acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldcs(rec + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n16; i += stride) { uint4 v = ldcs(rec + i); acc += v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x12345678u) atomicAdd(out, 1ull);
}

__global__ void k_smem(const uint4* rec, size_t n16, uint32_t bins, unsigned long long* table) {
  extern __shared__ uint32_t tab[];
  for (uint32_t b = threadIdx.x; b < bins; b += blockDim.x) tab[b] = 0;
  __syncthreads();
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldcs(rec + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      atomicAdd(&tab[binof(v[u].x, v[u].y)], v[u].y & 0xffffu);
      atomicAdd(&tab[binof(v[u].z, v[u].w)], v[u].w & 0xffffu);
    }
  }
  for (; i < n16; i += stride) {
    uint4 v = ldcs(rec + i);
    atomicAdd(&tab[binof(v.x, v.y)], v.y & 0xffffu);
    atomicAdd(&tab[binof(v.z, v.w)], v.w & 0xffffu);
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < bins; b += blockDim.x)
    if (tab[b]) atomicAdd(&table[b], (unsigned long long)tab[b]);
}

template <typename T>
__global__ void k_red(const uint4* rec, size_t n16, T* table) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldcs(rec + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      atomicAdd(&table[binof(v[u].x, v[u].y)], (T)(v[u].y & 0xffffu));
      atomicAdd(&table[binof(v[u].z, v[u].w)], (T)(v[u].w & 0xffffu));
    }
  }
  for (; i < n16; i += stride) {
    uint4 v = ldcs(rec + i);
    atomicAdd(&table[binof(v.x, v.y)], (T)(v.y & 0xffffu));
    atomicAdd(&table[binof(v.z, v.w)], (T)(v.w & 0xffffu));
  }
}

// cluster-distributed table: bin b lives in CTA (b % CS) at slot b / CS.
template <int CS>
__global__ void k_dsmem(const uint4* rec, size_t n16, uint32_t slot_bins, unsigned long long* table) {
  extern __shared__ uint32_t tab[];
  cg::cluster_group cluster = cg::this_cluster();
  for (uint32_t b = threadIdx.x; b < slot_bins; b += blockDim.x) tab[b] = 0;
  cluster.sync();
  uint32_t* remote[CS];
#pragma unroll
  for (int c = 0; c < CS; ++c) remote[c] = cluster.map_shared_rank(tab, c);
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i < n16; i += stride) {
    uint4 v = ldcs(rec + i);
    uint32_t b0 = binof(v.x, v.y), b1 = binof(v.z, v.w);
    atomicAdd(remote[b0 % CS] + b0 / CS, v.y & 0xffffu);
    atomicAdd(remote[b1 % CS] + b1 / CS, v.w & 0xffffu);
  }
  cluster.sync();
  uint32_t me = cluster.block_rank();
  for (uint32_t b = threadIdx.x; b < slot_bins; b += blockDim.x)
    if (tab[b]) atomicAdd(&table[(size_t)b * CS + me], (unsigned long long)tab[b]);
}

int main(int argc, char** argv) {
  size_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 1000000000ull;
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  printf("device %s sms %d smemOptin %zu l2 %d\n", p.name, sms, p.sharedMemPerBlockOptin, p.l2CacheSize);
  uint2* rec; CK(cudaMalloc(&rec, n * 8));
  unsigned long long* table; CK(cudaMalloc(&table, 64ull << 20));
  unsigned int* t32 = (unsigned int*)table;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  size_t n16 = n / 2;
  double bytes = n * 8.0;
  auto report = [&](const char* name, float ms) {
    printf("%-28s %8.3f ms  %8.1f GB/s  %.3e samples/s\n", name, ms, bytes / ms / 1e6, n / ms * 1e3);
  };
  auto timeit = [&](auto launch) {
    launch(); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    CK(cudaGetLastError());
    return best;
  };
  for (int skew = 0; skew < 2; ++skew) {
    for (uint32_t npc : {2000u, 50000u}) {
      gen<<<sms * 8, 512>>>(rec, n, npc, skew); CK(cudaDeviceSynchronize());
      uint32_t bins = npc * 18;
      printf("--- n_pc=%u bins=%u skew=%d\n", npc, bins, skew);
      for (int mult : {1, 2, 4}) {
        char nm[64]; snprintf(nm, 64, "read g=%dx%d", sms * mult, 512);
        report(nm, timeit([&] { k_read<<<sms * mult, 512>>>((const uint4*)rec, n16, table); }));
      }
      if (bins * 4 <= 200 * 1024) {
        size_t sm = bins * 4;
        CK(cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        for (int th : {512, 1024}) {
          char nm[64]; snprintf(nm, 64, "smem g=%d t=%d", sms, th);
          report(nm, timeit([&] { k_smem<<<sms, th, sm>>>((const uint4*)rec, n16, bins, table); }));
        }
      }
      for (int mult : {2, 4, 8}) {
        char nm[64]; snprintf(nm, 64, "red32 g=%dx512", sms * mult);
        report(nm, timeit([&] { k_red<unsigned int><<<sms * mult, 512>>>((const uint4*)rec, n16, t32); }));
        snprintf(nm, 64, "red64 g=%dx512", sms * mult);
        report(nm, timeit([&] { k_red<unsigned long long><<<sms * mult, 512>>>((const uint4*)rec, n16, table); }));
      }
      {
        constexpr int CS = 16;
        uint32_t slot = (bins + CS - 1) / CS;
        size_t sm = slot * 4;
        if (sm <= 220 * 1024) {
          CK(cudaFuncSetAttribute(k_dsmem<CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
          CK(cudaFuncSetAttribute(k_dsmem<CS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3((sms / CS) * CS); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = sm;
          cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = CS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
          cfg.attrs = at; cfg.numAttrs = 1;
          int ncl = 0; cudaOccupancyMaxActiveClusters(&ncl, k_dsmem<CS>, &cfg);
          printf("dsmem16 max active clusters %d\n", ncl);
          report("dsmem16 t=1024", timeit([&] { CK(cudaLaunchKernelEx(&cfg, k_dsmem<CS>, (const uint4*)rec, n16, slot, table)); }));
        }
      }
      {
        constexpr int CS = 8;
        uint32_t slot = (bins + CS - 1) / CS;
        size_t sm = slot * 4;
        if (sm <= 220 * 1024) {
          CK(cudaFuncSetAttribute(k_dsmem<CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3((sms / CS) * CS); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = sm;
          cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = CS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
          cfg.attrs = at; cfg.numAttrs = 1;
          report("dsmem8 t=1024", timeit([&] { CK(cudaLaunchKernelEx(&cfg, k_dsmem<CS>, (const uint4*)rec, n16, slot, table)); }));
        }
      }
    }
  }
  return 0;
}

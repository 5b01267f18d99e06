// gen_stream.cu -- host and device entry points of the seeded record generator.
// Input generation only (see gen_core.h); not part of GPA's hot path and never timed.
#include "gen_core.h"
#include <cuda_runtime.h>

extern "C" {

// Host: records [k0, k0 + n) into out (n * 8 bytes).
int gg_generate_host(const gg_stream_params *p, uint64_t k0, uint64_t n, uint64_t *out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = gg_record(p, k0 + i);
  return 0;
}

}  // extern "C"

__global__ void gg_generate_kernel(gg_stream_params p, uint64_t k0, uint64_t n, uint64_t *out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = gg_record(&p, k0 + i);
}

extern "C" {

// Device: all table pointers in *p are device pointers; out is a device buffer.
int gg_generate_device(const gg_stream_params *p, uint64_t k0, uint64_t n, uint64_t *out,
                       void *stream) {
  if (n == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  gg_generate_kernel<<<sms * 8, 256, 0, (cudaStream_t)stream>>>(*p, k0, n, out);
  return (int)cudaGetLastError();
}

}  // extern "C"

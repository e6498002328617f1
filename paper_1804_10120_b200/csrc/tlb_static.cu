// Statically compiled (nvcc, sm_100a) helper kernels of libtlb200.
//
// tlb_fill_uniform: counter-based synthetic inputs.  The reference seeds
// fixtures with np.random.default_rng(0xC0FFEE).uniform(0, 1) in field
// declaration order (pkg/src/tlang/bench.py:72-87); that stream cannot be
// produced on the device, and at 2^28 points not on the
// host either.  Here every value is a pure function of
// (seed, stream_id, index), so any slab can be regenerated on the host
// (oracle/counter_rng.py) for a slab-sampled parity check, and a grid's
// values do not depend on how it is partitioned across GPUs.

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/tlb200.h"

namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// 2 doubles (16 B) per thread per step, grid-stride
__global__ void __launch_bounds__(256) fill_uniform_kernel(double* __restrict__ dst, long long n,
                                                           uint64_t key, long long offset) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t h = mix64(key + (uint64_t)(offset + i + 1) * kGamma);
    dst[i] = (double)(h >> 11) * 0x1.0p-53;
  }
}

// FP64 throughput probe for the flop side of the roofline.  The fused
// kernels are compiled without FMA contraction (bit-exact parity), so their
// flops are separate DMUL/DADD instructions: the probe times exactly that
// mix — 8 independent mul+add chains per thread (__dmul_rn/__dadd_rn are
// never contracted), 2 flops per chain step.
__global__ void __launch_bounds__(256) fp64_probe_kernel(double* __restrict__ out, int iters) {
  double a[8], m = 1.0 + 1e-12 * threadIdx.x, c = 1e-9;
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1.0 + k * 1e-3 + blockIdx.x * 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __dadd_rn(__dmul_rn(a[k], m), c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 0.123456789) out[0] = s;  // keeps the chains live; never true in practice
}

}  // namespace

__attribute__((visibility("hidden"))) void tlb_internal_set_error(const char* msg);  // tlb_runtime.cpp

extern "C" int tlb_fp64_probe(double* out, int blocks, int iters, void* stream) {
  if (blocks < 1 || iters < 1) return 0;
  fp64_probe_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(out, iters);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    tlb_internal_set_error(cudaGetErrorString(e));
    return 1;
  }
  return 0;
}

extern "C" int tlb_fill_uniform(double* dst, long long n, unsigned long long seed,
                                unsigned long long stream_id, long long offset, void* stream) {
  if (n <= 0) return 0;
  const uint64_t key = mix64(seed ^ mix64(stream_id + kGamma));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long blocks = (n + 255) / 256;
  long long cap = (long long)sms * 8 * 4;
  if (blocks > cap) blocks = cap;
  fill_uniform_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(dst, n, key, offset);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    tlb_internal_set_error(cudaGetErrorString(e));
    return 1;
  }
  return 0;
}

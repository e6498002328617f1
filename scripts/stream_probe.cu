// stream_probe.cu — device streaming ceilings on one B200 for the roofline
// discussion of the fused P2 kernel: how fast can THIS part
// move bytes for (a) pure reads through LDG.128, (b) pure reads through the
// TMA bulk-copy engine into a shared-memory ring, (c) pure writes, and
// (d) the P2 byte mix (40 read streams : 24 write streams) with no
// arithmetic, plain per-point streaming as in tlk_flat_v2.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//        -o scripts/_probe/stream_probe.so scripts/stream_probe.cu
// Driven by scripts/stream_probe.py (ctypes; raw device pointers + stream).
#include <cuda_runtime.h>
#include <stdint.h>

template <int U>
__global__ void __launch_bounds__(256) probe_read(const double2* __restrict__ a, long long n2,
                                                  double* out) {
  double2 acc = make_double2(0.0, 0.0);
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                   : "=d"(v[u].x), "=d"(v[u].y) : "l"(a + i + u * stride));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; }
  }
  for (; i < n2; i += stride) { acc.x += a[i].x; acc.y += a[i].y; }
  if (acc.x == -1.2345) out[0] = acc.y;  // never true for [0,1) data: keeps the loads
}

// store flavours: 0 st.global.cs, 1 st.global (write-back), 2 st.global.L1::no_allocate,
// 3 st.global.L2::evict_last... (not used), 4 st.global.wt
template <int MODE>
__device__ __forceinline__ void st2(double2* p, double2 v) {
  if constexpr (MODE == 0) __stcs(p, v);
  else if constexpr (MODE == 1) *p = v;
  else if constexpr (MODE == 2)
    asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y)
                 : "memory");
  else __stwt(p, v);
}
template <int MODE>
__device__ __forceinline__ void st1(double* p, double v) {
  if constexpr (MODE == 0) __stcs(p, v);
  else if constexpr (MODE == 1) *p = v;
  else if constexpr (MODE == 2)
    asm volatile("st.global.L1::no_allocate.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
  else __stwt(p, v);
}

template <int MODE>
__global__ void __launch_bounds__(256) probe_write(double2* __restrict__ a, long long n2) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride)
    st2<MODE>(a + i, make_double2(1.0, 2.0));
}
template <int MODE>
__global__ void __launch_bounds__(256) probe_write1(double* __restrict__ a, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    st1<MODE>(a + i, 1.0);
}
// copy, one double per thread step (the light kernels' shape), store flavour MODE
template <int MODE>
__global__ void __launch_bounds__(256) probe_copy1(const double* __restrict__ a,
                                                   double* __restrict__ b, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    st1<MODE>(b + i, __ldcs(a + i));
}
// 256-bit accesses (LDG/STG.E.ENL2.256, sm_100) and non-persistent grids
// (one block per 256 x vector chunk, no stride loop — torch's elementwise shape)
__device__ __forceinline__ void st4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c),
               "d"(d) : "memory");
}
__global__ void __launch_bounds__(256) probe_write_v4(double* __restrict__ a, long long n4) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride)
    st4(a + 4 * i, 1.0, 2.0, 3.0, 4.0);
}
__global__ void __launch_bounds__(256) probe_write_np(double* __restrict__ a, long long n, int w) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (w == 4) {
    if (4 * i < n) st4(a + 4 * i, 1.0, 2.0, 3.0, 4.0);
  } else if (w == 2) {
    if (2 * i < n) *reinterpret_cast<double2*>(a + 2 * i) = make_double2(1.0, 2.0);
  } else {
    if (i < n) a[i] = 1.0;
  }
}
__global__ void __launch_bounds__(256) probe_copy_np(const double* __restrict__ a,
                                                     double* __restrict__ b, long long n, int w) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (w == 4) {
    if (4 * i < n) {
      double x, y, z, q;
      asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                   : "=d"(x), "=d"(y), "=d"(z), "=d"(q) : "l"(a + 4 * i));
      st4(b + 4 * i, x, y, z, q);
    }
  } else if (w == 2) {
    if (2 * i < n)
      reinterpret_cast<double2*>(b)[i] = __ldg(reinterpret_cast<const double2*>(a) + i);
  } else {
    if (i < n) b[i] = __ldg(a + i);
  }
}
__global__ void __launch_bounds__(256) probe_copy_v4(const double* __restrict__ a,
                                                     double* __restrict__ b, long long n4) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    double x, y, z, q;
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(x), "=d"(y), "=d"(z), "=d"(q) : "l"(a + 4 * i));
    st4(b + 4 * i, x, y, z, q);
  }
}

// TMA bulk store: each block fills a smem chunk once, then streams it out
template <int CH>
__global__ void __launch_bounds__(128) probe_bulk_store(char* __restrict__ a, long long bytes) {
  extern __shared__ __align__(128) char sm[];
  for (int i = threadIdx.x; i < CH / 8; i += blockDim.x) reinterpret_cast<double*>(sm)[i] = 1.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const long long nch = bytes / CH;
  unsigned src = (unsigned)__cvta_generic_to_shared(sm);
  int k = 0;
  for (long long c = blockIdx.x; c < nch; c += gridDim.x, ++k) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(a + c * CH), "r"(src), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// TMA bulk read: persistent blocks, one elected thread keeps NST copies of
// CH bytes in flight per block; consumers only wait (no data use).
template <int NST, int CH>
__global__ void __launch_bounds__(32) probe_bulk(const char* __restrict__ a, long long bytes) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) unsigned long long bar[NST];
  const long long nch = bytes / CH;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < NST; ++s) {
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto issue = [&](long long c, int s) {
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    unsigned d = (unsigned)__cvta_generic_to_shared(sm + (long long)s * CH);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(CH)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(d), "l"(a + c * CH), "r"(CH), "r"(b) : "memory");
  };
  int it = 0;
  for (int s = 0; s < NST; ++s) {
    long long c = blockIdx.x + (long long)s * gridDim.x;
    if (c < nch) issue(c, s);
  }
  for (long long c = blockIdx.x; c < nch; c += gridDim.x, ++it) {
    const int s = it % NST;
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    unsigned ph = (unsigned)(it / NST) & 1u;
    asm volatile(
        "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W_%=;\n}" ::"r"(b), "r"(ph) : "memory");
    long long cn = c + (long long)NST * gridDim.x;
    if (cn < nch) issue(cn, s);
  }
}

struct MixPtrs {
  const double2* r[64];
  double2* w[64];
};

template <int R, int W>
__global__ void __launch_bounds__(256) probe_mix(const __grid_constant__ MixPtrs P, long long n2) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
    double2 s = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < R; ++j) {
      double2 v;
      asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                   : "=d"(v.x), "=d"(v.y) : "l"(P.r[j] + i));
      s.x += v.x;
      s.y += v.y;
    }
#pragma unroll
    for (int j = 0; j < W; ++j) __stcs(P.w[j] + i, make_double2(s.x + j, s.y));
  }
}

// the same mix, one point (8-byte accesses) per thread, the shape of the
// policy-3 heavier kernels (tlk_flat_v1, 128-thread blocks)
struct MixPtrs1 {
  const double* r[64];
  double* w[64];
};
template <int R, int W>
__global__ void __launch_bounds__(256) probe_mix1(const __grid_constant__ MixPtrs1 P, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      double v;
      asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(P.r[j] + i));
      s += v;
    }
#pragma unroll
    for (int j = 0; j < W; ++j) __stcs(P.w[j] + i, s + j);
    if (W == 0 && s < -1.0) P.w[0][i] = s;  // read-only mixes: keep the loads live
  }
}

// the dispatch floor of a one-shot grid: every thread exits at once
__global__ void __launch_bounds__(256) probe_empty(long long n) {
  if ((long long)blockIdx.x * blockDim.x + threadIdx.x == n) asm volatile("trap;");
}

static int sms() {
  int d = 0, n = 0;
  cudaGetDevice(&d);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
  return n;
}

extern "C" {
int sp_read(const void* a, long long n2, void* out, int unroll, int blocks_per_sm,
            void* stream) {
  dim3 g(sms() * blocks_per_sm);
  cudaStream_t s = (cudaStream_t)stream;
  if (unroll == 1) probe_read<1><<<g, 256, 0, s>>>((const double2*)a, n2, (double*)out);
  else if (unroll == 2) probe_read<2><<<g, 256, 0, s>>>((const double2*)a, n2, (double*)out);
  else if (unroll == 4) probe_read<4><<<g, 256, 0, s>>>((const double2*)a, n2, (double*)out);
  else probe_read<8><<<g, 256, 0, s>>>((const double2*)a, n2, (double*)out);
  return (int)cudaGetLastError();
}
int sp_write(void* a, long long n2, int blocks_per_sm, void* stream, int mode, int width) {
  dim3 g(sms() * blocks_per_sm);
  cudaStream_t s = (cudaStream_t)stream;
  if (width == 16) {
    if (mode == 0) probe_write<0><<<g, 256, 0, s>>>((double2*)a, n2);
    else if (mode == 1) probe_write<1><<<g, 256, 0, s>>>((double2*)a, n2);
    else if (mode == 2) probe_write<2><<<g, 256, 0, s>>>((double2*)a, n2);
    else probe_write<4><<<g, 256, 0, s>>>((double2*)a, n2);
  } else {
    if (mode == 0) probe_write1<0><<<g, 256, 0, s>>>((double*)a, 2 * n2);
    else if (mode == 1) probe_write1<1><<<g, 256, 0, s>>>((double*)a, 2 * n2);
    else if (mode == 2) probe_write1<2><<<g, 256, 0, s>>>((double*)a, 2 * n2);
    else probe_write1<4><<<g, 256, 0, s>>>((double*)a, 2 * n2);
  }
  return (int)cudaGetLastError();
}
int sp_copy1(const void* a, void* b, long long n, int blocks_per_sm, void* stream, int mode) {
  dim3 g(sms() * blocks_per_sm);
  cudaStream_t s = (cudaStream_t)stream;
  if (mode == 0) probe_copy1<0><<<g, 256, 0, s>>>((const double*)a, (double*)b, n);
  else if (mode == 1) probe_copy1<1><<<g, 256, 0, s>>>((const double*)a, (double*)b, n);
  else if (mode == 2) probe_copy1<2><<<g, 256, 0, s>>>((const double*)a, (double*)b, n);
  else probe_copy1<4><<<g, 256, 0, s>>>((const double*)a, (double*)b, n);
  return (int)cudaGetLastError();
}
int sp_write_v4(void* a, long long n, int blocks_per_sm, void* stream) {
  probe_write_v4<<<sms() * blocks_per_sm, 256, 0, (cudaStream_t)stream>>>((double*)a, n / 4);
  return (int)cudaGetLastError();
}
int sp_write_np(void* a, long long n, int w, void* stream) {
  long long threads = (n + w - 1) / w;
  probe_write_np<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>((double*)a,
                                                                                     n, w);
  return (int)cudaGetLastError();
}
int sp_copy_np(const void* a, void* b, long long n, int w, void* stream) {
  long long threads = (n + w - 1) / w;
  probe_copy_np<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      (const double*)a, (double*)b, n, w);
  return (int)cudaGetLastError();
}
int sp_copy_v4(const void* a, void* b, long long n, int blocks_per_sm, void* stream) {
  probe_copy_v4<<<sms() * blocks_per_sm, 256, 0, (cudaStream_t)stream>>>((const double*)a,
                                                                        (double*)b, n / 4);
  return (int)cudaGetLastError();
}
int sp_bulk_store(void* a, long long bytes, int blocks_per_sm, void* stream) {
  auto k = probe_bulk_store<8192>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  k<<<sms() * blocks_per_sm, 128, 8192, (cudaStream_t)stream>>>((char*)a, bytes);
  return (int)cudaGetLastError();
}
int sp_bulk(const void* a, long long bytes, int chunk, int blocks_per_sm, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  dim3 g(sms() * blocks_per_sm);
  if (chunk == 4096) {
    auto k = probe_bulk<8, 4096>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4096);
    k<<<g, 32, 8 * 4096, s>>>((const char*)a, bytes);
  } else if (chunk == 16384) {
    auto k = probe_bulk<4, 16384>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384);
    k<<<g, 32, 4 * 16384, s>>>((const char*)a, bytes);
  } else {
    auto k = probe_bulk<6, 32768>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
    k<<<g, 32, 6 * 32768, s>>>((const char*)a, bytes);
  }
  return (int)cudaGetLastError();
}
// one point per thread; blocks_per_sm <= 0: one-shot grid (n / threads blocks)
int sp_mix1(const void* const* r, int nr, void* const* w, int nw, long long n, int blocks_per_sm,
            int threads, void* stream) {
  MixPtrs1 P;
  for (int j = 0; j < nr && j < 64; ++j) P.r[j] = (const double*)r[j];
  for (int j = 0; j < nw && j < 64; ++j) P.w[j] = (double*)w[j];
  if (nw == 0) P.w[0] = (double*)w[0];  // never written (inputs are >= 0)
  if (nr == 0) {  // no streams: the empty one-shot grid
    probe_empty<<<(unsigned)((n + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(n);
    return (int)cudaGetLastError();
  }
  long long g = blocks_per_sm > 0 ? (long long)sms() * blocks_per_sm : (n + threads - 1) / threads;
  cudaStream_t s = (cudaStream_t)stream;
  if (nr == 40 && nw == 24) probe_mix1<40, 24><<<(unsigned)g, threads, 0, s>>>(P, n);
  else if (nr == 1 && nw == 1) probe_mix1<1, 1><<<(unsigned)g, threads, 0, s>>>(P, n);
  else if (nr == 5 && nw == 3) probe_mix1<5, 3><<<(unsigned)g, threads, 0, s>>>(P, n);
  else if (nr == 16 && nw == 6) probe_mix1<16, 6><<<(unsigned)g, threads, 0, s>>>(P, n);
  else if (nr == 24 && nw == 18) probe_mix1<24, 18><<<(unsigned)g, threads, 0, s>>>(P, n);
  else if (nr == 16 && nw == 0) probe_mix1<16, 0><<<(unsigned)g, threads, 0, s>>>(P, n);
  else if (nr == 22 && nw == 0) probe_mix1<22, 0><<<(unsigned)g, threads, 0, s>>>(P, n);
  else if (nr == 1 && nw == 0) probe_mix1<1, 0><<<(unsigned)g, threads, 0, s>>>(P, n);
  else return -1;
  return (int)cudaGetLastError();
}
int sp_mix(const void* const* r, int nr, void* const* w, int nw, long long n2, int blocks_per_sm,
           void* stream) {
  MixPtrs P;
  for (int j = 0; j < nr && j < 64; ++j) P.r[j] = (const double2*)r[j];
  for (int j = 0; j < nw && j < 64; ++j) P.w[j] = (double2*)w[j];
  dim3 g(sms() * blocks_per_sm);
  cudaStream_t s = (cudaStream_t)stream;
  if (nr == 40 && nw == 24) probe_mix<40, 24><<<g, 256, 0, s>>>(P, n2);
  else if (nr == 1 && nw == 1) probe_mix<1, 1><<<g, 256, 0, s>>>(P, n2);
  else if (nr == 5 && nw == 3) probe_mix<5, 3><<<g, 256, 0, s>>>(P, n2);
  else if (nr == 16 && nw == 6) probe_mix<16, 6><<<g, 256, 0, s>>>(P, n2);
  else return -1;
  return (int)cudaGetLastError();
}
}

// tlk_template.cuh — hand-written sm_100a template for fused TLoops kernels.
//
// lowering.py generates, per assignment (or per program of assignments), a
// straight-line per-point body `tlk_point<T>(P, x)` in SSA form: every input
// component is loaded once into a register, the right-hand side runs in the
// reference's exact parse-tree / left-associated-sum order, and each written
// component is stored once.  This file supplies everything around it:
//
//   * T = double  (one point per thread step) or
//     T = double2 (two consecutive points: 128-bit LDG/STG per component);
//   * streaming loads/stores (evict-first: every byte is touched once);
//   * four entry points (plus the opt-in TMA-staged tlk_stage_v1 at the end):
//       tlk_flat_v1 / tlk_flat_v2   one grid, per-slot base pointers passed
//                                   by value in the parameter block (constant
//                                   bank) — no device pointer arrays, which
//                                   the paper names as its main loss
//                                   (PAPER.md:1813-1823);
//       tlk_batch_v1 / tlk_batch_v2 many subdomains in ONE launch: block row
//                                   y walks domains, the domain's slot
//                                   pointers are staged in shared memory.
//   * grid-stride loops over 64-bit point indices (no N <= 65535*bx cap,
//     reference codegen_cuda.py:187-189).
//
// Bit-exactness: compiled with --fmad=false (no DFMA contraction) and IEEE
// division/sqrt, so each generated operation rounds exactly like the
// reference's numpy float64 ufunc (pkg/src/tlang/evaluator.py:122-161).
//
// lowering.py prepends `#define TLK_NSLOTS <number of pointer slots>` and
// replaces the @@TLK_BODY@@ marker line below with the per-point body
// `template <typename T, int LD, typename P> tlk_point(const P& P_, long long x)`,
// which addresses slot j as `P_.p[j] + x` and loads with tl_ld<T, LD>.

#ifndef TLK_THREADS
#define TLK_THREADS 256
#endif
// Minimum resident blocks per SM the flat entries are compiled for (the
// second __launch_bounds__ argument: caps registers so a launch that is one
// wave at this occupancy never spills into a second, partial wave).
#ifndef TLK_MINB
#define TLK_MINB 1
#endif
// Unroll factor of the grid-stride loops (1 = one point group per trip; the
// per-point body already exposes all of its loads, occupancy does the rest).
#ifndef TLK_UNROLL
#define TLK_UNROLL 1
#endif
#define TLK_STR2(x) #x
#define TLK_STR(x) TLK_STR2(x)
#define TLK_LOOP _Pragma(TLK_STR(unroll TLK_UNROLL))

// ----------------------------------------------------------- lane arithmetic
__device__ __forceinline__ double2 operator+(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 operator-(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 operator*(double2 a, double2 b) { return make_double2(a.x * b.x, a.y * b.y); }
__device__ __forceinline__ double2 operator/(double2 a, double2 b) { return make_double2(a.x / b.x, a.y / b.y); }
__device__ __forceinline__ double2 operator+(double a, double2 b) { return make_double2(a + b.x, a + b.y); }
__device__ __forceinline__ double2 operator-(double a, double2 b) { return make_double2(a - b.x, a - b.y); }
__device__ __forceinline__ double2 operator*(double a, double2 b) { return make_double2(a * b.x, a * b.y); }
__device__ __forceinline__ double2 operator/(double a, double2 b) { return make_double2(a / b.x, a / b.y); }
__device__ __forceinline__ double2 operator+(double2 a, double b) { return make_double2(a.x + b, a.y + b); }
__device__ __forceinline__ double2 operator-(double2 a, double b) { return make_double2(a.x - b, a.y - b); }
__device__ __forceinline__ double2 operator*(double2 a, double b) { return make_double2(a.x * b, a.y * b); }
__device__ __forceinline__ double2 operator/(double2 a, double b) { return make_double2(a.x / b, a.y / b); }
__device__ __forceinline__ double2 operator-(double2 a) { return make_double2(-a.x, -a.y); }
__device__ __forceinline__ double tl_sqrt(double a) { return sqrt(a); }
__device__ __forceinline__ double2 tl_sqrt(double2 a) { return make_double2(sqrt(a.x), sqrt(a.y)); }

template <typename T> __device__ __forceinline__ T tl_splat(double c);
template <> __device__ __forceinline__ double tl_splat<double>(double c) { return c; }
template <> __device__ __forceinline__ double2 tl_splat<double2>(double c) { return make_double2(c, c); }

// ------------------------------------------------------------ memory access
// TLK_LDMODE 0: ld.global.cs (streaming)            [default]
//            1: ld.global.nc.L1::no_allocate as a movable asm (the lowering
//               only selects it when no slot is both read and written)
//            2: plain ld.global
//            3: plain dereference (only as tl_ld<T, 3>: the staged entry's
//               shared-memory tiles, LDS)
#ifndef TLK_LDMODE
#define TLK_LDMODE 0
#endif
// TLK_STMODE 0: st.global.cs (streaming)            [default]
//            1: plain st.global
//            2: st.global.L1::no_allocate
#ifndef TLK_STMODE
#define TLK_STMODE 0
#endif

// TLK_L2HINT 1: the read-only loads (mode 1) and the staged entry's bulk
//               copies carry an L2 evict-first cache policy (every input byte
//               is read exactly once)                        [tuning knob]
#ifndef TLK_L2HINT
#define TLK_L2HINT 0
#endif
__device__ __forceinline__ unsigned long long tl_evict_first_policy() {
  unsigned long long pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// LD is a template parameter so one module can hold entries with different
// load flavours (the staged entry reads its tiles with mode 3).
template <typename T, int LD = TLK_LDMODE>
__device__ __forceinline__ T tl_ld(const double* p) {
  if constexpr (sizeof(T) == sizeof(double)) {
    if constexpr (LD == 0) {
      return __ldcs(p);
    } else if constexpr (LD == 1) {
      double v;
#if TLK_L2HINT
      asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
          : "=d"(v) : "l"(p), "l"(tl_evict_first_policy()));
#else
      asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
#endif
      return v;
    } else {
      return *p;
    }
  } else {
    if constexpr (LD == 0) {
      return __ldcs(reinterpret_cast<const double2*>(p));
    } else if constexpr (LD == 1) {
      double2 v;
#if TLK_L2HINT
      asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
          : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(tl_evict_first_policy()));
#else
      asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
#endif
      return v;
    } else {
      return *reinterpret_cast<const double2*>(p);
    }
  }
}

__device__ __forceinline__ void tl_st(double* p, double v) {
#if TLK_STMODE == 0
  __stcs(p, v);
#elif TLK_STMODE == 2
  asm volatile("st.global.L1::no_allocate.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
#else
  *p = v;
#endif
}
__device__ __forceinline__ void tl_st(double* p, double2 v) {
#if TLK_STMODE == 0
  __stcs(reinterpret_cast<double2*>(p), v);
#elif TLK_STMODE == 2
  asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y)
               : "memory");
#else
  *reinterpret_cast<double2*>(p) = v;
#endif
}

// ------------------------------------------------------- generated body
// @@TLK_BODY@@

// ------------------------------------------------------------- entry points
struct tlk_flat_params {
  long long n;
  double* p[TLK_NSLOTS];
};

struct tlk_shared_ptrs {
  double* const* p;
};

// TLK_CHUNK > 1 (tuning): a block takes TLK_CHUNK consecutive block-sized
// runs of points before the grid strides on (one-shot grids then have
// n / (threads * TLK_CHUNK) blocks; the runtime reads TLK_CHUNK from the source)
#ifndef TLK_CHUNK
#define TLK_CHUNK 1
#endif
// TLK_PARTS > 1 (Variant.split): the program is independent statement parts
// (no field in common).  The grid's blocks are cut into TLK_PARTS equal runs
// and run p evaluates part p over every point: a one-shot grid dispatches the
// runs in order, so the parts stream one after another, each with fewer
// concurrent DRAM streams than the whole program (the runtime multiplies the
// grid by TLK_PARTS, read from the source).  Same bits: a point's statements
// of one part run in program order, and parts share no storage.
#ifndef TLK_PARTS
#define TLK_PARTS 1
#endif
extern "C" __global__ void __launch_bounds__(TLK_THREADS, TLK_MINB)
tlk_flat_v1(const __grid_constant__ tlk_flat_params prm) {
#if TLK_PARTS > 1
  const unsigned per = gridDim.x / TLK_PARTS;
  const unsigned part = blockIdx.x / per;
  if (part >= TLK_PARTS) return;
  const long long stride = (long long)per * blockDim.x;
  TLK_LOOP
  for (long long x = (long long)(blockIdx.x - part * per) * blockDim.x + threadIdx.x; x < prm.n;
       x += stride)
    tlk_part<double>(part, prm, x);
#elif TLK_CHUNK > 1
  const long long bstride = (long long)gridDim.x * blockDim.x * TLK_CHUNK;
  for (long long base = (long long)blockIdx.x * blockDim.x * TLK_CHUNK; base < prm.n;
       base += bstride) {
#pragma unroll 1
    for (int k = 0; k < TLK_CHUNK; ++k) {
      const long long x = base + (long long)k * blockDim.x + threadIdx.x;
      if (x < prm.n) tlk_point<double>(prm, x);
    }
  }
#else
  const long long stride = (long long)gridDim.x * blockDim.x;
  TLK_LOOP
  for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < prm.n; x += stride)
    tlk_point<double>(prm, x);
#endif
}

extern "C" __global__ void __launch_bounds__(TLK_THREADS, TLK_MINB)
tlk_flat_v2(const __grid_constant__ tlk_flat_params prm) {
  const long long pairs = prm.n >> 1;
  const long long stride = (long long)gridDim.x * blockDim.x;
  TLK_LOOP
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < pairs; i += stride)
    tlk_point<double2>(prm, i << 1);
  if ((prm.n & 1) && blockIdx.x == 0 && threadIdx.x == 0) tlk_point<double>(prm, prm.n - 1);
}

// table: per domain { long long n; double* p[TLK_NSLOTS]; } (tlb_batch_create)
// TLK_BATCH_PTRS 0: the block stages the domain's slot pointers in shared
//                   memory (one barrier pair per domain)            [default]
//                1: every thread reads them straight from the (read-only,
//                   L1-resident) table: no barriers, so pointer fetches of
//                   one warp overlap data traffic of the others
#ifndef TLK_BATCH_PTRS
#define TLK_BATCH_PTRS 0
#endif

struct tlk_table_ptrs {
  const long long* __restrict__ rec;
  struct view {
    const long long* __restrict__ r;
    __device__ __forceinline__ double* operator[](int j) const {
      return reinterpret_cast<double*>(__ldg(r + 1 + j));
    }
  } p;
};

template <typename T, typename P>
__device__ __forceinline__ void tlk_domain(const P& ptrs, const long long n, const long long stride) {
  if constexpr (sizeof(T) == 16) {
    const long long pairs = n >> 1;
    TLK_LOOP
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < pairs; i += stride)
      tlk_point<T>(ptrs, i << 1);
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) tlk_point<double>(ptrs, n - 1);
  } else {
    TLK_LOOP
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += stride)
      tlk_point<double>(ptrs, x);
  }
}

#if defined(TLK_BATCH_SPLIT) && TLK_PARTS > 1
// the 1-point batch entry over statement parts: block rows y walk (part,
// domain) pairs part-major, so every domain's part 0 streams before any
// part 1 (the runtime launches ndom x TLK_PARTS rows, capped at 65535)
template <typename P>
__device__ __forceinline__ void tlk_domain_part(const unsigned part, const P& ptrs,
                                                const long long n, const long long stride) {
  TLK_LOOP
  for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += stride)
    tlk_part<double>(part, ptrs, x);
}
#endif

template <typename T>
__device__ __forceinline__ void tlk_batch_body(const long long* __restrict__ table, int ndom) {
  const long long stride = (long long)gridDim.x * blockDim.x;
#if defined(TLK_BATCH_SPLIT) && TLK_PARTS > 1
  if constexpr (sizeof(T) == 8) {
    const int rows = ndom * TLK_PARTS;
#if TLK_BATCH_PTRS == 0
    __shared__ double* spp[TLK_NSLOTS];
#endif
    for (int y = blockIdx.y; y < rows; y += gridDim.y) {
      const unsigned part = (unsigned)(y / ndom);
      const int d = y - (int)part * ndom;
      const long long* rec = table + (long long)d * (TLK_NSLOTS + 1);
#if TLK_BATCH_PTRS == 0
      __syncthreads();
      for (int j = threadIdx.x; j < TLK_NSLOTS; j += blockDim.x)
        spp[j] = reinterpret_cast<double*>(rec[1 + j]);
      const long long n = rec[0];
      __syncthreads();
      tlk_domain_part(part, tlk_shared_ptrs{spp}, n, stride);
#else
      const tlk_table_ptrs P{rec, {rec}};
      tlk_domain_part(part, P, __ldg(rec), stride);
#endif
    }
    return;
  }
#endif
#if TLK_BATCH_PTRS == 0
  __shared__ double* sp[TLK_NSLOTS];
  for (int d = blockIdx.y; d < ndom; d += gridDim.y) {
    const long long* rec = table + (long long)d * (TLK_NSLOTS + 1);
    __syncthreads();  // readers of the previous domain's pointers are done
    for (int j = threadIdx.x; j < TLK_NSLOTS; j += blockDim.x)
      sp[j] = reinterpret_cast<double*>(rec[1 + j]);
    const long long n = rec[0];
    __syncthreads();
    tlk_domain<T>(tlk_shared_ptrs{sp}, n, stride);
  }
#else
  for (int d = blockIdx.y; d < ndom; d += gridDim.y) {
    const long long* rec = table + (long long)d * (TLK_NSLOTS + 1);
    const tlk_table_ptrs P{rec, {rec}};
    tlk_domain<T>(P, __ldg(rec), stride);
  }
#endif
}

// the batch entries' own launch bound (lowering: TLK_BATCH_BOUND, default
// the flat entries' TLK_THREADS); their blocks are at most this large
#ifndef TLK_BATCH_BOUND
#define TLK_BATCH_BOUND TLK_THREADS
#endif
extern "C" __global__ void __launch_bounds__(TLK_BATCH_BOUND)
tlk_batch_v1(const long long* __restrict__ table, int ndom) {
  tlk_batch_body<double>(table, ndom);
}

extern "C" __global__ void __launch_bounds__(TLK_BATCH_BOUND)
tlk_batch_v2(const long long* __restrict__ table, int ndom) {
  tlk_batch_body<double2>(table, ndom);
}

// ------------------------------------------------ TMA-staged entry (opt-in)
// tlk_stage_v1: persistent blocks walk tiles of TLK_STAGE_THREADS points (one
// per thread; its own block size and launch bounds); for each
// tile one elected thread issues one 1-D bulk copy (cp.async.bulk, the TMA
// engine) per read slot into a TLK_NSTAGE-deep shared-memory ring, completion
// tracked by an mbarrier (complete_tx); every thread then runs the per-point
// body with its read slots pointing into the tile and its write slots at the
// global arrays.  The copies of the next TLK_NSTAGE-1 tiles are in flight
// while a tile computes.  Points past the last whole tile take the plain
// path.  Compiled only when the lowering defines TLK_NSTAGE (with TLK_NREAD,
// TLK_STAGE_THREADS and the per-slot read ordinals TLK_RORD); needs every
// read slot 16-byte aligned (the runtime checks).
#ifdef TLK_NSTAGE
#ifndef TLK_TILE_ORDER
#define TLK_TILE_ORDER 0
#endif
#if TLK_NREAD < 1
#error "a staged kernel needs at least one staged read slot (its mbarrier would never complete)"
#endif
__device__ __forceinline__ unsigned tlk_smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

#ifndef TLK_STAGE_WS
#define TLK_STAGE_WS 0
#endif
#if TLK_STAGE_WS
// Warp-specialised form (TLK_STAGE_WS 1): block = TLK_STAGE_THREADS consumer
// threads + one producer warp.  Lane 0 of the producer waits on the stage's
// `empty` barrier (one arrival per consumer warp), then re-arms `full` with
// the tile's byte count and issues its bulk copies; consumer warps release a
// stage as soon as they are done with it — no block-wide barrier per tile, and
// no consumer thread serialises the copy issue.
extern "C" __global__ void __launch_bounds__(TLK_STAGE_THREADS + 32)
tlk_stage_v1(const tlk_flat_params prm) {
  constexpr int kRord[TLK_NSLOTS] = TLK_RORD;
  constexpr int kTile = TLK_STAGE_THREADS;
  constexpr int kWarps = TLK_STAGE_THREADS / 32;
  extern __shared__ __align__(128) double tlk_sm[];  // [NSTAGE][NREAD][kTile]
  __shared__ __align__(8) unsigned long long full[TLK_NSTAGE], empty[TLK_NSTAGE];
  const long long ntiles = prm.n / kTile;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < TLK_NSTAGE; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tlk_smem_addr(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tlk_smem_addr(&empty[s])),
                   "r"(kWarps));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid >= kTile) {  // producer warp: lane 0 issues, the other lanes exit
    if (tid != kTile) return;
#if TLK_L2HINT
    const unsigned long long pol = tl_evict_first_policy();
#endif
    int it = 0;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int s = it % TLK_NSTAGE;
      if (it >= TLK_NSTAGE) {
        const unsigned eb = tlk_smem_addr(&empty[s]);
        const unsigned ph = (unsigned)(it / TLK_NSTAGE - 1) & 1u;
        asm volatile(
            "{\n .reg .pred p;\n"
            "TLK_EWAIT_%=:\n"
            " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            " @!p bra TLK_EWAIT_%=;\n}" ::"r"(eb), "r"(ph) : "memory");
      }
      const unsigned b = tlk_smem_addr(&full[s]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                   ::"r"(b), "r"((unsigned)(TLK_NREAD * kTile * sizeof(double))) : "memory");
#pragma unroll
      for (int j = 0; j < TLK_NSLOTS; ++j) {
        if (kRord[j] < 0) continue;
        const double* src = prm.p[j] + t * kTile;
        double* dst = tlk_sm + ((long long)s * TLK_NREAD + kRord[j]) * kTile;
#if TLK_L2HINT
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
            "[%0], [%1], %2, [%3], %4;"
            ::"r"(tlk_smem_addr(dst)), "l"(src), "r"((unsigned)(kTile * sizeof(double))), "r"(b),
              "l"(pol)
            : "memory");
#else
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(tlk_smem_addr(dst)), "l"(src), "r"((unsigned)(kTile * sizeof(double))), "r"(b)
            : "memory");
#endif
      }
    }
    return;
  }
  int it = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int s = it % TLK_NSTAGE;
    const unsigned phase = (unsigned)(it / TLK_NSTAGE) & 1u;
    const unsigned b = tlk_smem_addr(&full[s]);
    asm volatile(
        "{\n .reg .pred p;\n"
        "TLK_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra TLK_WAIT_%=;\n}" ::"r"(b), "r"(phase) : "memory");
    tlk_flat_params q;
    q.n = prm.n;
#pragma unroll
    for (int j = 0; j < TLK_NSLOTS; ++j)
      q.p[j] = kRord[j] >= 0 ? tlk_sm + ((long long)s * TLK_NREAD + kRord[j]) * kTile
                             : prm.p[j] + t * kTile;
    tlk_point<double, 3>(q, tid);
    __syncwarp();  // the warp's reads of stage s are done
    if ((tid & 31) == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tlk_smem_addr(&empty[s]))
                   : "memory");
  }
  const long long stride = (long long)gridDim.x * kTile;
  for (long long x = ntiles * kTile + (long long)blockIdx.x * kTile + tid; x < prm.n;
       x += stride)
    tlk_point<double>(prm, x);
}
#else
extern "C" __global__ void __launch_bounds__(TLK_STAGE_THREADS)
tlk_stage_v1(const tlk_flat_params prm) {
  constexpr int kRord[TLK_NSLOTS] = TLK_RORD;
  constexpr int kTile = TLK_STAGE_THREADS;
  extern __shared__ __align__(128) double tlk_sm[];  // [NSTAGE][NREAD][kTile]
  __shared__ __align__(8) unsigned long long bar[TLK_NSTAGE];
  const long long ntiles = prm.n / kTile;
  const int tid = threadIdx.x;
  // tile order: 0 = interleaved (block b takes b, b + grid, ...), so the
  // blocks sweep the grid together; 1 = one contiguous run of tiles per block
#if TLK_TILE_ORDER == 1
  const long long per = (ntiles + gridDim.x - 1) / gridDim.x;
  const long long t0 = (long long)blockIdx.x * per;
  const long long t1 = ntiles < t0 + per ? ntiles : t0 + per;
  const long long tstep = 1;
#else
  const long long t0 = blockIdx.x, t1 = ntiles, tstep = gridDim.x;
#endif
  if (tid == 0) {
    for (int s = 0; s < TLK_NSTAGE; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tlk_smem_addr(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](long long t, int s) {
    const unsigned b = tlk_smem_addr(&bar[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 ::"r"(b), "r"((unsigned)(TLK_NREAD * kTile * sizeof(double))) : "memory");
#if TLK_L2HINT
    const unsigned long long pol = tl_evict_first_policy();
#endif
#pragma unroll
    for (int j = 0; j < TLK_NSLOTS; ++j) {
      if (kRord[j] < 0) continue;
      const double* src = prm.p[j] + t * kTile;
      double* dst = tlk_sm + ((long long)s * TLK_NREAD + kRord[j]) * kTile;
#if TLK_L2HINT
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
          "[%0], [%1], %2, [%3], %4;"
          ::"r"(tlk_smem_addr(dst)), "l"(src), "r"((unsigned)(kTile * sizeof(double))), "r"(b),
            "l"(pol)
          : "memory");
#else
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          ::"r"(tlk_smem_addr(dst)), "l"(src), "r"((unsigned)(kTile * sizeof(double))), "r"(b)
          : "memory");
#endif
    }
  };
  if (tid == 0)
    for (int s = 0; s < TLK_NSTAGE; ++s) {
      const long long t = t0 + (long long)s * tstep;
      if (t < t1) issue(t, s);
    }
  int it = 0;
  for (long long t = t0; t < t1; t += tstep, ++it) {
    const int s = it % TLK_NSTAGE;
    const unsigned phase = (unsigned)(it / TLK_NSTAGE) & 1u;
    const unsigned b = tlk_smem_addr(&bar[s]);
    asm volatile(
        "{\n .reg .pred p;\n"
        "TLK_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra TLK_WAIT_%=;\n}" ::"r"(b), "r"(phase) : "memory");
    tlk_flat_params q;
    q.n = prm.n;
#pragma unroll
    for (int j = 0; j < TLK_NSLOTS; ++j)
      q.p[j] = kRord[j] >= 0 ? tlk_sm + ((long long)s * TLK_NREAD + kRord[j]) * kTile
                             : prm.p[j] + t * kTile;
    tlk_point<double, 3>(q, tid);
    __syncthreads();  // every thread is done with stage s
    if (tid == 0) {
      const long long tn = t + (long long)TLK_NSTAGE * tstep;
      if (tn < t1) issue(tn, s);
    }
  }
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long x = ntiles * kTile + (long long)blockIdx.x * blockDim.x + tid; x < prm.n;
       x += stride)
    tlk_point<double>(prm, x);
}
#endif  // TLK_STAGE_WS

// tlk_stage_batch_v1: the multi-domain batch through the same ring, with a
// dedicated producer warp (block = TLK_STAGE_THREADS consumers + 32).  Work
// items are (domain, tile) pairs, built on the host at tlb_batch_create:
// items[w] = {domain | count << 32, first point}.  Per item the producer warp
// fetches the record and the domain's slot pointers one item ahead into
// registers (lanes stride over slots), writes them to the stage's pointer
// block once the stage is free, then lane 0 issues the bulk
// copies of the staged read slots (full[s] completes on their bytes plus 32
// lane arrivals).  Tiles with an odd count or any slot not 16-byte aligned
// are not copied: their count is stored negated and consumers read every
// slot from global memory.  Consumers release a stage through empty[s]; the
// producer refills it NSTAGE items later.  Pointer block: NSTAGE x NSLOTS
// pointers after the ring.
#ifdef TLK_STAGE_BATCH  // opt-in (Variant.batch_vec = 3): measured slower than tlk_batch_v1
__device__ __forceinline__ void tlk_mbar_wait(unsigned b, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "TLK_BWAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TLK_BWAIT_%=;\n}" ::"r"(b), "r"(phase) : "memory");
}
__device__ __forceinline__ void tlk_mbar_arrive(unsigned b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}

extern "C" __global__ void __launch_bounds__(TLK_STAGE_THREADS + 32)
tlk_stage_batch_v1(const long long* __restrict__ table, const longlong2* __restrict__ items,
                   long long nitems) {
  constexpr int kRord[TLK_NSLOTS] = TLK_RORD;
  constexpr int kTile = TLK_STAGE_THREADS;
  extern __shared__ __align__(128) double tlk_sm[];
  double** ptrs = reinterpret_cast<double**>(tlk_sm + (long long)TLK_NSTAGE * TLK_NREAD * kTile);
  __shared__ int cnts[TLK_NSTAGE];
  __shared__ __align__(8) unsigned long long full[TLK_NSTAGE], empty[TLK_NSTAGE];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < TLK_NSTAGE; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(tlk_smem_addr(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tlk_smem_addr(&empty[s])),
                   "r"(kTile));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid >= kTile) {  // producer warp
    // item records and slot pointers are fetched one item ahead, into
    // registers, so their latency overlaps the wait for a free stage
    constexpr int kPer = (TLK_NSLOTS + 31) / 32;
    const int lane = tid - kTile;
    double* pre[kPer];
    long long pd = 0, pbase = 0;
    int pcnt = 0;
    auto fetch = [&](long long w) {
      const longlong2 item = items[w];
      pd = item.x & 0xffffffffLL;
      pcnt = (int)(item.x >> 32);
      pbase = item.y;
      const long long* rec = table + pd * (TLK_NSLOTS + 1);
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int j = lane + 32 * q;
        pre[q] = j < TLK_NSLOTS ? reinterpret_cast<double*>(__ldg(rec + 1 + j)) + pbase
                                : nullptr;
      }
    };
    if (blockIdx.x < nitems) fetch(blockIdx.x);
    int k = 0;
    for (long long w = blockIdx.x; w < nitems; w += gridDim.x, ++k) {
      const int s = k % TLK_NSTAGE;
      if (k >= TLK_NSTAGE)
        tlk_mbar_wait(tlk_smem_addr(&empty[s]), (unsigned)(k / TLK_NSTAGE - 1) & 1u);
      const int cnt = pcnt;
      bool ok = (cnt & 1) == 0;
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int j = lane + 32 * q;
        if (j < TLK_NSLOTS) {
          ok = ok && (reinterpret_cast<unsigned long long>(pre[q]) & 15ull) == 0;
          ptrs[s * TLK_NSLOTS + j] = pre[q];
        }
      }
      ok = __all_sync(0xffffffffu, ok);
      if (lane == 0) cnts[s] = ok ? cnt : -cnt;
      __syncwarp();
      if (w + gridDim.x < nitems) fetch(w + gridDim.x);  // next item, in flight
      const unsigned fb = tlk_smem_addr(&full[s]);
      if (ok && lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     ::"r"(fb), "r"((unsigned)(TLK_NREAD * cnt * sizeof(double))) : "memory");
#pragma unroll
        for (int j = 0; j < TLK_NSLOTS; ++j) {
          if (kRord[j] < 0) continue;
          double* dst = tlk_sm + ((long long)s * TLK_NREAD + kRord[j]) * kTile;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
              "[%3];" ::"r"(tlk_smem_addr(dst)), "l"(ptrs[s * TLK_NSLOTS + j]),
              "r"((unsigned)(cnt * sizeof(double))), "r"(fb) : "memory");
        }
      } else {
        tlk_mbar_arrive(fb);
      }
    }
  } else {  // consumers
    int k = 0;
    for (long long w = blockIdx.x; w < nitems; w += gridDim.x, ++k) {
      const int s = k % TLK_NSTAGE;
      tlk_mbar_wait(tlk_smem_addr(&full[s]), (unsigned)(k / TLK_NSTAGE) & 1u);
      const int c = cnts[s];
      tlk_flat_params q;
      q.n = 0;
#pragma unroll
      for (int j = 0; j < TLK_NSLOTS; ++j)
        q.p[j] = (c > 0 && kRord[j] >= 0)
                     ? tlk_sm + ((long long)s * TLK_NREAD + kRord[j]) * kTile
                     : ptrs[s * TLK_NSLOTS + j];
      if (tid < (c < 0 ? -c : c)) tlk_point<double, 3>(q, tid);
      tlk_mbar_arrive(tlk_smem_addr(&empty[s]));
    }
  }
}
#endif  // TLK_STAGE_BATCH
#endif

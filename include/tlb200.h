/* tlb200.h — C-ABI of libtlb200.so, the B200 (sm_100a) execution layer of the
 * fused TLoops evaluator.
 *
 * Everything here is plain C: opaque handles, raw pointers, 64-bit sizes and
 * int status codes (0 = ok; on failure tlb_last_error() holds a message for
 * the calling thread).  No torch or CUDA types appear in any signature:
 * streams are passed as `void*` (a CUstream / cudaStream_t, NULL = legacy
 * default stream of the current context).
 *
 * Which reference interface each entry point replaces (paths relative to the
 * reference checkout, see INTEGRATION.md for the bindings a maintainer adds):
 *
 *   tlb_compile / tlb_kernel_set_slots
 *       replace the emit step `codegen_cuda.emit_cuda` + nvcc
 *       (pkg/src/tlang/codegen_cuda.py:135-204): one fused kernel per
 *       assignment (or per program), JIT-compiled for sm_100a with
 *       --fmad=false, cached on disk by the source hash.
 *   tlb_launch
 *       replaces `CUDAWrapper_g_NNNN` + `g_NNNN<<<>>>`
 *       (codegen_cuda.py:182-201) and the pointer cache
 *       `tl_ptrcache_device` (codegen_cuda.py:219-291): per-component base
 *       pointers travel by value in the kernel parameter block, so there is
 *       no device pointer array and no N <= 65535*bx limit.
 *   tlb_batch_create / tlb_batch_launch
 *       new (SURVEY.md 8b "API gap"): one launch over a device table of
 *       subdomains; replaces a host loop of per-domain wrapper calls.
 *   tlb_exec_host
 *       replaces `tl_call_NNNN` of the emitted CUDA bindings
 *       (pkg/src/tlang/registry.py:241-257, goldens/suite/tloops_bindings.cu:289)
 *       which passed *host* pointer arrays to a kernel: here host component
 *       arrays are staged through device slabs (H2D -> fused kernel -> D2H),
 *       pipelined on three streams, synchronously like the reference `call`.
 *   tlb_fill_uniform
 *       counter-based replacement for `bench.make_env`'s
 *       np.random.default_rng(seed).uniform(0,1) (pkg/src/tlang/bench.py:72-87)
 *       at sizes the host cannot generate.
 */
#ifndef TLB200_H
#define TLB200_H

#ifdef __cplusplus
extern "C" {
#endif

#define TLB_ABI_VERSION 1

/* tlb_launch max_blocks at or above this: a one-shot grid (one block per
 * `threads` points or point pairs, no grid-stride trips; small launches get
 * smaller blocks so every SM has work) */
#define TLB_ONE_SHOT (1LL << 62)

/* slot flags for tlb_kernel_set_slots */
#define TLB_SLOT_READ 1
#define TLB_SLOT_WRITE 2

typedef struct tlb_kernel tlb_kernel;
typedef struct tlb_batch tlb_batch;

/* ---- library ------------------------------------------------------------ */

int tlb_abi_version(void);
/* dlopen libcuda.so.1 (driver) and libnvrtc.so.12.  Called implicitly by the
 * other entry points; `want_driver` = 0 loads only NVRTC (compile-only use on
 * a machine without a GPU). */
int tlb_init(int want_driver);
const char* tlb_last_error(void);
int tlb_nvrtc_version(int* major, int* minor);
/* number of SMs of the device owning the current context */
int tlb_device_sm_count(int* out);

/* ---- compile -------------------------------------------------------------- */

/* Compile `src` with NVRTC (options verbatim, e.g. "--gpu-architecture=sm_100a",
 * "--fmad=false").  If `cache_path` names an existing file its cubin is used
 * instead; after a successful compile the cubin is written there atomically.
 * The module is loaded lazily, per CUDA context, at first launch, so
 * compiling needs no GPU.  The source must define the four entry points
 * tlk_flat_v1, tlk_flat_v2, tlk_batch_v1, tlk_batch_v2 (see lowering.py),
 * and may define the TMA-staged tlk_stage_v1; the launch geometry is read
 * from its `#define`s: TLK_THREADS (block size of the plain entries, default
 * 256) and, for the staged entry, TLK_STAGE_THREADS (its block = tile, in
 * points) and TLK_NSTAGE x TLK_NREAD tiles of dynamic shared memory. */
int tlb_compile(const char* src, const char* const* opts, int nopts,
                const char* cache_path, tlb_kernel** out);
/* Compile log (warnings) of the last compile of `k` (empty when cached). */
const char* tlb_kernel_log(const tlb_kernel* k);
/* Raw cubin bytes of `k`. */
int tlb_kernel_cubin(const tlb_kernel* k, const void** data, long long* size);
void tlb_kernel_destroy(tlb_kernel* k);

/* Describe the kernel's pointer slots: slot j addresses component
 * slot_comp[j] of field slot_field[j] (0 <= field < nfields); flags say
 * whether the kernel reads and/or writes it. */
int tlb_kernel_set_slots(tlb_kernel* k, int nfields, int nslots, const int* slot_field,
                         const long long* slot_comp, const int* slot_flags);

/* registers / local (spill) bytes / max threads of one entry point, loading
 * the module into the current context if needed (needs a GPU). */
int tlb_kernel_attrs(tlb_kernel* k, const char* entry, int* regs, int* local_bytes,
                     int* max_threads);

/* ---- launch -------------------------------------------------------------- */

/* One fused launch over points [0, n) of one grid.  field_bases[f] is the
 * device address of component 0 of field f, components `pitches[f]` doubles
 * apart.  vec: 0 = choose (2-point 128-bit path when every slot is 16-byte
 * aligned), 1 or 2 = force, 3 = the TMA-staged entry (modules lowered with a staged variant;
 * falls back to the 1-point entry when a slot is not 16-byte aligned).
 * threads: block size (0 = the kernel's compiled TLK_THREADS; must not
 * exceed it).  max_blocks: grid cap (0 = one full wave at occupancy, -w = w
 * waves, > 0 that many blocks at most, >= TLB_ONE_SHOT a one-shot grid).
 * Modules lowered in independent statement parts (TLK_PARTS = p > 1 in the
 * source) run the 1-point entry as p equal runs of blocks, one per part: the
 * grid above is computed per part (a cap is shared, at least one block per
 * part) and multiplied by p.
 * Asynchronous on `stream`. */
int tlb_launch(tlb_kernel* k, long long n, const void* const* field_bases,
               const long long* pitches, int vec, int threads, long long max_blocks,
               void* stream);

/* tlb_launch with the launch geometry the lowering chose for this kernel,
 * read from its source (TLK_VEC, TLK_GRID_WAVES; the staged entry when the
 * module has one): what a C caller without a tuning opinion should call —
 * it is the shape the Python API, the host-staged path and the harness
 * bindings launch (e.g. a one-shot grid of 1-point 128-thread blocks for
 * the benchmark program).  Asynchronous on `stream`. */
int tlb_launch_default(tlb_kernel* k, long long n, const void* const* field_bases,
                       const long long* pitches, void* stream);

/* Multi-domain batch: ndom subdomains, each with its own field bases
 * (field_bases[d*nfields+f]), pitches and point count ns[d].  The table is
 * resolved to per-slot pointers and uploaded once (synchronously, in the
 * context owning `stream`); tlb_batch_launch is then a single kernel launch
 * (CUDA-graph capturable). */
int tlb_batch_create(tlb_kernel* k, int ndom, const void* const* field_bases,
                     const long long* pitches, const long long* ns, void* stream,
                     tlb_batch** out);
/* vec: 0 = 2-point variant when every slot of every domain is 16-byte
 * aligned, 1 = force the 1-point variant, 3 = the TMA-staged batch entry
 * tlk_stage_batch_v1 (modules lowered with a staged variant; otherwise the
 * 1-point variant; its work-item list is built and uploaded by the first
 * staged launch, so make that one outside stream capture).  `threads`
 * applies to the plain entries only. */
int tlb_batch_launch(tlb_batch* b, int vec, int threads, void* stream);
void tlb_batch_destroy(tlb_batch* b);

/* Host-resident fields: comp_ptrs[f][c] is the host address of canonical
 * component c of field f (n doubles each).  Read slots are copied H2D, the
 * fused kernel runs, written slots are copied D2H, in slabs of `slab` points
 * (0 = automatic, <= 4 GiB of staging) pipelined over three streams/buffers.
 * Synchronous on return. */
int tlb_exec_host(tlb_kernel* k, long long n, const double* const* const* comp_ptrs,
                  long long slab, void* stream);

/* Free the host-staging buffers (tlb_exec_host) of the current context. */
int tlb_release_staging(void);

/* ---- reference-harness bindings --------------------------------------------
 *
 * Lets the reference's UNCHANGED conformance harness (pkg/harness/tl_harness.c)
 * drive the fused GPU kernels: paper_1804_10120_b200.registry writes a
 * tloops_bindings_b200.c whose tloops_entries[] has the reference layout
 * (pkg/src/tlang/registry.py:134-167) and whose per-entry `call(N, T, S, D)`
 * forwards to tlb_harness_call with the host pointer arrays the harness
 * built (flattened, symmetric images aliased — tl_harness.c:200-205).
 */
typedef struct tlb_harness_kernel {
  const char* source;            /* fused kernel source (lowering.py) */
  int nopts;
  const char* const* opts;       /* NVRTC options */
  int nfields;                   /* kernel fields, lowering order */
  const int* field_kind;         /* 0: tensor argument T[field_arg], 1: scalar S[field_arg] */
  const int* field_arg;
  const int* field_ncomp;
  const long* const* field_comp_flat; /* per tensor field: flat index of each component */
  int nslots;
  const int* slot_field;
  const long long* slot_comp;
  const int* slot_flags;
  tlb_kernel* compiled;          /* filled on first call */
} tlb_harness_kernel;

/* Stage the harness's host arrays through the GPU and run the kernel
 * (compiling it on first use; cubins cached under $TLB_CACHE_DIR if set).
 * The generated `call` wrappers exit the harness process with
 * TLB_HARNESS_EXIT_GPU (after printing tlb_last_error() with the kernel's
 * tl_NNNN name) when this fails: the reference `call` returns void, and the
 * harness's own exit codes 2-6 (tl_harness.c:14-15) keep their meaning. */
#define TLB_HARNESS_EXIT_GPU 7
int tlb_harness_call(tlb_harness_kernel* hk, long n, double** const* tensors,
                     const double* const* scalars);

/* ---- synthetic data ------------------------------------------------------ */

/* dst[i] = u01(seed, stream_id, offset + i) for i in [0, n): a counter-based
 * uniform [0,1) double (splitmix64 hash, 53 random bits), reproducible on the
 * host by oracle/counter_rng.py for slab-sampled parity checks. */
int tlb_fill_uniform(double* dst, long long n, unsigned long long seed,
                     unsigned long long stream_id, long long offset, void* stream);

/* FP64 throughput probe (the flop side of the roofline): `blocks` blocks of
 * 256 threads, each thread running 8 independent chains of `iters` uncontracted
 * DMUL+DADD steps (2 flops each) — the instruction mix of the fused kernels,
 * which are compiled without FMA contraction.  `out` (one double) is written
 * only to keep the chains live.  Asynchronous on `stream`; time it with
 * events: flops = blocks * 256 * iters * 16. */
int tlb_fp64_probe(double* out, int blocks, int iters, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TLB200_H */

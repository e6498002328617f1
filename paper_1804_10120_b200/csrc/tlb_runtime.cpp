// libtlb200 — host runtime of the fused TLoops evaluator (C-ABI, see include/tlb200.h).
//
// The CUDA driver (libcuda.so.1) and NVRTC (libnvrtc.so.12) are dlopen'ed on
// first use, so the library loads — and compiles kernels — on a machine
// without a GPU; only module loading and launches need the driver.
//
// Reference interfaces replaced (paths relative to the reference checkout):
//   * emit + nvcc of g_NNNN           pkg/src/tlang/codegen_cuda.py:135-204
//   * CUDAWrapper_g_NNNN launch       pkg/src/tlang/codegen_cuda.py:182-201
//   * GPUPointers cache               pkg/src/tlang/codegen_cuda.py:219-291
//   * tl_call_NNNN host invoker       pkg/src/tlang/registry.py:241-257

#include <cuda.h>
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <sys/stat.h>
#include <unistd.h>

#include "../../include/tlb200.h"

namespace {

// ---------------------------------------------------------------- errors ----

thread_local std::string g_err;

int fail(const char* fmt, ...) {
  char buf[2048];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return 1;
}

// ------------------------------------------------------ dynamic symbols ----

// Driver API subset, resolved by explicit (versioned) symbol names.
struct Driver {
  void* handle = nullptr;
  CUresult (*Init)(unsigned) = nullptr;
  CUresult (*GetErrorString)(CUresult, const char**) = nullptr;
  CUresult (*CtxGetCurrent)(CUcontext*) = nullptr;
  CUresult (*CtxSetCurrent)(CUcontext) = nullptr;
  CUresult (*CtxGetDevice)(CUdevice*) = nullptr;
  CUresult (*DeviceGet)(CUdevice*, int) = nullptr;
  CUresult (*DeviceGetAttribute)(int*, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*DevicePrimaryCtxRetain)(CUcontext*, CUdevice) = nullptr;
  CUresult (*StreamGetCtx)(CUstream, CUcontext*) = nullptr;
  CUresult (*StreamCreate)(CUstream*, unsigned) = nullptr;
  CUresult (*StreamSynchronize)(CUstream) = nullptr;
  CUresult (*StreamWaitEvent)(CUstream, CUevent, unsigned) = nullptr;
  CUresult (*EventCreate)(CUevent*, unsigned) = nullptr;
  CUresult (*EventRecord)(CUevent, CUstream) = nullptr;
  CUresult (*EventDestroy)(CUevent) = nullptr;
  CUresult (*ModuleLoadData)(CUmodule*, const void*) = nullptr;
  CUresult (*ModuleUnload)(CUmodule) = nullptr;
  CUresult (*CtxSynchronize)(void) = nullptr;
  CUresult (*ModuleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*FuncGetAttribute)(int*, CUfunction_attribute, CUfunction) = nullptr;
  CUresult (*FuncSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned,
                           unsigned, unsigned, CUstream, void**, void**) = nullptr;
  CUresult (*OccupancyMaxActiveBlocksPerMultiprocessor)(int*, CUfunction, int, size_t) = nullptr;
  CUresult (*MemAlloc)(CUdeviceptr*, size_t) = nullptr;
  CUresult (*MemFree)(CUdeviceptr) = nullptr;
  CUresult (*MemcpyHtoD)(CUdeviceptr, const void*, size_t) = nullptr;
  CUresult (*MemcpyHtoDAsync)(CUdeviceptr, const void*, size_t, CUstream) = nullptr;
  CUresult (*MemcpyDtoHAsync)(void*, CUdeviceptr, size_t, CUstream) = nullptr;
  CUresult (*MemHostRegister)(void*, size_t, unsigned) = nullptr;
  CUresult (*MemHostUnregister)(void*) = nullptr;
  CUresult (*PointerGetAttributes)(unsigned, CUpointer_attribute*, void**, CUdeviceptr) = nullptr;
  CUresult (*MemHostAlloc)(void**, size_t, unsigned) = nullptr;
  CUresult (*MemFreeHost)(void*) = nullptr;
  CUresult (*EventSynchronize)(CUevent) = nullptr;
};

// NVRTC subset (the nvrtcProgram handle is an opaque pointer).
typedef void* nvrtcProgram_t;
struct Nvrtc {
  void* handle = nullptr;
  int (*Version)(int*, int*) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  int (*CreateProgram)(nvrtcProgram_t*, const char*, const char*, int, const char* const*,
                       const char* const*) = nullptr;
  int (*CompileProgram)(nvrtcProgram_t, int, const char* const*) = nullptr;
  int (*GetProgramLogSize)(nvrtcProgram_t, size_t*) = nullptr;
  int (*GetProgramLog)(nvrtcProgram_t, char*) = nullptr;
  int (*GetCUBINSize)(nvrtcProgram_t, size_t*) = nullptr;
  int (*GetCUBIN)(nvrtcProgram_t, char*) = nullptr;
  int (*DestroyProgram)(nvrtcProgram_t*) = nullptr;
};

Driver g_cu;
Nvrtc g_rtc;
std::mutex g_init_mu;
bool g_driver_ok = false, g_nvrtc_ok = false;

template <typename F>
bool bind(void* h, F& fn, const char* name) {
  fn = reinterpret_cast<F>(dlsym(h, name));
  return fn != nullptr;
}

int load_nvrtc_locked() {
  if (g_nvrtc_ok) return 0;
  // the toolkit's NVRTC first (matches the nvcc that built this library)
  const char* names[] = {"/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12",
                         "libnvrtc.so", nullptr};
  for (int i = 0; names[i] && !g_rtc.handle; ++i)
    g_rtc.handle = dlopen(names[i], RTLD_NOW | RTLD_GLOBAL);
  if (!g_rtc.handle) return fail("tlb: cannot dlopen libnvrtc.so.12: %s", dlerror());
  void* h = g_rtc.handle;
  bool ok = bind(h, g_rtc.Version, "nvrtcVersion") &&
            bind(h, g_rtc.GetErrorString, "nvrtcGetErrorString") &&
            bind(h, g_rtc.CreateProgram, "nvrtcCreateProgram") &&
            bind(h, g_rtc.CompileProgram, "nvrtcCompileProgram") &&
            bind(h, g_rtc.GetProgramLogSize, "nvrtcGetProgramLogSize") &&
            bind(h, g_rtc.GetProgramLog, "nvrtcGetProgramLog") &&
            bind(h, g_rtc.GetCUBINSize, "nvrtcGetCUBINSize") &&
            bind(h, g_rtc.GetCUBIN, "nvrtcGetCUBIN") &&
            bind(h, g_rtc.DestroyProgram, "nvrtcDestroyProgram");
  if (!ok) return fail("tlb: libnvrtc lacks a required symbol");
  g_nvrtc_ok = true;
  return 0;
}

int load_driver_locked() {
  if (g_driver_ok) return 0;
  if (!g_cu.handle) g_cu.handle = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
  if (!g_cu.handle)
    return fail("tlb: no CUDA driver (dlopen libcuda.so.1 failed: %s) — a B200 is required",
                dlerror());
  void* h = g_cu.handle;
  bool ok = bind(h, g_cu.Init, "cuInit") && bind(h, g_cu.GetErrorString, "cuGetErrorString") &&
            bind(h, g_cu.CtxGetCurrent, "cuCtxGetCurrent") &&
            bind(h, g_cu.CtxSetCurrent, "cuCtxSetCurrent") &&
            bind(h, g_cu.CtxGetDevice, "cuCtxGetDevice") &&
            bind(h, g_cu.DeviceGet, "cuDeviceGet") &&
            bind(h, g_cu.DeviceGetAttribute, "cuDeviceGetAttribute") &&
            bind(h, g_cu.DevicePrimaryCtxRetain, "cuDevicePrimaryCtxRetain") &&
            bind(h, g_cu.StreamGetCtx, "cuStreamGetCtx") &&
            bind(h, g_cu.StreamCreate, "cuStreamCreate") &&
            bind(h, g_cu.StreamSynchronize, "cuStreamSynchronize") &&
            bind(h, g_cu.StreamWaitEvent, "cuStreamWaitEvent") &&
            bind(h, g_cu.EventCreate, "cuEventCreate") &&
            bind(h, g_cu.EventRecord, "cuEventRecord") &&
            bind(h, g_cu.EventDestroy, "cuEventDestroy_v2") &&
            bind(h, g_cu.ModuleLoadData, "cuModuleLoadData") &&
            bind(h, g_cu.ModuleUnload, "cuModuleUnload") &&
            bind(h, g_cu.CtxSynchronize, "cuCtxSynchronize") &&
            bind(h, g_cu.ModuleGetFunction, "cuModuleGetFunction") &&
            bind(h, g_cu.FuncGetAttribute, "cuFuncGetAttribute") &&
            bind(h, g_cu.FuncSetAttribute, "cuFuncSetAttribute") &&
            bind(h, g_cu.LaunchKernel, "cuLaunchKernel") &&
            bind(h, g_cu.OccupancyMaxActiveBlocksPerMultiprocessor,
                 "cuOccupancyMaxActiveBlocksPerMultiprocessor") &&
            bind(h, g_cu.MemAlloc, "cuMemAlloc_v2") && bind(h, g_cu.MemFree, "cuMemFree_v2") &&
            bind(h, g_cu.MemcpyHtoD, "cuMemcpyHtoD_v2") &&
            bind(h, g_cu.MemcpyHtoDAsync, "cuMemcpyHtoDAsync_v2") &&
            bind(h, g_cu.MemcpyDtoHAsync, "cuMemcpyDtoHAsync_v2") &&
            bind(h, g_cu.MemHostRegister, "cuMemHostRegister_v2") &&
            bind(h, g_cu.MemHostUnregister, "cuMemHostUnregister") &&
            bind(h, g_cu.PointerGetAttributes, "cuPointerGetAttributes") &&
            bind(h, g_cu.MemHostAlloc, "cuMemHostAlloc") &&
            bind(h, g_cu.MemFreeHost, "cuMemFreeHost") &&
            bind(h, g_cu.EventSynchronize, "cuEventSynchronize");
  if (!ok) return fail("tlb: libcuda.so.1 lacks a required symbol");
  CUresult r = g_cu.Init(0);
  if (r != CUDA_SUCCESS) return fail("tlb: cuInit failed (%d)", (int)r);
  g_driver_ok = true;
  return 0;
}

int ensure(bool driver) {
  std::lock_guard<std::mutex> lk(g_init_mu);
  if (load_nvrtc_locked() && !driver) return 1;
  if (driver) return load_driver_locked();
  return 0;
}

int cu_check(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return 0;
  const char* s = nullptr;
  if (g_cu.GetErrorString) g_cu.GetErrorString(r, &s);
  return fail("tlb: %s failed: %s (%d)", what, s ? s : "?", (int)r);
}

#define CU(call, what)                          \
  do {                                          \
    if (cu_check((call), (what))) return 1;     \
  } while (0)

// Resolve (and make current) the context a launch on `stream` must use.
int bind_context(void* stream, CUcontext* out) {
  CUcontext ctx = nullptr;
  if (stream) {
    CU(g_cu.StreamGetCtx((CUstream)stream, &ctx), "cuStreamGetCtx");
  } else {
    CU(g_cu.CtxGetCurrent(&ctx), "cuCtxGetCurrent");
    if (!ctx) {
      CUdevice dev;
      CU(g_cu.DeviceGet(&dev, 0), "cuDeviceGet");
      CU(g_cu.DevicePrimaryCtxRetain(&ctx, dev), "cuDevicePrimaryCtxRetain");
    }
  }
  CUcontext cur = nullptr;
  g_cu.CtxGetCurrent(&cur);
  if (cur != ctx) CU(g_cu.CtxSetCurrent(ctx), "cuCtxSetCurrent");
  *out = ctx;
  return 0;
}

// --------------------------------------------------- per-context state ----

constexpr int kStageBuffers = 3;  // host-staged pipeline depth (buffers = streams)
constexpr int kMaxStageSets = 2;  // concurrent host-staged runs per context

// One host-staged pipeline's device buffers and streams.  A tlb_exec_host
// call owns a set from acquisition until its final stream synchronisation;
// the context's lock is held only to pick or return a set, so launches and
// other staged runs (on this or any other context) never wait on a
// synchronisation they are not part of.
struct StageSet {
  CUstream side[kStageBuffers] = {};
  CUdeviceptr scratch = 0;
  size_t scratch_bytes = 0;
  // pinned host bounce ring for PAGEABLE callers (kStageBuffers x m x slab
  // doubles, kept across calls) and one completion event per buffer
  void* hpin = nullptr;
  size_t hpin_bytes = 0;
  CUevent done[kStageBuffers] = {};
  bool busy = false;
};

// Host copy workers for the pageable bounce path: run(ntasks, fn) calls
// fn(0..ntasks-1) across the pool and the calling thread, returning when
// all are done.  One run at a time (a mutex), workers created on first use.
class CopyPool {
 public:
  void run(long long ntasks, const std::function<void(long long)>& fn) {
    std::lock_guard<std::mutex> one(run_mu_);
    start();
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      ntasks_ = ntasks;
      next_.store(0);
      active_ = nworkers_;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return active_ == 0; });
    fn_ = nullptr;
  }

 private:
  void start() {
    // a forked child inherits the pool's state but none of its threads:
    // start its own
    if (started_ && pid_ == getpid()) return;
    started_ = true;
    pid_ = getpid();
    int n = (int)std::thread::hardware_concurrency();
    if (const char* e = getenv("TLB_COPY_THREADS")) n = atoi(e);
    n = std::max(1, std::min(n, 32));
    // detached: the pool lives for the process (never destroyed), so exit
    // never waits on or tears down a worker
    for (int i = 1; i < n; ++i) std::thread([this] { loop(); }).detach();
    nworkers_ = n - 1;
  }
  void work() {
    for (long long t; (t = next_.fetch_add(1)) < ntasks_;) (*fn_)(t);
  }
  void loop() {
    unsigned long long seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
      }
      work();
      std::lock_guard<std::mutex> lk(mu_);
      if (--active_ == 0) done_cv_.notify_all();
    }
  }
  std::mutex run_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  int nworkers_ = 0;
  const std::function<void(long long)>* fn_ = nullptr;
  std::atomic<long long> next_{0};
  long long ntasks_ = 0;
  int active_ = 0;
  unsigned long long gen_ = 0;
  bool started_ = false;
  pid_t pid_ = 0;
};
CopyPool& g_copy_pool = *new CopyPool;  // intentionally never destroyed

struct CopyTask {
  void* dst;
  const void* src;
  size_t bytes;
};

// memcpy of every task, split into <= 1 MiB pieces spread over the pool
void parallel_copy(const std::vector<CopyTask>& tasks) {
  constexpr size_t kPiece = 1 << 20;
  std::vector<CopyTask> pieces;
  for (const auto& t : tasks)
    for (size_t off = 0; off < t.bytes; off += kPiece)
      pieces.push_back({(char*)t.dst + off, (const char*)t.src + off,
                        std::min(kPiece, t.bytes - off)});
  g_copy_pool.run((long long)pieces.size(), [&](long long i) {
    memcpy(pieces[i].dst, pieces[i].src, pieces[i].bytes);
  });
}

struct CtxState {
  int sm_count = 0;
  std::mutex stage_mu;
  std::condition_variable stage_cv;
  std::vector<std::unique_ptr<StageSet>> sets;
};
std::mutex g_ctx_mu;  // the map only (lookups and first-use initialisation)
std::map<CUcontext, CtxState> g_ctx;

int ctx_state(CUcontext ctx, CtxState** out) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  CtxState& st = g_ctx[ctx];
  if (!st.sm_count) {
    CUdevice dev;
    CU(g_cu.CtxGetDevice(&dev), "cuCtxGetDevice");
    CU(g_cu.DeviceGetAttribute(&st.sm_count, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev),
       "cuDeviceGetAttribute");
  }
  *out = &st;
  return 0;
}

StageSet* acquire_stage_set(CtxState* st) {
  std::unique_lock<std::mutex> lk(st->stage_mu);
  for (;;) {
    for (auto& s : st->sets)
      if (!s->busy) {
        s->busy = true;
        return s.get();
      }
    if ((int)st->sets.size() < kMaxStageSets) {
      st->sets.emplace_back(new StageSet);
      st->sets.back()->busy = true;
      return st->sets.back().get();
    }
    st->stage_cv.wait(lk);
  }
}

void release_stage_set(CtxState* st, StageSet* set) {
  {
    std::lock_guard<std::mutex> lk(st->stage_mu);
    set->busy = false;
  }
  st->stage_cv.notify_one();
}

// Whether `p` is memory the driver knows (device, cudaHostAlloc'd or
// registered host memory).  cuPointerGetAttributes, unlike the singular
// cuPointerGetAttribute, answers "unknown" (memory type 0) for plain
// pageable memory without raising an API error — so sanitizer runs over
// host-staged calls stay free of expected-error reports.
bool driver_known(const void* p) {
  unsigned int mt = 0;
  CUpointer_attribute a = CU_POINTER_ATTRIBUTE_MEMORY_TYPE;
  void* data[] = {&mt};
  return g_cu.PointerGetAttributes(1, &a, data, (CUdeviceptr)p) == CUDA_SUCCESS && mt != 0;
}

// Page-lock pageable host ranges for the duration of one staged run
// (TLB_HOST_REGISTER=1), so the copies are DMA'd directly instead of
// through the driver's internal bounce buffers.  Ranges already pinned
// (cudaHostAlloc / torch pin_memory, or registered by the caller) are left
// alone; failures fall back to pageable copies.
struct HostPins {
  std::vector<void*> regs;
  ~HostPins() {
    for (void* p : regs) g_cu.MemHostUnregister(p);
  }
};

bool host_register_enabled() {
  const char* e = getenv("TLB_HOST_REGISTER");  // read per call (cheap next to a staged run)
  return e && atoi(e) != 0;
}

void pin_host_ranges(std::vector<std::pair<uintptr_t, uintptr_t>> spans, HostPins* pins) {
  const uintptr_t page = (uintptr_t)sysconf(_SC_PAGESIZE);
  for (auto& sp : spans) {
    sp.first = sp.first / page * page;
    sp.second = (sp.second + page - 1) / page * page;
  }
  std::sort(spans.begin(), spans.end());
  std::vector<std::pair<uintptr_t, uintptr_t>> merged;
  for (auto& sp : spans) {
    if (!merged.empty() && sp.first <= merged.back().second)
      merged.back().second = std::max(merged.back().second, sp.second);
    else
      merged.push_back(sp);
  }
  for (auto& m : merged) {
    if (driver_known((const void*)m.first)) continue;  // already page-locked (or device memory)
    void* p = (void*)m.first;
    if (g_cu.MemHostRegister(p, m.second - m.first, CU_MEMHOSTREGISTER_PORTABLE) == CUDA_SUCCESS)
      pins->regs.push_back(p);
  }
}

// ---------------------------------------------------------------- kernel ----

// STAGE_V1 / STAGE_BATCH_V1 (the TMA-staged entries) exist only in modules
// lowered with a staged variant; the others are in every module
enum Entry { FLAT_V1 = 0, FLAT_V2, BATCH_V1, BATCH_V2, STAGE_V1, STAGE_BATCH_V1, N_ENTRIES };
const char* kEntryNames[N_ENTRIES] = {"tlk_flat_v1",  "tlk_flat_v2",  "tlk_batch_v1",
                                      "tlk_batch_v2", "tlk_stage_v1", "tlk_stage_batch_v1"};

struct Loaded {
  CUmodule mod = nullptr;
  CUfunction fn[N_ENTRIES] = {};
  int occ[N_ENTRIES] = {};  // resident blocks per SM at the kernel's block size
};

}  // namespace

struct tlb_kernel {
  std::vector<char> cubin;
  std::string log;
  int nfields = 0;
  std::vector<int> slot_field;
  std::vector<long long> slot_comp;
  std::vector<int> slot_flags;
  int threads = 256;   // compiled TLK_THREADS: default block size (from the source)
  int stage_threads = 0;  // tile (points) of tlk_stage_v1 (from the source)
  int stage_block = 0;    // its block: the tile, + a producer warp when TLK_STAGE_WS
  // default launch geometry of the flat entry for callers that do not pass
  // one (tlb_exec_host, the harness bindings): TLK_GRID_WAVES (0 = one-shot
  // grid, w = w waves) and TLK_VEC (1 or 2 points per thread) from the source
  int dflt_waves = 1;
  int dflt_vec = 2;
  int batch_bound = 256;  // TLK_BATCH_BOUND: the batch entries' largest block
  int chunk = 1;          // TLK_CHUNK: block-sized runs per block in tlk_flat_v1
  int parts = 1;          // TLK_PARTS: independent statement parts (one block run each)
  int batch_parts = 1;    // ... run as (part, domain) row runs by tlk_batch_v1 (TLK_BATCH_SPLIT)
  int stage_smem = 0;     // its dynamic shared memory (from the source)
  int stage_batch_smem = 0;  // tlk_stage_batch_v1's: the ring + NSTAGE x NSLOTS pointers
  std::mutex mu;
  std::map<CUcontext, Loaded> loaded;
};

struct tlb_batch {
  tlb_kernel* k = nullptr;
  CUcontext ctx = nullptr;
  CUdeviceptr table = 0;
  CUdeviceptr items = 0;  // staged batch: {domain | count << 32, first point} per tile
  long long nitems = -1;  // -1: not built yet (first staged launch builds them)
  std::vector<long long> ns;
  int ndom = 0;
  long long max_n = 0;
  bool vec2 = false;
};

namespace {

int load_module(tlb_kernel* k, CUcontext ctx, Loaded** out) {
  std::lock_guard<std::mutex> lk(k->mu);
  auto it = k->loaded.find(ctx);
  if (it != k->loaded.end()) {
    *out = &it->second;
    return 0;
  }
  Loaded L;
  CU(g_cu.ModuleLoadData(&L.mod, k->cubin.data()), "cuModuleLoadData");
  for (int e = 0; e < N_ENTRIES; ++e) {
    int block = (e == BATCH_V1 || e == BATCH_V2) ? std::min(k->threads, k->batch_bound)
                                                  : k->threads,
        smem = 0;
    if (e == STAGE_V1 || e == STAGE_BATCH_V1) {
      smem = e == STAGE_V1 ? k->stage_smem : k->stage_batch_smem;
      block = e == STAGE_V1 ? k->stage_block : k->stage_threads + 32;
      if (smem <= 0 ||
          g_cu.ModuleGetFunction(&L.fn[e], L.mod, kEntryNames[e]) != CUDA_SUCCESS) {
        L.fn[e] = nullptr;
        continue;
      }
      CU(g_cu.FuncSetAttribute(L.fn[e], CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem),
         "cuFuncSetAttribute(stage smem)");
    } else {
      CU(g_cu.ModuleGetFunction(&L.fn[e], L.mod, kEntryNames[e]), kEntryNames[e]);
    }
    CU(g_cu.OccupancyMaxActiveBlocksPerMultiprocessor(&L.occ[e], L.fn[e], block, smem),
       "cuOccupancyMaxActiveBlocksPerMultiprocessor");
    if (L.occ[e] < 1) L.occ[e] = 1;
  }
  *out = &(k->loaded[ctx] = L);
  return 0;
}

bool file_exists(const char* p) {
  struct stat sb;
  return p && *p && stat(p, &sb) == 0 && S_ISREG(sb.st_mode);
}

bool read_file(const char* p, std::vector<char>* out) {
  FILE* f = fopen(p, "rb");
  if (!f) return false;
  fseek(f, 0, SEEK_END);
  long sz = ftell(f);
  fseek(f, 0, SEEK_SET);
  out->resize(sz > 0 ? (size_t)sz : 0);
  bool ok = sz > 0 && fread(out->data(), 1, (size_t)sz, f) == (size_t)sz;
  fclose(f);
  return ok;
}

void write_file_atomic(const char* p, const std::vector<char>& data) {
  std::string tmp = std::string(p) + ".tmp." + std::to_string((long)getpid());
  FILE* f = fopen(tmp.c_str(), "wb");
  if (!f) return;  // cache is best effort
  bool ok = fwrite(data.data(), 1, data.size(), f) == data.size();
  ok = (fclose(f) == 0) && ok;
  if (ok) rename(tmp.c_str(), p);
  else unlink(tmp.c_str());
}

// Per-slot device addresses of one grid from field bases and pitches.
int resolve_slots(const tlb_kernel* k, const void* const* bases, const long long* pitches,
                  uint64_t* out, bool* aligned16) {
  bool al = true;
  for (size_t j = 0; j < k->slot_field.size(); ++j) {
    int f = k->slot_field[j];
    if (!bases[f]) return fail("tlb: field %d has a null base pointer", f);
    uint64_t a = (uint64_t)(uintptr_t)bases[f] +
                 (uint64_t)(k->slot_comp[j] * pitches[f]) * sizeof(double);
    out[j] = a;
    al = al && (a % 16 == 0);
  }
  *aligned16 = al;
  return 0;
}

}  // namespace

__attribute__((visibility("hidden"))) void tlb_internal_set_error(const char* msg) {
  g_err = std::string("tlb: ") + msg;
}

// ================================================================ C-ABI ====

extern "C" {

int tlb_abi_version(void) { return TLB_ABI_VERSION; }

int tlb_init(int want_driver) { return ensure(want_driver != 0); }

const char* tlb_last_error(void) { return g_err.c_str(); }

int tlb_nvrtc_version(int* major, int* minor) {
  if (ensure(false)) return 1;
  int r = g_rtc.Version(major, minor);
  return r ? fail("tlb: nvrtcVersion failed (%d)", r) : 0;
}

int tlb_device_sm_count(int* out) {
  if (ensure(true)) return 1;
  CUcontext ctx;
  if (bind_context(nullptr, &ctx)) return 1;
  CtxState* st;
  if (ctx_state(ctx, &st)) return 1;
  *out = st->sm_count;
  return 0;
}

// Value of `#define NAME <int>` in a generated source (lowering.py writes the
// launch geometry there), or `dflt`.
// A numeric `#define NAME value` of the generated header.  Only the header
// is searched (it ends where the template's own text begins), so the
// template's `#ifndef NAME / #define NAME <fallback expression>` defaults
// never shadow an absent header define; a non-numeric value also yields
// `dflt`.
static long long source_define(const char* src, const char* name, long long dflt) {
  const std::string key = std::string("#define ") + name + " ";
  const char* end = strstr(src, "// tlk_template.cuh");
  const char* p = strstr(src, key.c_str());
  if (!p || (end && p > end)) return dflt;
  const char* v = p + key.size();
  if (!(*v == '-' || (*v >= '0' && *v <= '9'))) return dflt;
  return atoll(v);
}

int tlb_compile(const char* src, const char* const* opts, int nopts, const char* cache_path,
                tlb_kernel** out) {
  if (!src || !out) return fail("tlb_compile: null argument");
  std::unique_ptr<tlb_kernel> k(new tlb_kernel);
  // launch geometry from the source: block size, and the staged entry's
  // tile ring (TLK_NSTAGE x TLK_NREAD x TLK_THREADS doubles)
  k->threads = (int)source_define(src, "TLK_THREADS", 256);
  k->batch_bound = (int)source_define(src, "TLK_BATCH_BOUND", k->threads);
  k->chunk = (int)std::max(1LL, source_define(src, "TLK_CHUNK", 1));
  k->parts = (int)std::max(1LL, source_define(src, "TLK_PARTS", 1));
  k->batch_parts = source_define(src, "TLK_BATCH_SPLIT", 0) ? k->parts : 1;
  k->dflt_waves = (int)source_define(src, "TLK_GRID_WAVES", 1);
  k->dflt_vec = (int)source_define(src, "TLK_VEC", 2) == 1 ? 1 : 2;
  const long long nstage = source_define(src, "TLK_NSTAGE", 0);
  if (k->threads < 32 || k->threads > 1024 || k->threads % 32)
    return fail("tlb_compile: TLK_THREADS %d is not a block size", k->threads);
  if (nstage > 0) {
    k->stage_threads = (int)source_define(src, "TLK_STAGE_THREADS", 128);
    if (k->stage_threads < 32 || k->stage_threads > 1024 || k->stage_threads % 32)
      return fail("tlb_compile: TLK_STAGE_THREADS %d is not a block size", k->stage_threads);
    k->stage_block = k->stage_threads + (source_define(src, "TLK_STAGE_WS", 0) ? 32 : 0);
    if (k->stage_block > 1024)
      return fail("tlb_compile: staged block of %d threads", k->stage_block);
    const long long smem =
        nstage * source_define(src, "TLK_NREAD", 1) * k->stage_threads * 8;
    if (smem > 227 * 1024) return fail("tlb_compile: staged tile ring of %lld bytes", smem);
    k->stage_smem = (int)smem;
    const long long bsmem = smem + nstage * source_define(src, "TLK_NSLOTS", 0) * 8;
    // the staged batch entry is compiled only into modules that ask for it
    // (TLK_STAGE_BATCH, lowering Variant.batch_vec = 3); 0: no staged batch
    k->stage_batch_smem =
        source_define(src, "TLK_STAGE_BATCH", 0) && bsmem <= 227 * 1024 ? (int)bsmem : 0;
  }
  if (file_exists(cache_path) && read_file(cache_path, &k->cubin)) {
    *out = k.release();
    return 0;
  }
  if (ensure(false)) return 1;
  nvrtcProgram_t prog = nullptr;
  int r = g_rtc.CreateProgram(&prog, src, "tlb_fused.cu", 0, nullptr, nullptr);
  if (r) return fail("tlb: nvrtcCreateProgram: %s", g_rtc.GetErrorString(r));
  r = g_rtc.CompileProgram(prog, nopts, opts);
  size_t log_size = 0;
  g_rtc.GetProgramLogSize(prog, &log_size);
  if (log_size > 1) {
    k->log.resize(log_size);
    g_rtc.GetProgramLog(prog, &k->log[0]);
    k->log.resize(strlen(k->log.c_str()));
  }
  if (r) {
    std::string msg = "tlb: NVRTC compile failed: " + std::string(g_rtc.GetErrorString(r)) +
                      "\n" + k->log;
    g_rtc.DestroyProgram(&prog);
    g_err = msg;
    return 1;
  }
  size_t n = 0;
  g_rtc.GetCUBINSize(prog, &n);
  if (n == 0) {
    g_rtc.DestroyProgram(&prog);
    return fail("tlb: NVRTC produced no cubin (is --gpu-architecture a real sm_ target?)");
  }
  k->cubin.resize(n);
  g_rtc.GetCUBIN(prog, k->cubin.data());
  g_rtc.DestroyProgram(&prog);
  if (cache_path && *cache_path) write_file_atomic(cache_path, k->cubin);
  *out = k.release();
  return 0;
}

const char* tlb_kernel_log(const tlb_kernel* k) { return k ? k->log.c_str() : ""; }

int tlb_kernel_cubin(const tlb_kernel* k, const void** data, long long* size) {
  if (!k) return fail("tlb_kernel_cubin: null kernel");
  *data = k->cubin.data();
  *size = (long long)k->cubin.size();
  return 0;
}

void tlb_kernel_destroy(tlb_kernel* k) {
  if (!k) return;
  if (g_driver_ok && !k->loaded.empty()) {
    // unload the module from every context it was loaded into, after that
    // context's pending work (a launch of it may still be queued)
    CUcontext cur = nullptr;
    g_cu.CtxGetCurrent(&cur);
    for (auto& kv : k->loaded) {
      if (g_cu.CtxSetCurrent(kv.first) != CUDA_SUCCESS) continue;
      g_cu.CtxSynchronize();
      g_cu.ModuleUnload(kv.second.mod);
    }
    g_cu.CtxSetCurrent(cur);
  }
  delete k;
}

int tlb_kernel_set_slots(tlb_kernel* k, int nfields, int nslots, const int* slot_field,
                         const long long* slot_comp, const int* slot_flags) {
  if (!k || nfields < 0 || nslots < 1) return fail("tlb_kernel_set_slots: bad arguments");
  for (int j = 0; j < nslots; ++j)
    if (slot_field[j] < 0 || slot_field[j] >= nfields || slot_comp[j] < 0)
      return fail("tlb_kernel_set_slots: slot %d out of range", j);
  k->nfields = nfields;
  k->slot_field.assign(slot_field, slot_field + nslots);
  k->slot_comp.assign(slot_comp, slot_comp + nslots);
  k->slot_flags.assign(slot_flags, slot_flags + nslots);
  return 0;
}

int tlb_kernel_attrs(tlb_kernel* k, const char* entry, int* regs, int* local_bytes,
                     int* max_threads) {
  if (ensure(true)) return 1;
  CUcontext ctx;
  if (bind_context(nullptr, &ctx)) return 1;
  Loaded* L;
  if (load_module(k, ctx, &L)) return 1;
  for (int e = 0; e < N_ENTRIES; ++e) {
    if (strcmp(entry, kEntryNames[e])) continue;
    if (!L->fn[e]) return fail("tlb_kernel_attrs: entry %s not in this module", entry);
    CU(g_cu.FuncGetAttribute(regs, CU_FUNC_ATTRIBUTE_NUM_REGS, L->fn[e]), "attr regs");
    CU(g_cu.FuncGetAttribute(local_bytes, CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, L->fn[e]),
       "attr local");
    CU(g_cu.FuncGetAttribute(max_threads, CU_FUNC_ATTRIBUTE_MAX_THREADS_PER_BLOCK, L->fn[e]),
       "attr threads");
    return 0;
  }
  return fail("tlb_kernel_attrs: unknown entry %s", entry);
}

namespace {

static int launch_flat(tlb_kernel* k, Loaded* L, CtxState* st, long long n,
                       const uint64_t* slots, bool vec2, int threads, long long max_blocks,
                       CUstream stream, bool stage = false) {
  const size_t m = k->slot_field.size();
  // parameter block: { long long n; double* p[m]; } — passed by value
  std::vector<uint64_t> param(1 + m);
  param[0] = (uint64_t)n;
  memcpy(&param[1], slots, m * sizeof(uint64_t));
  if (threads <= 0) threads = k->threads;
  if (stage) {
    // persistent: one block per resident slot, each walks whole tiles of the
    // compiled TLK_STAGE_THREADS points (block: the tile, + a producer warp
    // in the warp-specialised form)
    threads = k->stage_block;
    // (max_blocks > 0: that many blocks, at most one per tile — e.g. one
    // block per tile, a one-shot grid instead of a persistent one)
    long long tiles = std::max(1LL, n / k->stage_threads);
    long long blocks = max_blocks > 0
                           ? std::min(tiles, max_blocks)
                           : std::min<long long>(tiles, (long long)st->sm_count * L->occ[STAGE_V1]);
    void* args[] = {param.data()};
    CU(g_cu.LaunchKernel(L->fn[STAGE_V1], (unsigned)blocks, 1, 1, (unsigned)threads, 1, 1,
                         (unsigned)k->stage_smem, stream, args, nullptr),
       "cuLaunchKernel(stage)");
    return 0;
  }
  const int e = vec2 ? FLAT_V2 : FLAT_V1;
  long long units = vec2 ? n / 2 : n;
  if (units < 1) units = 1;
  if (max_blocks >= TLB_ONE_SHOT && units < (long long)st->sm_count * 4 * threads) {
    // one-shot grid of a small launch: smaller blocks, so that every SM
    // gets ~4 of them (a 512-thread block per 512 points would leave most
    // SMs idle below ~300K points)
    const long long per = (units + st->sm_count * 4 - 1) / (st->sm_count * 4);
    threads = (int)std::max(64LL, std::min<long long>(threads, (per + 31) / 32 * 32));
  }
  long long blocks = (units + threads - 1) / threads;
  if (!vec2 && k->chunk > 1) blocks = (blocks + k->chunk - 1) / k->chunk;
  // max_blocks > 0: explicit cap; 0: one full wave at occupancy; -w: w waves
  int occ = L->occ[e];
  if (threads != k->threads) {
    g_cu.OccupancyMaxActiveBlocksPerMultiprocessor(&occ, L->fn[e], threads, 0);
    occ = std::max(occ, 1);
  }
  long long waves = max_blocks < 0 ? -max_blocks : 1;
  long long cap = max_blocks > 0 ? max_blocks : (long long)st->sm_count * occ * waves;
  if (!vec2 && k->parts > 1) {
    // tlk_flat_v1 under TLK_PARTS: one equal run of blocks per part (each run
    // a full one-shot grid of the points; a capped grid shares the cap)
    const long long p = k->parts;
    blocks = std::max(1LL, std::min(std::min(blocks, std::max(1LL, cap / p)), 0x7fffffffLL / p));
    blocks *= p;
  } else {
    blocks = std::max(1LL, std::min(std::min(blocks, cap), 0x7fffffffLL));
  }
  void* args[] = {param.data()};
  CU(g_cu.LaunchKernel(L->fn[e], (unsigned)blocks, 1, 1, (unsigned)threads, 1, 1, 0, stream,
                       args, nullptr),
     "cuLaunchKernel(flat)");
  return 0;
}

}  // namespace

int tlb_launch(tlb_kernel* k, long long n, const void* const* field_bases,
               const long long* pitches, int vec, int threads, long long max_blocks,
               void* stream) {
  if (!k || k->slot_field.empty()) return fail("tlb_launch: kernel has no slots");
  if (n < 0) return fail("tlb_launch: negative point count");
  if (n == 0) return 0;
  if (ensure(true)) return 1;
  CUcontext ctx;
  if (bind_context(stream, &ctx)) return 1;
  CtxState* st;
  if (ctx_state(ctx, &st)) return 1;
  Loaded* L;
  if (load_module(k, ctx, &L)) return 1;
  std::vector<uint64_t> slots(k->slot_field.size());
  bool al;
  if (resolve_slots(k, field_bases, pitches, slots.data(), &al)) return 1;
  if (vec == 3) {
    // TMA-staged entry: bulk copies need 16-byte aligned sources (its block
    // size is the compiled tile; `threads` applies to the plain entries)
    if (!L->fn[STAGE_V1]) return fail("tlb_launch: vec=3 but the module has no staged entry");
    if (al)
      return launch_flat(k, L, st, n, slots.data(), false, threads, max_blocks,
                         (CUstream)stream, true);
    vec = 1;  // unaligned slab view: the plain 1-point entry (same results)
  }
  bool vec2 = vec == 2 ? true : (vec == 1 ? false : al);
  if (vec2 && !al) return fail("tlb_launch: vec=2 requested but a slot is not 16-byte aligned");
  return launch_flat(k, L, st, n, slots.data(), vec2, threads, max_blocks, (CUstream)stream);
}

int tlb_launch_default(tlb_kernel* k, long long n, const void* const* field_bases,
                       const long long* pitches, void* stream) {
  if (!k) return fail("tlb_launch_default: null kernel");
  // the lowering's geometry from the source: TLK_VEC 2 = the 2-point entry
  // where every slot is 16-byte aligned (vec 0), 1 = the 1-point entry; a
  // staged module takes its staged entry; TLK_GRID_WAVES 0 = one-shot grid,
  // w = w waves of resident blocks
  const int vec = k->stage_threads > 0 ? 3 : (k->dflt_vec == 2 ? 0 : 1);
  const long long mb = k->dflt_waves == 0 ? TLB_ONE_SHOT
                                          : (k->dflt_waves > 1 ? -(long long)k->dflt_waves : 0);
  return tlb_launch(k, n, field_bases, pitches, vec, 0, mb, stream);
}

// $TLB_CACHE_DIR, else <directory of this library>/_kcache (created if
// missing); empty when neither is usable
static std::string harness_cache_dir() {
  if (const char* e = getenv("TLB_CACHE_DIR")) return e;
  Dl_info info;
  if (!dladdr((void*)&tlb_harness_call, &info) || !info.dli_fname) return "";
  std::string lib = info.dli_fname;
  const size_t slash = lib.rfind('/');
  std::string dir = (slash == std::string::npos ? std::string(".") : lib.substr(0, slash)) +
                    "/_kcache";
  mkdir(dir.c_str(), 0755);
  struct stat sb;
  return stat(dir.c_str(), &sb) == 0 && S_ISDIR(sb.st_mode) ? dir : "";
}

int tlb_batch_create(tlb_kernel* k, int ndom, const void* const* field_bases,
                     const long long* pitches, const long long* ns, void* stream,
                     tlb_batch** out) {
  if (!k || k->slot_field.empty() || ndom < 1) return fail("tlb_batch_create: bad arguments");
  if (ensure(true)) return 1;
  CUcontext ctx;
  if (bind_context(stream, &ctx)) return 1;
  const size_t m = k->slot_field.size();
  const int nf = k->nfields;
  // device record per domain: { long long n; double* p[m]; }
  std::vector<uint64_t> table((size_t)ndom * (1 + m));
  bool all_al = true;
  long long max_n = 0;
  for (int d = 0; d < ndom; ++d) {
    uint64_t* rec = &table[(size_t)d * (1 + m)];
    rec[0] = (uint64_t)ns[d];
    bool al;
    if (resolve_slots(k, field_bases + (size_t)d * nf, pitches + (size_t)d * nf, rec + 1, &al))
      return 1;
    all_al = all_al && al;
    max_n = std::max(max_n, ns[d]);
  }
  std::unique_ptr<tlb_batch> b(new tlb_batch);
  b->k = k;
  b->ctx = ctx;
  b->ndom = ndom;
  b->max_n = max_n;
  b->vec2 = all_al;
  CU(g_cu.MemAlloc(&b->table, table.size() * sizeof(uint64_t)), "cuMemAlloc(batch table)");
  CU(g_cu.MemcpyHtoD(b->table, table.data(), table.size() * sizeof(uint64_t)),
     "cuMemcpyHtoD(batch table)");
  if (k->stage_batch_smem > 0) b->ns.assign(ns, ns + ndom);  // staged items: built on demand
  *out = b.release();
  return 0;
}

int tlb_batch_launch(tlb_batch* b, int vec, int threads, void* stream) {
  if (!b) return fail("tlb_batch_launch: null batch");
  if (ensure(true)) return 1;
  CUcontext ctx;
  if (bind_context(stream, &ctx)) return 1;
  if (ctx != b->ctx) return fail("tlb_batch_launch: stream belongs to another context");
  CtxState* st;
  if (ctx_state(ctx, &st)) return 1;
  Loaded* L;
  if (load_module(b->k, ctx, &L)) return 1;
  if (vec == 3 && L->fn[STAGE_BATCH_V1] && b->nitems < 0) {
    // work items of the staged batch entry: every (domain, tile) pair
    const long long tile = b->k->stage_threads;
    std::vector<long long> items;
    for (size_t d = 0; d < b->ns.size(); ++d)
      for (long long x = 0; x < b->ns[d]; x += tile) {
        const long long cnt = std::min(tile, b->ns[d] - x);
        items.push_back((long long)d | (cnt << 32));
        items.push_back(x);
      }
    if (!items.empty()) {
      CU(g_cu.MemAlloc(&b->items, items.size() * sizeof(long long)), "cuMemAlloc(batch items)");
      CU(g_cu.MemcpyHtoD(b->items, items.data(), items.size() * sizeof(long long)),
         "cuMemcpyHtoD(batch items)");
    }
    b->nitems = (long long)items.size() / 2;
  }
  if (vec == 3 && b->nitems == 0) return 0;  // only empty domains
  if (vec == 3 && b->items && L->fn[STAGE_BATCH_V1]) {
    // staged batch: persistent blocks of stage_threads consumers + a producer warp
    long long blocks =
        std::min<long long>(b->nitems, (long long)st->sm_count * L->occ[STAGE_BATCH_V1]);
    CUdeviceptr table = b->table, items = b->items;
    long long nitems = b->nitems;
    void* args[] = {&table, &items, &nitems};
    CU(g_cu.LaunchKernel(L->fn[STAGE_BATCH_V1], (unsigned)std::max(1LL, blocks), 1, 1,
                         (unsigned)(b->k->stage_threads + 32), 1, 1,
                         (unsigned)b->k->stage_batch_smem, (CUstream)stream, args, nullptr),
       "cuLaunchKernel(stage batch)");
    return 0;
  }
  if (vec == 3) vec = 1;  // no staged batch entry: the 1-point batch entry
  const bool v2 = b->vec2 && vec != 1;
  const int e = v2 ? BATCH_V2 : BATCH_V1;
  if (threads <= 0) threads = std::min(b->k->threads, b->k->batch_bound);
  if (threads > b->k->batch_bound)
    return fail("tlb_batch_launch: %d threads exceed the batch entry's bound %d", threads,
                b->k->batch_bound);
  long long units = v2 ? (b->max_n + 1) / 2 : b->max_n;
  long long gx = std::max(1LL, (units + threads - 1) / threads);
  long long gy = std::min<long long>((long long)b->ndom * (v2 ? 1 : b->k->batch_parts), 65535);
  // optional cap of the grid at a few waves (TLB_BATCH_WAVES; default 0 =
  // one block per (domain, chunk): measured 190 us vs 195 us at 4 waves for
  // C4); capped blocks loop over x chunks and domains
  static const long long waves = [] {
    const char* e = getenv("TLB_BATCH_WAVES");
    return e ? atoll(e) : 0LL;
  }();
  if (waves > 0) {
    long long cap = (long long)st->sm_count * L->occ[e] * waves;
    if (gx * gy > cap) gx = std::max(1LL, cap / gy);
  }
  // tuning knob (TLB_BATCH_CHUNKS=c): c chunks of a domain per block, so a
  // block stages the domain's slot pointers once per c x threads points
  static const long long chunks = [] {
    const char* e = getenv("TLB_BATCH_CHUNKS");
    return e ? std::max(1LL, atoll(e)) : 1LL;
  }();
  if (chunks > 1) gx = std::max(1LL, (gx + chunks - 1) / chunks);
  CUdeviceptr table = b->table;
  int ndom = b->ndom;
  void* args[] = {&table, &ndom};
  CU(g_cu.LaunchKernel(L->fn[e], (unsigned)gx, (unsigned)gy, 1, (unsigned)threads, 1, 1, 0,
                       (CUstream)stream, args, nullptr),
     "cuLaunchKernel(batch)");
  return 0;
}

void tlb_batch_destroy(tlb_batch* b) {
  if (!b) return;
  if (b->table && g_driver_ok) {
    CUcontext cur = nullptr;
    g_cu.CtxGetCurrent(&cur);
    if (cur != b->ctx) g_cu.CtxSetCurrent(b->ctx);
    g_cu.CtxSynchronize();  // a queued batch launch may still read the table
    g_cu.MemFree(b->table);
    if (b->items) g_cu.MemFree(b->items);
    if (cur && cur != b->ctx) g_cu.CtxSetCurrent(cur);
  }
  delete b;
}

int tlb_exec_host(tlb_kernel* k, long long n, const double* const* const* comp_ptrs,
                  long long slab, void* stream) {
  if (!k || k->slot_field.empty()) return fail("tlb_exec_host: kernel has no slots");
  if (n < 0) return fail("tlb_exec_host: negative point count");
  if (n == 0) return 0;
  if (ensure(true)) return 1;
  CUcontext ctx;
  if (bind_context(stream, &ctx)) return 1;
  CtxState* st;
  if (ctx_state(ctx, &st)) return 1;
  Loaded* L;
  if (load_module(k, ctx, &L)) return 1;
  const size_t m = k->slot_field.size();
  const int nb = kStageBuffers;
  // pageable host arrays (not cudaHostAlloc'd, not registered): unless the
  // caller asks for registration, copy them through a pinned bounce ring with
  // the host copy pool, overlapped with the DMA of the neighbouring slabs —
  // instead of the driver's serial internal staging of pageable copies
  bool bounce = false;
  const bool do_register = host_register_enabled();
  if (!do_register) {
    for (size_t j = 0; j < m && !bounce; ++j)
      bounce = !driver_known(comp_ptrs[k->slot_field[j]][k->slot_comp[j]]);
  }
  if (slab <= 0) {
    // nb buffers of m*slab doubles, at most ~4 GiB in total; bounced runs use
    // ~64 MiB per buffer (the pinned ring is the same size on the host)
    long long cap = (bounce ? (64LL << 20) * nb : (4LL << 30)) /
                    (long long)(nb * m * sizeof(double));
    slab = std::min<long long>(n, std::max<long long>(bounce ? 4096 : 1 << 16, cap));
  }
  if (bounce)  // an explicit slab too: the pinned ring stays ~64 MiB per buffer
    slab = std::min<long long>(
        slab, std::max<long long>(4096, (64LL << 20) / (long long)(m * sizeof(double))));
  slab = std::min(slab, n);
  slab = (slab + 255) / 256 * 256;  // keeps every slot slice 2 KiB aligned
  HostPins pins;
  if (do_register) {
    std::vector<std::pair<uintptr_t, uintptr_t>> spans;
    for (size_t j = 0; j < m; ++j) {
      const uintptr_t a = (uintptr_t)(comp_ptrs[k->slot_field[j]][k->slot_comp[j]]);
      spans.emplace_back(a, a + (uintptr_t)n * sizeof(double));
    }
    pin_host_ranges(std::move(spans), &pins);
  }
  StageSet* set = acquire_stage_set(st);
  struct Release {
    CtxState* st;
    StageSet* set;
    ~Release() { release_stage_set(st, set); }
  } release{st, set};
  size_t need = (size_t)nb * m * (size_t)slab * sizeof(double);
  if (set->scratch_bytes < need) {
    if (set->scratch) g_cu.MemFree(set->scratch);
    set->scratch = 0;
    set->scratch_bytes = 0;
    CU(g_cu.MemAlloc(&set->scratch, need), "cuMemAlloc(staging)");
    set->scratch_bytes = need;
  }
  for (int s = 0; s < nb; ++s)
    if (!set->side[s])
      CU(g_cu.StreamCreate(&set->side[s], CU_STREAM_NON_BLOCKING), "cuStreamCreate");
  if (bounce) {
    if (set->hpin_bytes < need) {
      if (set->hpin) g_cu.MemFreeHost(set->hpin);
      set->hpin = nullptr;
      set->hpin_bytes = 0;
      CU(g_cu.MemHostAlloc(&set->hpin, need, CU_MEMHOSTALLOC_PORTABLE), "cuMemHostAlloc(bounce)");
      set->hpin_bytes = need;
    }
    for (int s = 0; s < nb; ++s)
      if (!set->done[s])
        CU(g_cu.EventCreate(&set->done[s], CU_EVENT_DISABLE_TIMING), "cuEventCreate");
  }
  // order after prior work of the caller's stream
  CUevent ev;
  CU(g_cu.EventCreate(&ev, CU_EVENT_DISABLE_TIMING), "cuEventCreate");
  CU(g_cu.EventRecord(ev, (CUstream)stream), "cuEventRecord");
  for (int s = 0; s < nb; ++s)
    CU(g_cu.StreamWaitEvent(set->side[s], ev, 0), "cuStreamWaitEvent");
  g_cu.EventDestroy(ev);
  std::vector<uint64_t> slots(m);
  // bounce ring: buffer b holds slot j of its slab at hpin + (b*m + j)*slab
  auto pinned = [&](int b, size_t j) {
    return (double*)set->hpin + ((size_t)b * m + j) * (size_t)slab;
  };
  struct Pending {
    long long lo = -1, cnt = 0;
  } pend[kStageBuffers];
  auto drain = [&](int b) -> int {  // outputs of buffer b's slab: pinned -> caller
    if (pend[b].lo < 0) return 0;
    CU(g_cu.EventSynchronize(set->done[b]), "cuEventSynchronize(bounce)");
    std::vector<CopyTask> out;
    for (size_t j = 0; j < m; ++j)
      if (k->slot_flags[j] & TLB_SLOT_WRITE)
        out.push_back({const_cast<double*>(comp_ptrs[k->slot_field[j]][k->slot_comp[j]]) +
                           pend[b].lo,
                       pinned(b, j), (size_t)pend[b].cnt * sizeof(double)});
    parallel_copy(out);
    pend[b].lo = -1;
    return 0;
  };
  long long slab_idx = 0;
  for (long long lo = 0; lo < n; lo += slab, ++slab_idx) {
    const long long cnt = std::min(slab, n - lo);
    const int b = (int)(slab_idx % nb);
    CUstream s = set->side[b];
    CUdeviceptr buf = set->scratch + (size_t)b * m * (size_t)slab * sizeof(double);
    if (bounce) {
      if (drain(b)) return 1;  // buffer b's previous slab (nb slabs ago) is done
      std::vector<CopyTask> in;
      for (size_t j = 0; j < m; ++j)
        if (k->slot_flags[j] & TLB_SLOT_READ)
          in.push_back({pinned(b, j), comp_ptrs[k->slot_field[j]][k->slot_comp[j]] + lo,
                        (size_t)cnt * sizeof(double)});
      parallel_copy(in);
    }
    for (size_t j = 0; j < m; ++j) {
      slots[j] = buf + j * (size_t)slab * sizeof(double);
      if (k->slot_flags[j] & TLB_SLOT_READ) {
        const double* src =
            bounce ? pinned(b, j) : comp_ptrs[k->slot_field[j]][k->slot_comp[j]] + lo;
        CU(g_cu.MemcpyHtoDAsync(slots[j], src, (size_t)cnt * sizeof(double), s), "H2D");
      }
    }
    // the kernel's own launch geometry (staging buffers are 16-byte aligned)
    if (launch_flat(k, L, st, cnt, slots.data(), k->dflt_vec == 2, 0,
                    k->dflt_waves == 0 ? TLB_ONE_SHOT
                                       : (k->dflt_waves > 1 ? -k->dflt_waves : 0),
                    s))
      return 1;
    for (size_t j = 0; j < m; ++j) {
      if (k->slot_flags[j] & TLB_SLOT_WRITE) {
        double* dst = bounce ? pinned(b, j)
                             : const_cast<double*>(comp_ptrs[k->slot_field[j]][k->slot_comp[j]]) +
                                   lo;
        CU(g_cu.MemcpyDtoHAsync(dst, slots[j], (size_t)cnt * sizeof(double), s), "D2H");
      }
    }
    if (bounce) {
      CU(g_cu.EventRecord(set->done[b], s), "cuEventRecord(bounce)");
      pend[b].lo = lo;
      pend[b].cnt = cnt;
    }
  }
  if (bounce)  // the last nb slabs, oldest first
    for (long long i = std::max(0LL, slab_idx - nb); i < slab_idx; ++i)
      if (drain((int)(i % nb))) return 1;
  for (int s = 0; s < nb; ++s)
    CU(g_cu.StreamSynchronize(set->side[s]), "cuStreamSynchronize");
  return 0;
}

int tlb_release_staging(void) {
  if (!g_driver_ok) return 0;
  CUcontext ctx = nullptr;
  g_cu.CtxGetCurrent(&ctx);
  CtxState* st = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    auto it = g_ctx.find(ctx);
    if (it == g_ctx.end()) return 0;
    st = &it->second;
  }
  std::lock_guard<std::mutex> lk(st->stage_mu);
  for (auto& set : st->sets) {
    if (set->busy) continue;  // a running pipeline keeps its buffers
    if (set->scratch) CU(g_cu.MemFree(set->scratch), "cuMemFree(staging)");
    set->scratch = 0;
    set->scratch_bytes = 0;
    if (set->hpin) CU(g_cu.MemFreeHost(set->hpin), "cuMemFreeHost(bounce)");
    set->hpin = nullptr;
    set->hpin_bytes = 0;
  }
  return 0;
}

int tlb_harness_call(tlb_harness_kernel* hk, long n, double** const* tensors,
                     const double* const* scalars) {
  if (!hk) return fail("tlb_harness_call: null kernel");
  static std::mutex mu;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!hk->compiled) {
      // on-disk cubin cache keyed by FNV-1a of source + options: $TLB_CACHE_DIR,
      // else the library's own kernel cache (<dir of libtlb200.so>/_kcache, the
      // Python side's default too), where Registry.build_shared precompiles
      // every entry — a harness process then loads cubins instead of running NVRTC
      std::string cache;
      std::string dir_s = harness_cache_dir();
      if (!dir_s.empty()) {
        const char* dir = dir_s.c_str();
        uint64_t h = 1469598103934665603ull;
        auto mixin = [&h](const char* p) {
          for (; *p; ++p) h = (h ^ (unsigned char)*p) * 1099511628211ull;
          h = (h ^ 0xff) * 1099511628211ull;
        };
        mixin(hk->source);
        for (int i = 0; i < hk->nopts; ++i) mixin(hk->opts[i]);
        char name[40];
        snprintf(name, sizeof name, "/harness_%016llx.cubin", (unsigned long long)h);
        cache = std::string(dir) + name;
      }
      tlb_kernel* k = nullptr;
      if (tlb_compile(hk->source, hk->opts, hk->nopts, cache.empty() ? nullptr : cache.c_str(),
                      &k))
        return 1;
      if (tlb_kernel_set_slots(k, hk->nfields, hk->nslots, hk->slot_field, hk->slot_comp,
                               hk->slot_flags)) {
        tlb_kernel_destroy(k);
        return 1;
      }
      hk->compiled = k;
    }
  }
  // host address of every component of every kernel field
  std::vector<std::vector<const double*>> comps(hk->nfields);
  std::vector<const double* const*> rows(hk->nfields);
  for (int f = 0; f < hk->nfields; ++f) {
    if (hk->field_kind[f] == 1) {
      comps[f].push_back(scalars[hk->field_arg[f]]);
    } else {
      double** const flat = tensors[hk->field_arg[f]];
      for (int c = 0; c < hk->field_ncomp[f]; ++c)
        comps[f].push_back(flat[hk->field_comp_flat[f][c]]);
    }
    rows[f] = comps[f].data();
  }
  return tlb_exec_host(hk->compiled, n, rows.data(), 0, nullptr);
}

}  // extern "C"

import ctypes, time
t0 = time.perf_counter()
cu = ctypes.CDLL("libcuda.so.1")
t1 = time.perf_counter()
assert cu.cuInit(0) == 0
t2 = time.perf_counter()
dev = ctypes.c_int(); cu.cuDeviceGet(ctypes.byref(dev), 0)
ctx = ctypes.c_void_p()
assert cu.cuDevicePrimaryCtxRetain(ctypes.byref(ctx), dev) == 0
cu.cuCtxSetCurrent(ctx)
t3 = time.perf_counter()
p = ctypes.c_uint64(); cu.cuMemAlloc_v2(ctypes.byref(p), ctypes.c_size_t(1 << 20))
t4 = time.perf_counter()
print({"dlopen_s": round(t1-t0,4), "cuInit_s": round(t2-t1,4), "ctx_s": round(t3-t2,4), "first_alloc_s": round(t4-t3,4)})

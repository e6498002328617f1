"""ncu target: one persistent grid-stride write (st.global.cs, 128-bit, 4
blocks/SM) and one one-shot write of the same 2 GB buffer — the pair behind
DESIGN §3.0's one-shot finding, for `ncu --set full` side by side.
Usage: ncu --set full -c 2 python scripts/stream_probe_ncu.py"""
import ctypes
import os

import torch

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "_probe",
                               "stream_probe.so"))
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
n = 1 << 28
a = torch.empty(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
lib.sp_write(ctypes.c_void_p(a.data_ptr()), ctypes.c_longlong(n // 2), 4, st, 0, 16)
lib.sp_write_np(ctypes.c_void_p(a.data_ptr()), ctypes.c_longlong(n), 2, st)
torch.cuda.synchronize()

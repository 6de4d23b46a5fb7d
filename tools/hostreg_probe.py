"""Cost of page-locking the caller's pageable buffers in place (cudaHostRegister)
against staging them through pinned slots: register / unregister time and the
H2D rate from a registered numpy array."""
import ctypes as C
import time
import numpy as np
import torch

torch.cuda.init()
rt = C.CDLL("libcudart.so") if False else None
try:
    rt = C.CDLL("libcudart.so.12")
except OSError:
    import glob
    rt = C.CDLL(sorted(glob.glob("/usr/local/cuda/lib64/libcudart.so*"))[0])
for mb in (64, 256, 512):
    a = np.ones(mb * 1024 * 1024 // 4, np.float32)  # touched pages
    d = torch.empty(a.size, dtype=torch.float32, device="cuda")
    for it in range(2):
        t0 = time.perf_counter()
        r = rt.cudaHostRegister(C.c_void_p(a.ctypes.data), C.c_size_t(a.nbytes), C.c_uint(0))
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        d.copy_(torch.from_numpy(a), non_blocking=True)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        rt.cudaHostUnregister(C.c_void_p(a.ctypes.data))
        t4 = time.perf_counter()
        print(f"{mb} MiB rc={r}: register {1e3*(t1-t0):.2f} ms, H2D {1e3*(t3-t2):.2f} ms ({a.nbytes/(t3-t2)/1e9:.1f} GB/s), unregister {1e3*(t4-t3):.2f} ms", flush=True)
    t0 = time.perf_counter()
    d.copy_(torch.from_numpy(a))
    torch.cuda.synchronize()
    print(f"{mb} MiB pageable copy_: {1e3*(time.perf_counter()-t0):.2f} ms", flush=True)

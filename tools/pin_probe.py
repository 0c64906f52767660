"""Is torch's pin_memory() seen as pinned by the CUDA runtime our library links?
cudaPointerGetAttributes + H2D bandwidth through that runtime for a torch-pinned
tensor, a cudaHostAlloc buffer and a cudaHostRegister'd buffer."""
import ctypes, time, sys
import numpy as np
import torch

rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
n = 53 * 10**6
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()


class Attr(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int), ("device", ctypes.c_int), ("devicePointer", ctypes.c_void_p),
                ("hostPointer", ctypes.c_void_p)]


def attr(p):
    a = Attr()
    rc = rt.cudaPointerGetAttributes(ctypes.byref(a), ctypes.c_void_p(p))
    return rc, a.type


def bw(p, chunk=5_250_000, reps=10):
    for r in range(reps + 2):
        if r == 2:
            torch.cuda.synchronize()
            t = time.perf_counter()
        for off in range(0, n, chunk):
            rt.cudaMemcpyAsync(ctypes.c_void_p(d.data_ptr() + off), ctypes.c_void_p(p + off),
                               ctypes.c_size_t(min(chunk, n - off)), ctypes.c_int(1), ctypes.c_void_p(s.cuda_stream))
        torch.cuda.synchronize()
    return n * reps / (time.perf_counter() - t) / 1e9


print("torch", torch.__version__, "cuda", torch.version.cuda)
for k in range(2):
    t = torch.from_numpy(np.ones(n, dtype=np.uint8)).pin_memory()
    print(f"torch pin_memory   : attr {attr(t.data_ptr())}  is_pinned {t.is_pinned()}  {bw(t.data_ptr()):.1f} GB/s")
    p = ctypes.c_void_p()
    rt.cudaHostAlloc(ctypes.byref(p), ctypes.c_size_t(n), 0)
    ctypes.memset(p, 1, n)
    print(f"cudaHostAlloc      : attr {attr(p.value)}  {bw(p.value):.1f} GB/s")
    a = np.ones(n, dtype=np.uint8)
    rt.cudaHostRegister(ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(n), 0)
    print(f"cudaHostRegister   : attr {attr(a.ctypes.data)}  {bw(a.ctypes.data):.1f} GB/s")
    b = np.ones(n, dtype=np.uint8)
    print(f"pageable numpy     : attr {attr(b.ctypes.data)}  {bw(b.ctypes.data):.1f} GB/s")

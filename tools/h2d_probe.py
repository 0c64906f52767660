"""Pinned host<->device copy bandwidth through cudaMemcpyAsync, one stream vs
the same bytes split over 2 / 4 streams (copy engines), for the e2e path's
53 MB of inputs."""
import ctypes, time
import torch

rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
n = 53 * 10**6
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]


def run(kind, ns, reps=10):
    part = n // ns
    for r in range(reps + 2):
        if r == 2:
            torch.cuda.synchronize()
            t = time.perf_counter()
        for k in range(ns):
            dst, src = (d.data_ptr(), h.data_ptr()) if kind == 1 else (h.data_ptr(), d.data_ptr())
            rt.cudaMemcpyAsync(ctypes.c_void_p(dst + k * part), ctypes.c_void_p(src + k * part),
                               ctypes.c_size_t(part), ctypes.c_int(kind), ctypes.c_void_p(streams[k].cuda_stream))
        torch.cuda.synchronize()
    return n * reps / (time.perf_counter() - t) / 1e9


for ns in (1, 2, 4):
    print(f"H2D {ns} stream(s): {run(1, ns):.1f} GB/s   D2H: {run(2, ns):.1f} GB/s")

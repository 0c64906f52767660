"""H2D bandwidth (5.25 MB copies of a 53 MB buffer) from host memory pinned with
cudaHostRegister over (a) 2 MB-aligned, MADV_HUGEPAGE memory and (b) the same with
MADV_NOHUGEPAGE (4 KB pages), plus torch's pin_memory(), several allocations each:
under an IOMMU, 4 KB pages cost translation misses on every DMA."""
import ctypes, mmap, time
import torch

rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
libc = ctypes.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = ctypes.c_void_p
libc.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long]
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
n = 53 * 10**6
HUGE = 2 << 20
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())


def region(huge):
    size = (n + HUGE) // HUGE * HUGE + HUGE
    p = libc.mmap(None, size, 3, 0x22, -1, 0)  # PROT_READ|WRITE, MAP_PRIVATE|ANONYMOUS
    a = (p + HUGE - 1) // HUGE * HUGE
    libc.madvise(ctypes.c_void_p(a), ctypes.c_size_t(size - (a - p)), 14 if huge else 15)  # MADV_(NO)HUGEPAGE
    ctypes.memset(a, 1, n)
    assert rt.cudaHostRegister(ctypes.c_void_p(a), ctypes.c_size_t(n), 0) == 0
    return a


def bw(p, chunk=5_250_000, reps=10):
    for r in range(reps + 2):
        if r == 2:
            torch.cuda.synchronize()
            t = time.perf_counter()
        for off in range(0, n, chunk):
            m = min(chunk, n - off)
            rt.cudaMemcpyAsync(ctypes.c_void_p(d.data_ptr() + off), ctypes.c_void_p(p + off), ctypes.c_size_t(m),
                               ctypes.c_int(1), ctypes.c_void_p(s.cuda_stream))
        torch.cuda.synchronize()
    return n * reps / (time.perf_counter() - t) / 1e9


def smaps_huge(a):
    tot = 0
    with open("/proc/self/smaps") as f:
        cur = None
        for line in f:
            if "-" in line.split()[0] and len(line.split()) > 4:
                lo, hi = (int(x, 16) for x in line.split()[0].split("-"))
                cur = lo <= a < hi
            elif cur and line.startswith("AnonHugePages:"):
                tot += int(line.split()[1])
    return tot


for k in range(3):
    for huge in (True, False):
        a = region(huge)
        print(f"alloc {k} {'MADV_HUGEPAGE  ' if huge else 'MADV_NOHUGEPAGE'}: {bw(a):.1f} GB/s  (AnonHugePages {smaps_huge(a)} kB)")
    t = torch.empty(n, dtype=torch.uint8).pin_memory()
    print(f"alloc {k} torch pin_memory : {bw(t.data_ptr()):.1f} GB/s")

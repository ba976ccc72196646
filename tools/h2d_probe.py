"""H2D bandwidth of an 80 MB block from pinned host memory: default pinned,
write-combined pinned, and split over two streams (the e2e leg's copy)."""
import ctypes
import torch

rt = ctypes.CDLL("libcudart.so.12")
n = 80_000_000
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def bench(ptr, label, split=False):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(8):
        torch.cuda.synchronize()
        a.record()
        if split:
            h = n // 2
            s1.wait_stream(torch.cuda.current_stream())
            s2.wait_stream(torch.cuda.current_stream())
            rt.cudaMemcpyAsync(ctypes.c_void_p(dev.data_ptr()), ctypes.c_void_p(ptr), ctypes.c_size_t(h), 1, ctypes.c_void_p(s1.cuda_stream))
            rt.cudaMemcpyAsync(ctypes.c_void_p(dev.data_ptr() + h), ctypes.c_void_p(ptr + h), ctypes.c_size_t(n - h), 1, ctypes.c_void_p(s2.cuda_stream))
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
        else:
            rt.cudaMemcpyAsync(ctypes.c_void_p(dev.data_ptr()), ctypes.c_void_p(ptr), ctypes.c_size_t(n), 1, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"{label}: {best:.3f} ms  {n / best / 1e6:.1f} GB/s", flush=True)


for flags, label in ((0, "pinned (default)"), (4, "pinned write-combined"), (1, "pinned portable")):
    p = ctypes.c_void_p()
    rc = rt.cudaHostAlloc(ctypes.byref(p), ctypes.c_size_t(n), ctypes.c_uint(flags))
    assert rc == 0, rc
    ctypes.memset(p, 1, n)
    bench(p.value, label)
    bench(p.value, label + ", two streams", split=True)
    rt.cudaFreeHost(p)
t = torch.empty(n, dtype=torch.uint8).pin_memory()
bench(t.data_ptr(), "torch pin_memory")

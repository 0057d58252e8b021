"""Diagnostic: PCIe bandwidth of 1-D vs pitched (cudaMemcpy2DAsync) copies between a device chunk
and a strided pinned host buffer — the copies of the pinned pipeline's chunks (C3: 2048 output
lanes x 1024 hops x 128 samples per chunk)."""
import torch
from cuda.bindings import runtime as rt

n_rows, row = 2048, 1024 * 128
d = torch.empty((n_rows, row), device="cuda")
h = torch.empty((n_rows, row * 4), pin_memory=True)  # the chunk's columns of a 4-chunk-wide host buffer
h1 = torch.empty((n_rows * row,), pin_memory=True)
s = torch.cuda.Stream()


def timed(fn, reps=5):
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


nb = d.numel() * 4
D2H, H2D = rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, rt.cudaMemcpyKind.cudaMemcpyHostToDevice
for name, fn in [
    ("D2H 1D", lambda: rt.cudaMemcpyAsync(h1.data_ptr(), d.data_ptr(), nb, D2H, s.cuda_stream)),
    ("D2H 2D", lambda: rt.cudaMemcpy2DAsync(h.data_ptr() + row * 4, row * 16, d.data_ptr(), row * 4, row * 4, n_rows,
                                            D2H, s.cuda_stream)),
    ("H2D 1D", lambda: rt.cudaMemcpyAsync(d.data_ptr(), h1.data_ptr(), nb, H2D, s.cuda_stream)),
    ("H2D 2D", lambda: rt.cudaMemcpy2DAsync(d.data_ptr(), row * 4, h.data_ptr() + row * 4, row * 16, row * 4, n_rows,
                                            H2D, s.cuda_stream)),
]:
    print(f"{name} {nb / timed(fn) / 1e6:.1f} GB/s")

# Bandwidth ceilings on the headline buffers (131072 x 151936 bf16): torch copy / read / write.
import torch
T, V = 131072, 151936
a = torch.empty(T, V, dtype=torch.bfloat16, device="cuda")
b = torch.empty_like(a)
a.normal_()
n = a.numel() * 2

def timeit(f, reps=5):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

ms = timeit(lambda: b.copy_(a))
print(f"copy   {2 * n / ms / 1e6:.0f} GB/s  ({ms:.2f} ms)")
ms = timeit(lambda: b.fill_(1.0))
print(f"write  {n / ms / 1e6:.0f} GB/s")
ms = timeit(lambda: a.view(torch.int16).max())
print(f"read   {n / ms / 1e6:.0f} GB/s (int16 max reduction)")
# strided-half copy: every row's first half (like a 2-CTA slice pattern)
h = V // 2
ms = timeit(lambda: b[:, :h].copy_(a[:, :h]))
print(f"half-row copy {2 * T * h * 2 / ms / 1e6:.0f} GB/s")

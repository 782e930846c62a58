# Read-only and write-only stream ceilings on the R3 operand size (3.2 GB fp32):
# torch's reduction (read) and fill (write) kernels, for the R3 roofline notes.
import torch
dev = torch.device("cuda", 0)
z = torch.randn(48, 32 * 4096, 128, device=dev)
out = torch.empty_like(z)
nb = z.numel() * 4
for name, fn, by in [("read (sum)", lambda: z.sum(), nb), ("write (fill_)", lambda: out.fill_(1.0), nb),
                     ("copy (copy_)", lambda: out.copy_(z), 2 * nb)]:
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name}: {ms:.3f} ms {by / ms / 1e6:.0f} GB/s", flush=True)

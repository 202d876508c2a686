"""HBM write-bandwidth probes (context for the full-output roofline): plain
fills, and fills of 128-byte row segments at a 4 KB row stride (c4's [N][1024]
fp32 output written one 32-query column block at a time)."""
import torch

y = torch.empty(100_000 * 1024, dtype=torch.float32, device="cuda")  # c4 output, 409.6 MB
v = y.view(100_000, 32, 32)  # [row][128-byte segment][fp32]


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


ms = timed(lambda: y.fill_(1.0))
print(f"contiguous fill: {y.numel() * 4 / ms / 1e6:.0f} GB/s")
ms = timed(lambda: [v[:, c, :].fill_(2.0) for c in range(32)])
print(f"128 B segments at 4 KB stride (32 column passes): {y.numel() * 4 / ms / 1e6:.0f} GB/s")
ms = timed(lambda: [v[:, c:c + 8, :].fill_(3.0) for c in range(0, 32, 8)])
print(f"1 KB segments at 4 KB stride (4 passes): {y.numel() * 4 / ms / 1e6:.0f} GB/s")

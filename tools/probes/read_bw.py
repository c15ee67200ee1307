"""Achievable HBM read bandwidth on this box for a 1 GB fp32 array (torch reductions), as the
yardstick for the K3 count pass (dev tool)."""
import torch

x = torch.rand(256 * (1 << 20), device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, fn in (("sum", lambda: x.sum()), ("amin", lambda: x.amin()), ("count_le", lambda: (x <= 0.01).sum())):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[5]
    print(f"{name}: {ms:.4f} ms  {x.numel() * 4 / ms / 1e9:.2f} TB/s (read only)")

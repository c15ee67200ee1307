"""Dev check: device-call vs host-buffer-call time of one C5 detect, and the D2H time alone."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import synth  # noqa: E402
from paper_2601_18548_b200 import FP16, Context  # noqa: E402

cfg = synth.get_config("C5")
pts, _ = synth.make_scene_points(cfg)
q = torch.from_numpy(synth.make_waypoints(cfg))
tau = synth.load_tau(cfg.name)
cap = 1 << 23
ctx = Context(0, precision=FP16, scene_capacity=cfg.M + 4096, max_waypoints=cfg.B * cfg.N, max_active=cap)
ctx.load_weights(synth.weights_path(cfg.H))
ctx.update_scene(pts)
outs = ctx.alloc_detect_outputs(cfg.B * cfg.N, cap)
qd = q.cuda()
ho = ctx.alloc_host_outputs(cfg.B * cfg.N, cap, pinned=True)
for _ in range(2):
    ctx.detect_active_set(qd, 0.1, tau, outputs=outs)
    ctx.detect_active_set_host(q, 0.1, tau, ho)
torch.cuda.synchronize()
for name, fn in (("device call", lambda: ctx.detect_active_set(qd, 0.1, tau, outputs=outs)),
                 ("host-buffer call", lambda: ctx.detect_active_set_host(q, 0.1, tau, ho))):
    t0 = time.perf_counter()
    for _ in range(5):
        o = fn()
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms per call, n = {o['n']}")
n = int(ho["n"])
src = outs["records"][:n]
t0 = time.perf_counter()
for _ in range(5):
    ho["records"][:n].copy_(src, non_blocking=True)
    torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 5
print(f"D2H of {n * 48 / 1e6:.1f} MB pinned: {dt * 1e3:.2f} ms ({n * 48 / dt / 1e9:.1f} GB/s)")

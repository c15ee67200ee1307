"""Diagnostics: clock64 pipeline trace of the tensor-core kernel (CTA 0) on C5.

    python tools/trace_tc.py [--config C5] [--precision fp16] > gpurun_out/trace.txt
Roles: MMA issuer stamps (epi wait done / commit) per phase and slot; slot-0/1 epilogue
stamps per phase: [wait start, wait end (MMA done), compute done, arrive done].
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import synth  # noqa: E402
from paper_2601_18548_b200 import BF16, FP16, Context  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--precision", default="fp16")
a = ap.parse_args()
cfg = synth.get_config(a.config)
pts, _ = synth.make_scene_points(cfg)
q = torch.from_numpy(synth.make_waypoints(cfg)).cuda()
ctx = Context(0, precision=FP16 if a.precision == "fp16" else BF16, scene_capacity=cfg.M + 4096,
              max_waypoints=cfg.B * cfg.N, max_active=1 << 23)
ctx.load_weights(synth.weights_path(cfg.H))
ctx.update_scene(pts)
tau = synth.load_tau(cfg.name)
for _ in range(2):
    ctx.detect_active_set(q, synth.inputs.DELTA, tau)
buf = torch.zeros(3 * 4 * 13 * 4, dtype=torch.int64, device="cuda")
ctx.debug_trace(buf)
ctx.detect_active_set(q, synth.inputs.DELTA, tau)
torch.cuda.synchronize()
ctx.debug_trace(None)
t = buf.cpu().numpy().reshape(3, 4, 13, 4).astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, np.nan)
np.set_printoptions(linewidth=200, suppress=True)
print("MMA issuer [tile][phase]: s0 wait-done, s0 commit, s1 wait-done, s1 commit (cycles from first stamp)")
for it in range(4):
    for p in range(12):
        print(f"  tile{it} p{p:2d}: " + " ".join(f"{v:10.0f}" for v in t[0, it, p]))
for r in (1, 2):
    print(f"slot {r - 1} epilogue (warp h0 q0 lane0) [tile][k]: wait-start, wait-end, compute-done, arrived")
    for it in range(4):
        for k in range(13):
            v = t[r, it, k]
            print(f"  tile{it} k{k:2d}: " + " ".join(f"{x:10.0f}" for x in v) +
                  f"   | wait {v[1] - v[0]:7.0f} compute {v[2] - v[1]:7.0f} st+arrive {v[3] - v[2]:7.0f}")
# per-phase summary over tiles 1..3 (steady state)
print("steady-state means (tiles 1..3), slot 0 per k: wait (prev handoff -> mma done), tmem load, "
      "compute (after load), handoff (st wait + barrier + issue)")
for k in range(1, 13):
    v = t[1, 1:, k]
    prev = t[1, 1:, k - 1, 3]
    print(f"  k{k:2d}: wait {np.nanmean(v[:, 1] - prev):7.0f}  load {np.nanmean(v[:, 0] - v[:, 1]):7.0f}  "
          f"compute {np.nanmean(v[:, 2] - v[:, 0]):7.0f}  handoff {np.nanmean(v[:, 3] - v[:, 2]):7.0f}")
tile_cycles = np.nanmean(np.diff(t[1, :, 0, 0]))
print(f"slot-0 tile period: {tile_cycles:.0f} cycles")

"""Diagnostics: clock64 pipeline trace of the tensor-core kernel K2b (CTA 0) on C5.

    python tools/trace_tc.py [--config C5] [--precision fp16] > gpurun_out/trace.txt
Roles: MMA issuer stamps (epi wait done / commit) per phase and slot; per epilogue warp
(lane 0) stamps per phase k (k = MMA phase + 1): [tmem load done, mma done, compute done,
arrived].
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import synth  # noqa: E402
from paper_2601_18548_b200 import BF16, FP16, Context  # noqa: E402

ROLES, TILES, PH = 18, 4, 13
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
buf = torch.zeros(ROLES * TILES * PH * 4, dtype=torch.int64, device="cuda")
ctx.debug_trace(buf)
ctx.detect_active_set(q, synth.inputs.DELTA, tau)
torch.cuda.synchronize()
ctx.debug_trace(None)
raw = buf.cpu().numpy()
t = raw.reshape(ROLES, TILES, PH, 4).astype(np.float64)
t0 = t[t > 0].min()
wo = 6 * TILES * PH * 4
tw = raw[wo:wo + 24 * TILES * 12].reshape(24, TILES, 12).astype(np.float64)
tw = np.where(tw > 0, tw - t0, np.nan)
t = np.where(t > 0, t - t0, np.nan)
np.set_printoptions(linewidth=200, suppress=True)
# K2b (3 slots): role s = MMA warp of slot s [A ready, turn, commit returned];
# role 3 + s = epilogue warp 0 of slot s [D ready (woke), epilogue done]
print("per slot, per (tile, phase): MMA warp [A ready, turn, committed] | epilogue warp 0 [D ready, +computed, +arrived, +done]")
for it in range(TILES):
    for p in range(12):
        def ep(s_):
            v = t[3 + s_, it, p]
            return f"{v[0]:8.0f} +{v[2] - v[0]:5.0f} +{v[3] - v[0]:5.0f} +{v[1] - v[0]:5.0f}"
        print(f"  tile{it} p{p:2d}: " + "  ||".join(
            " ".join(f"{v:8.0f}" for v in t[s_, it, p, :3]) + " | " + ep(s_) for s_ in range(3)))
print("per-warp hand-off (cycles after the slot's first warp; warp = 8 s + 4 h + q) -- last warp and spread")
for it in range(1, TILES):
    for p in range(12):
        line = f"  tile{it} p{p:2d}: "
        for s_ in range(3):
            v = tw[8 * s_:8 * s_ + 8, it, p]
            if np.isfinite(v).all():
                line += f" s{s_}: first {np.nanmin(v):8.0f} +" + " ".join(f"{x - np.nanmin(v):4.0f}" for x in v) + " |"
        print(line)

"""Diagnostics: clock64 pipeline trace of the tensor-core kernel (CTA 0) on C5.

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
t = buf.cpu().numpy().reshape(ROLES, TILES, PH, 4).astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, np.nan)
np.set_printoptions(linewidth=200, suppress=True)
print("MMA issuer [tile][phase]: s0 wait-done, s0 commit, s1 wait-done, s1 commit (cycles from first stamp)")
for it in range(TILES):
    for p in range(12):
        print(f"  tile{it} p{p:2d}: " + " ".join(f"{v:10.0f}" for v in t[0, it, p]))
for slot in (0, 1):
    w0 = 1 + 8 * slot
    print(f"slot {slot}: per phase k, warp 0 of the slot [load-done, mma-done, compute-done, arrived] and "
          "the arrival spread over its 8 warps (last warp, cycles after the first)")
    for it in range(TILES):
        for k in range(PH):
            v = t[w0, it, k]
            arr = t[w0:w0 + 8, it, k, 3]
            last = int(np.nanargmax(arr)) if np.isfinite(arr).any() else -1
            spread = np.nanmax(arr) - np.nanmin(arr) if np.isfinite(arr).any() else np.nan
            comp = t[w0:w0 + 8, it, k, 2] - t[w0:w0 + 8, it, k, 1]
            print(f"  tile{it} k{k:2d}: " + " ".join(f"{x:9.0f}" for x in v) +
                  f" | compute {v[2] - v[1]:6.0f} (max over warps {np.nanmax(comp) if np.isfinite(comp).any() else np.nan:6.0f})"
                  f" last warp {8 * slot + last:2d} +{spread:5.0f}")
# MMA-side phase timing: per slot, time from MMA issue (commit) to the slot's next epi arrival
print("steady-state (tiles 1..2, slot 0): per k: mma wait (commit -> mma done seen by warp 0), "
      "compute (warp 0), slowest-warp arrival after mma done")
for k in range(1, PH):
    md = t[1, 1:3, k, 1]
    arr = np.nanmax(t[1:9, 1:3, k, 3], axis=0)
    comp = t[1, 1:3, k, 2] - t[1, 1:3, k, 1]
    print(f"  k{k:2d}: compute(w0) {np.nanmean(comp):7.0f}  last arrival - mma done {np.nanmean(arr - md):7.0f}")
tile_cycles = np.nanmean(np.diff(t[0, :, 0, 0]))
print(f"slot-0 tile period: {tile_cycles:.0f} cycles")
# critical path per phase (tile 1): MMA issue of slot s -> epilogue sees mma done -> last
# warp arrives -> MMA thread sees it (next issue of slot s)
print("tile1 critical path: slot, p, issue start, issue end, epi mma-done, last arrival, next issue start")
for s in (0, 1):
    for p in range(11):
        v = t[0, 1, p]
        md = t[1 + 8 * s, 1, p + 1, 1]
        last = np.nanmax(t[1 + 8 * s:9 + 8 * s, 1, p + 1, 3])
        nxt = t[0, 1, p + 1, 2 * s]
        w = t[17, 1, p + 1]
        print(f"  s{s} p{p:2d}: issue {v[2 * s]:7.0f} .. {v[2 * s + 1]:7.0f} | mma done {md - v[2 * s + 1]:+6.0f} after issue end"
              f" | epi {last - md:5.0f} | MMA thread wakes {nxt - last:+6.0f} after last arrival"
              f" (wait {w[2 * s] - last:+6.0f} .. {w[2 * s + 1] - last:+6.0f}, fence {nxt - w[2 * s + 1]:4.0f})")
# per-warp view of the two long phases (k = 6: output layer, k = 12: tile boundary)
print("per warp (slot 0, tiles 1..2 mean): k, warp: mma-done -> load-done, load-done -> compute-done, mma-done -> arrived")
for k in (6, 12):
    for w in range(8):
        v = t[1 + w, 1:3, k]
        print(f"  k{k:2d} w{w}: {np.nanmean(v[:, 0] - v[:, 1]):7.0f} {np.nanmean(v[:, 2] - v[:, 0]):7.0f} "
              f"{np.nanmean(v[:, 3] - v[:, 1]):7.0f}")
print("phase 11 detail (slot 0, tiles 1..2 mean), per warp: stage_a1 end -> tile_pair done -> barrier -> end")
for w in range(4):
    v = t[1 + w, 1:3]
    a0 = v[:, 12, 2]
    print(f"  w{w}: tile_pair {np.nanmean(v[:, 0, 1] - a0):6.0f}  barrier {np.nanmean(v[:, 0, 2] - a0):6.0f}  "
          f"end {np.nanmean(v[:, 12, 3] - a0):6.0f}")

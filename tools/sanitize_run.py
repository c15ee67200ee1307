"""Small runs of every device path, for compute-sanitizer.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py [--paths k2b,k2c,...]

Each path runs one small detect (and the K2b dense query / partitioned detect) on a C2-shaped
scene cut to a few tiles per waypoint, so that the instrumented kernels finish in seconds.
The results are checked only for sanity here (the parity tests own correctness); the point
is the sanitizer's report on the hand-rolled mbarrier / named-barrier / TMEM protocols.
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import synth  # noqa: E402
from paper_2601_18548_b200 import BF16, FP16, FP16X3, FP32, Context  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--paths", default="k2b,k2b_bf16,k2b_se2,k2b_part,k2c,k2s,k2w,simt,k3")
ap.add_argument("--points", type=int, default=1500)
ap.add_argument("--waypoints", type=int, default=6)
a = ap.parse_args()

cfg = synth.get_config("C2")
pts, _ = synth.make_scene_points(cfg)
pts = pts[:a.points]
q = torch.from_numpy(synth.make_waypoints(cfg)[:, :a.waypoints]).cuda()
tau = synth.load_tau("C2")
D = synth.inputs.DELTA


def ctx_for(prec, H=128, act=1, **kw):
    c = Context(0, precision=prec, scene_capacity=len(pts) + 256, max_waypoints=64, max_active=1 << 16, **kw)
    c.load_weights(synth.weights_path(H, act=act))
    c.update_scene(pts)
    return c


for name in a.paths.split(","):
    if name in ("k2b", "k2b_bf16", "k2b_se2"):
        kw = {"frame": 1} if name == "k2b_se2" else {}
        c = ctx_for(BF16 if name == "k2b_bf16" else FP16, **kw)
        out = c.detect_active_set(q, D, tau)
        v, g = c.query_values_grads(q)
        torch.cuda.synchronize()
        print(name, "detect", int(out["n"]), "dense finite", bool(torch.isfinite(v).any()))
    elif name == "k2b_part":
        c = ctx_for(FP16, max_candidates=1 << 16)
        out = c.detect_active_set_partitioned(q, 1.8, D, tau)
        torch.cuda.synchronize()
        print(name, int(out["n"]))
    elif name == "k2c":
        c = ctx_for(FP16X3)
        out = c.detect_active_set(q, D, tau)
        torch.cuda.synchronize()
        print(name, int(out["n"]))
    elif name == "k2s":
        c = ctx_for(FP16, act=2)
        out = c.detect_active_set(q, D, synth.load_tau("C2", act=2))
        torch.cuda.synchronize()
        print(name, int(out["n"]))
    elif name == "k2w":
        c = ctx_for(FP16, H=256)
        out = c.detect_active_set(q, D, synth.load_tau("C2", hidden=256))
        torch.cuda.synchronize()
        print(name, int(out["n"]))
    elif name == "simt":
        c = ctx_for(FP32)
        out = c.detect_active_set(q, D, tau)
        torch.cuda.synchronize()
        print(name, int(out["n"]))
    elif name == "k3":
        c = ctx_for(FP16)
        v, g = c.query_values_grads(q)
        out = c.compact_dense(v, g, D, tau)
        torch.cuda.synchronize()
        print(name, int(out["n"]))
print("sanitize_run done", flush=True)

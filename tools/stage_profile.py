"""Dev tool: run one hot-path stage repeatedly on C5 for an ncu launch list.

    python tools/stage_profile.py partitioned|compact|pairgen [--reps 3]
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import synth  # noqa: E402
from paper_2601_18548_b200 import FP16, Context  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("stage")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--config", default="C5")
ap.add_argument("--time", action="store_true", help="CUDA-event timing instead of a profiler target")
a = ap.parse_args()
cfg = synth.get_config(a.config)
pts, _ = synth.make_scene_points(cfg)
q = torch.from_numpy(synth.make_waypoints(cfg)).cuda()
tau = synth.load_tau(cfg.name)
ctx = Context(0, precision=FP16, scene_capacity=cfg.M + 4096, max_waypoints=cfg.B * cfg.N, max_active=1 << 23,
              max_candidates=cfg.pairs)
ctx.load_weights(synth.weights_path(cfg.H))
ctx.update_scene(pts)
outs = ctx.alloc_detect_outputs(cfg.B * cfg.N, 1 << 23)
if a.stage == "compact":
    v, g = ctx.query_values_grads(q)
def one():
    if a.stage == "partitioned":
        ctx.detect_active_set_partitioned(q, 1.8, 0.1, tau, outputs=outs)
    elif a.stage == "compact":
        ctx.compact_dense(v, g, 0.1, tau, outputs=outs)
    elif a.stage == "pairgen":
        ctx.pairgen_transform(q)


if a.time:  # CUDA-event time per call (after 3 warm-ups), L2 flushed before each call
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        one()
    ts = []
    for _ in range(a.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        one()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(a.stage, "ms per call: median %.4f min %.4f" % (sorted(ts)[len(ts) // 2], min(ts)))
    sys.exit(0)
for _ in range(a.reps):
    if a.stage == "partitioned":
        ctx.detect_active_set_partitioned(q, 1.8, 0.1, tau, outputs=outs)
    elif a.stage == "compact":
        ctx.compact_dense(v, g, 0.1, tau, outputs=outs)
    elif a.stage == "pairgen":
        ctx.pairgen_transform(q)
torch.cuda.synchronize()
print("done", a.stage)

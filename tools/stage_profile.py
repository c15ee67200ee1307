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
for _ in range(a.reps):
    if a.stage == "partitioned":
        ctx.detect_active_set_partitioned(q, 1.8, 0.1, tau, outputs=outs)
    elif a.stage == "compact":
        ctx.compact_dense(v, g, 0.1, tau, outputs=outs)
    elif a.stage == "pairgen":
        ctx.pairgen_transform(q)
torch.cuda.synchronize()
print("done", a.stage)

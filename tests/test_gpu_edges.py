"""Degenerate inputs on every compiled tensor-core kernel and the fp32 path (R14,
R15): an empty scene, a scene whose points were all removed, and a single live point (one
tile of 127 padding rows).  Checked against the float64 oracle (or its definition of the
empty case: +INF minimum, argmin -1, no records, zero offsets)."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import DELTA

pytestmark = pytest.mark.gpu
NT = max(1, min(os.cpu_count() or 1, 16))

# (precision name, H, activation, frame, value tolerance vs the exact oracle)
PATHS = [("fp32", 128, 1, 0, 1e-4), ("fp16", 128, 1, 0, 2e-2), ("bf16", 128, 1, 0, 3e-2), ("fp16x3", 128, 1, 0, 1e-4),
         ("fp16", 128, 1, 1, 2e-2), ("fp16", 128, 2, 0, 2e-2), ("fp16", 256, 1, 0, 2e-2), ("fp32", 256, 2, 0, 1e-4),
         ("bf16x3", 128, 1, 0, 1e-3)]


def _ctx(prec, H, act, frame):
    from paper_2601_18548_b200 import BF16, BF16X3, FP16, FP16X3, FP32, Context
    p = {"fp32": FP32, "fp16": FP16, "bf16": BF16, "fp16x3": FP16X3, "bf16x3": BF16X3}[prec]
    ctx = Context(0, precision=p, scene_capacity=512, max_waypoints=16, max_active=1 << 12, max_candidates=1 << 12,
                  frame=frame)
    ctx.load_weights(synth.weights_path(H, act=act))
    return ctx


@pytest.mark.parametrize("prec,H,act,frame,tol", PATHS)
def test_empty_removed_and_single_point(prec, H, act, frame, tol):
    cfg = synth.get_config("C2")
    pts, _ = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg)[:, :5]
    qt = torch.from_numpy(q)
    ctx = _ctx(prec, H, act, frame)
    # empty scene: no records, +INF minimum, argmin -1, zero offsets (R14)
    for out in (ctx.detect_active_set(qt, DELTA, 100.0), ctx.detect_active_set_partitioned(qt, 2.0, DELTA, 100.0)):
        torch.cuda.synchronize()
        assert out["n"] == 0
        assert torch.all(torch.isinf(out["wp_min"])) and torch.all(out["wp_argmin"] == -1)
        assert torch.all(out["wp_offsets"] == 0)
    # every point removed again (R15): the same
    ids = ctx.update_scene(pts[:200])
    ctx.update_scene(remove_ids=ids)
    out = ctx.detect_active_set(qt, DELTA, 100.0)
    torch.cuda.synchronize()
    assert out["n"] == 0 and torch.all(out["wp_argmin"] == -1)
    # a single live point: one tile with 127 padding rows; every waypoint's minimum is that
    # point, and with a huge tau it is active at every waypoint
    (pid,) = ctx.update_scene(pts[7:8])
    out = ctx.detect_active_set(qt, DELTA, 100.0)
    v, _ = ctx.query_values_grads(qt)
    torch.cuda.synchronize()
    m = oracle.MLP(synth.weights_path(H, act=act))
    flags = oracle.FRAME_SE2 if frame else 0
    ref = m.eval(pts[7:8], q.reshape(-1, 9), flags=flags, want_grad=False, nthreads=NT)["f"][:, 0]
    assert out["n"] == q.shape[1]
    assert torch.all(out["wp_argmin"] == int(pid))
    got = out["wp_min"].cpu().numpy().astype(np.float64)
    assert np.all(np.abs(got - ref) <= tol * np.maximum(1.0, np.abs(ref))), np.abs(got - ref).max()
    vv = v.cpu().numpy()
    assert np.all(np.isinf(np.delete(vv, int(pid), axis=1)))  # padding / dead slots stay +INF
    assert np.array_equal(vv[:, int(pid)], out["wp_min"].cpu().numpy())

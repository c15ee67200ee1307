"""NEXT-4 (R24): the SE(2) base-frame variant on the GPU against the float64
oracle's FRAME_SE2 mode.  Points are rotated into the base frame,
p'_xy = R(-theta)(p_xy - b), the theta channel is fed zero, and the gradient follows by the
chain rule: d f / d b = -R(theta) g0_xy, d f / d theta = g0_x p'_y - g0_y p'_x.  The oracle
mode itself is pinned in tests/test_oracle_pins.py (rigid-motion invariance, central
finite differences, theta = 0 reduces to the translation frame)."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import (BAND_FP32, BF16_VAL_ATOL, DELTA, KINK_FP32, check_fp32_dense, compare_active_sets, fp32_close,
                      oracle_detect, oracle_mlp, records_np)
from test_gpu_tensor import stats_and_gates

pytestmark = pytest.mark.gpu
NT = max(1, min(os.cpu_count() or 1, 64))
SE2 = oracle.FRAME_SE2


def _ctx(cfg, precision, **kw):
    from paper_2601_18548_b200 import FRAME_SE2, Context
    ctx = Context(0, precision=precision, scene_capacity=cfg.M + 4096, max_waypoints=cfg.B * cfg.N,
                  max_active=min(cfg.pairs, 1 << 22), frame=FRAME_SE2, **kw)
    ctx.load_weights(synth.weights_path(cfg.H))
    return ctx


@pytest.fixture(scope="module")
def c2se2():
    cfg = synth.get_config("C2")
    pts, _ = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg)[:, :12]
    m = oracle_mlp(cfg)
    Q = q.reshape(-1, 9)
    exact = m.eval(pts, Q, flags=SE2, want_kappa=True, want_hash=True, nthreads=NT)
    emu = m.eval(pts, Q, flags=SE2 | oracle.EMU_FP16, want_kappa=True, want_hash=True, nthreads=NT)
    return cfg, pts, q, m, exact, emu


def test_se2_theta_nonzero(c2se2):
    """The workload exercises the rotation (|theta| spans the paper's range)."""
    q = c2se2[2].reshape(-1, 9)
    assert np.abs(q[:, 2]).max() > 0.5


def test_se2_pairgen_transform(c2se2):
    """K1 standalone in SE(2): fp32 rotation of the f64-exact transform (sincosf ~1 ulp)."""
    cfg, pts, q, *_ = c2se2
    ctx = _ctx(cfg, 0)
    ctx.update_scene(pts)
    out = ctx.pairgen_transform(torch.from_numpy(q)).cpu().numpy()
    qq = q.reshape(-1, 9).astype(np.float64)
    M = len(pts)
    dx = pts[None, :, 0].astype(np.float64) - qq[:, None, 0]
    dy = pts[None, :, 1].astype(np.float64) - qq[:, None, 1]
    c, s = np.cos(qq[:, 2])[:, None], np.sin(qq[:, 2])[:, None]
    ex, ey = c * dx + s * dy, -s * dx + c * dy
    scale = np.abs(dx) + np.abs(dy)
    assert np.all(np.abs(out[:, :M, 0] - ex) <= 1e-6 * scale + 1e-7)
    assert np.all(np.abs(out[:, :M, 1] - ey) <= 1e-6 * scale + 1e-7)
    assert np.array_equal(out[:, :M, 2], np.broadcast_to(pts[:, 2], (qq.shape[0], M)))
    assert np.all(out[:, :M, 3] == 1.0) and np.all(out[:, M:, 3] == 0.0)


def test_se2_dense_fp32(c2se2):
    cfg, pts, q, m, exact, _ = c2se2
    ctx = _ctx(cfg, 0)
    ctx.update_scene(pts)
    v, g = ctx.query_values_grads(torch.from_numpy(q))
    torch.cuda.synchronize()
    M = len(pts)
    v, g = v.cpu().numpy(), g.cpu().numpy()
    # theta gradient = g0_x p'_y - g0_y p'_x cancels when the two terms are close: compare it
    # relative to the size of its terms (fp32 error of each product), the other 8 as usual
    gq = g[:, :M].copy()
    og = exact["g"].copy()
    check_fp32_dense(v[:, :M], np.delete(gq, 2, axis=-1), exact["f"], np.delete(og, 2, axis=-1), exact["kappa"],
                     what="C2 SE(2) fp32")
    Q = q.reshape(-1, 9)
    r = np.hypot(pts[None, :, 0] - Q[:, None, 0], pts[None, :, 1] - Q[:, None, 1])
    gxy = np.hypot(og[..., 0], og[..., 1])
    dth = np.abs(gq[..., 2] - og[..., 2])
    bad = dth > 1e-5 + 1e-4 * (np.abs(og[..., 2]) + r * gxy)
    assert not (bad & (exact["kappa"] > KINK_FP32)).any(), dth.max()
    assert bad.sum() <= 1e-3 * bad.size + 1
    assert np.all(np.isinf(v[:, M:])) and np.all(g[:, M:] == 0)


def test_se2_dense_fp16(c2se2):
    """The gates of tests/test_gpu_tensor.py (R17, R28) in the SE(2) frame."""
    cfg, pts, q, m, exact, emu = c2se2
    ctx = _ctx(cfg, 2)
    ctx.update_scene(pts)
    v, g = ctx.query_values_grads(torch.from_numpy(q))
    torch.cuda.synchronize()
    M = len(pts)
    stats_and_gates(v.cpu().numpy()[:, :M], g.cpu().numpy()[:, :M], exact, emu, "fp16", "C2 SE(2) dense")
    assert np.all(np.isinf(v.cpu().numpy()[:, M:])) and np.all(g.cpu().numpy()[:, M:] == 0)


@pytest.mark.parametrize("prec", [0, 2])
def test_se2_detect(c2se2, prec):
    cfg, pts, q, m, exact, _ = c2se2
    tau = synth.load_tau(cfg.name)
    ctx = _ctx(cfg, prec)
    ids = ctx.update_scene(pts)
    out = ctx.detect_active_set(torch.from_numpy(q), DELTA, tau)
    torch.cuda.synchronize()
    gpu = records_np(out)
    orc = oracle_detect(m, pts, ids, q.reshape(-1, 9), tau, flags=SE2, nthreads=NT)
    if prec == 0:
        nd, nc = compare_active_sets(gpu, orc, exact["f"], ids, BAND_FP32, what="SE(2) fp32")
        assert np.all(fp32_close(out["wp_min"].cpu().numpy(), orc["wp_min"]))
    else:
        nd, nc = compare_active_sets(gpu, orc, exact["f"], ids, 1e-3 + BF16_VAL_ATOL, val_atol=BF16_VAL_ATOL,
                                     what="SE(2) fp16")
        assert np.all(np.abs(out["wp_min"].cpu().numpy() - orc["wp_min"]) <= BF16_VAL_ATOL)
    assert nc > 0
    # the fused detect equals the dense query + compaction of the same context
    v, g = ctx.query_values_grads(torch.from_numpy(q))
    a = records_np(ctx.compact_dense(v, g, DELTA, tau))
    for k in ("wp", "pt", "value", "grad"):
        assert np.array_equal(a[k], gpu[k]), k


def test_se2_differs_from_translation(c2se2):
    """Guard: the SE(2) context really rotates (its values differ from the translation
    frame's wherever theta != 0)."""
    from paper_2601_18548_b200 import Context
    cfg, pts, q, *_ = c2se2
    a = _ctx(cfg, 2)
    b = Context(0, precision=2, scene_capacity=cfg.M + 4096, max_waypoints=cfg.B * cfg.N, max_active=1 << 20)
    b.load_weights(synth.weights_path(cfg.H))
    a.update_scene(pts[:1000])
    b.update_scene(pts[:1000])
    va, _ = a.query_values_grads(torch.from_numpy(q))
    vb, _ = b.query_values_grads(torch.from_numpy(q))
    d = (va - vb).abs()[:, :1000]
    assert torch.isfinite(d).all() and d.max().item() > 1e-2

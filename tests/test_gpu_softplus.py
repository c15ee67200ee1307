"""GPU parity of the softplus activation variant (NEXT-4, R26; MLPW activation 2)
against the float64 oracle, through the C ABI.

Softplus is smooth, so unlike the ReLU network no pair is exempt from the gradient check:
the fp32 path must meet the north-star fp32 tolerance (1e-4 relative / 1e-5 absolute) on
every value and every gradient component.  Sizes: C1 in full (H = 32, 2 tiles per
waypoint) and 8 waypoints of C2 (H = 128, 79 tiles per waypoint, ragged last tile).
"""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import BAND_FP32, DELTA, compare_active_sets, fp32_close, oracle_detect, records_np

pytestmark = pytest.mark.gpu
NT = max(1, min(os.cpu_count() or 1, 64))


def _ctx(cfg, precision=0, **kw):
    from paper_2601_18548_b200 import Context
    ctx = Context(0, precision=precision, scene_capacity=cfg.M + 4096, max_waypoints=cfg.B * cfg.N,
                  max_active=min(cfg.pairs, 1 << 22), **kw)
    ctx.load_weights(synth.weights_path(cfg.H, act=2))
    return ctx


def _case(name, n_wp):
    cfg = synth.get_config(name)
    pts, _ = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg)[:, :n_wp]
    m = oracle.MLP(synth.weights_path(cfg.H, act=2))
    assert m.act == 2
    full = m.eval(pts, q.reshape(-1, 9), nthreads=NT)
    return cfg, pts, q, m, full


@pytest.fixture(scope="module")
def c1():
    return _case("C1", 16)


@pytest.fixture(scope="module")
def c2():
    return _case("C2", 8)


@pytest.mark.parametrize("which", ["c1", "c2"])
def test_softplus_query_dense_fp32(which, request):
    cfg, pts, q, m, full = request.getfixturevalue(which)
    ctx = _ctx(cfg)
    ctx.update_scene(pts)
    v, g = ctx.query_values_grads(torch.from_numpy(q))
    torch.cuda.synchronize()
    v = v.cpu().numpy()[:, : len(pts)]
    g = g.cpu().numpy()[:, : len(pts)]
    assert np.all(fp32_close(v, full["f"])), np.abs(v - full["f"]).max()
    bad = ~fp32_close(g, full["g"])
    assert not bad.any(), (bad.sum(), np.abs(g - full["g"]).max())


@pytest.mark.parametrize("which", ["c1", "c2"])
def test_softplus_detect_fp32(which, request):
    cfg, pts, q, m, full = request.getfixturevalue(which)
    # tau: the oracle's 1 % (C1: 5 %) quantile of this network's values (R12's recipe)
    tau = float(np.quantile(full["f"], 0.05 if cfg.name == "C1" else 0.01)) - DELTA
    ctx = _ctx(cfg)
    ids = ctx.update_scene(pts)
    out = ctx.detect_active_set(torch.from_numpy(q), DELTA, tau)
    torch.cuda.synchronize()
    gpu = records_np(out)
    orc = oracle_detect(m, pts, ids, q.reshape(-1, 9), tau, nthreads=NT)

    def gchk(gg, og, kap):
        assert np.all(fp32_close(gg, og))

    nd, nc = compare_active_sets(gpu, orc, full["f"], ids, BAND_FP32, grad_check=gchk, what=which)
    assert nc > 0 and nd <= 0.01 * nc + 2
    assert np.all(fp32_close(out["wp_min"].cpu().numpy(), orc["wp_min"]))


def test_softplus_rejected_by_unsupported_precisions():
    """Softplus runs on GCDF_FP32 and GCDF_FP16; the bf16 and split-fp16 paths refuse it
    (DIM_MISMATCH) instead of silently evaluating ReLU."""
    from paper_2601_18548_b200 import BF16, FP16X3, Context, GcdfError
    for prec in (BF16, FP16X3):
        ctx = Context(0, precision=prec, scene_capacity=1024, max_waypoints=16, max_active=1024)
        with pytest.raises(GcdfError) as e:
            ctx.load_weights(synth.weights_path(128, act=2))
        assert e.value.name == "DIM_MISMATCH"

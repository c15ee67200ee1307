"""NEXT-2 (sparse Jacobian, Eq. 14-19) and NEXT-3 (single-step projection, Theorem 1.2)
on the GPU against the float64 oracle."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import DELTA, records_np

pytestmark = pytest.mark.gpu


def _ctx(cfg, precision):
    from paper_2601_18548_b200 import Context
    ctx = Context(0, precision=precision, scene_capacity=cfg.M + 4096, max_waypoints=cfg.B * cfg.N,
                  max_active=min(cfg.pairs, 1 << 22), max_candidates=cfg.pairs)
    ctx.load_weights(synth.weights_path(cfg.H))
    return ctx


@pytest.mark.parametrize("prec", [0, 2])
@pytest.mark.parametrize("partitioned", [False, True])
def test_sparse_jacobian_matches_oracle_definition(prec, partitioned):
    cfg = synth.get_config("C2")
    pts, _ = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg)[:, :16]
    tau = synth.load_tau(cfg.name)
    ctx = _ctx(cfg, prec)
    ctx.update_scene(pts)
    qt = torch.from_numpy(q)
    out = (ctx.detect_active_set_partitioned(qt, 1.8, DELTA, tau) if partitioned
           else ctx.detect_active_set(qt, DELTA, tau))
    n = int(out["n"])
    assert n > 0
    sj = ctx.sparse_jacobian(out, DELTA)
    torch.cuda.synchronize()
    rec = records_np(out)
    ref = oracle.sparse_jacobian({"value": rec["value"].astype(np.float64), "grad": rec["grad"].astype(np.float64),
                                  "wp": rec["wp"]}, DELTA)
    np.testing.assert_array_equal(sj["row_ptr"][: n + 1].cpu().numpy(), ref["row_ptr"])
    np.testing.assert_array_equal(sj["col"][: 9 * n].cpu().numpy().astype(np.int64), ref["col"])
    np.testing.assert_array_equal(sj["val"][: 9 * n].cpu().numpy(), ref["val"].astype(np.float32))
    # c = f - delta, evaluated in fp32 on the device
    np.testing.assert_array_equal(sj["c"][:n].cpu().numpy(), rec["value"] - np.float32(DELTA))


@pytest.mark.parametrize("prec", [0, 2])
def test_projection_fused_matches_formula_and_oracle(prec):
    """NEXT-3: the fused projection equals q - f M^-1 grad f of the same kernel's dense
    query (tight: only the three fp32 operations differ from f64), and the oracle's
    projection within the path's value/gradient tolerances."""
    from gpu_util import oracle_mlp
    cfg = synth.get_config("C2")
    pts, _ = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg)[:, :4]
    ctx = _ctx(cfg, prec)
    ids = ctx.update_scene(pts)
    qt = torch.from_numpy(q)
    minv = np.random.default_rng(3).uniform(0.2, 3.0, 9)
    v, qz = ctx.project_dense(qt, minv)
    v2, g2 = ctx.query_values_grads(qt)
    torch.cuda.synchronize()
    v, qz, v2, g2 = (x.cpu().numpy() for x in (v, qz, v2, g2))
    np.testing.assert_array_equal(v, v2)
    Q = q.reshape(-1, 9)
    live = np.isfinite(v)
    f64 = np.where(live, v2, 0.0).astype(np.float64)   # dead slots hold +INF
    want = Q[:, None, :].astype(np.float64) - f64[..., None] * (minv * g2.astype(np.float64))
    err = np.abs(qz - want)[live]
    scale = np.abs(Q[:, None, :]).repeat(v.shape[1], 1)[live] + np.abs(f64[..., None] * minv * g2)[live]
    assert np.all(err <= 1e-6 * scale + 1e-6), err.max()
    assert np.all(qz[~live] == 0.0)
    # vs the float64 oracle on a sample of pairs
    m = oracle_mlp(cfg)
    rng = np.random.default_rng(8)
    psel = np.sort(rng.choice(len(pts), 512, replace=False))
    ex = m.eval(pts[psel], Q, want_kappa=True)
    oz = oracle.project(ex["f"], ex["g"], Q, minv)
    gz = qz[:, ids[psel]]
    if prec == 0:   # fp32 path: allclose on pairs away from ReLU kinks
        ok = ex["kappa"] > 1e-4
        d = np.abs(gz - oz)[ok]
        assert np.all(d <= 1e-4 * (np.abs(oz[ok]) + np.abs((ex["f"][..., None] * minv * ex["g"]))[ok]) + 1e-5)
    else:           # tensor path: |f| error <= 2e-2 and the gradient-norm gate bound the step
        dz = np.linalg.norm(gz - oz, axis=-1)
        step = np.abs(ex["f"]) * np.linalg.norm(minv * ex["g"], axis=-1)
        assert np.median(dz / (step + 1e-3)) < 0.05


@pytest.mark.parametrize("radius", [0.0, 1.8])
def test_detect_graph_replays_direct_call(radius):
    """The CUDA-graph detect equals the direct call bit for bit: for new q contents written
    in place, and across scene updates (automatic re-capture)."""
    cfg = synth.get_config("C2")
    pts, boxes = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg)[:, :16]
    tau = synth.load_tau(cfg.name)
    ctx = _ctx(cfg, 2)
    osc = oracle.Scene(cfg.M + 4096)
    ctx.update_scene(pts)
    osc.update(pts)
    qd = torch.from_numpy(q).cuda()
    g = ctx.detect_graph(qd, DELTA, tau, radius=radius)
    rng = np.random.default_rng(5)
    for it in range(4):
        if it == 2:  # scene update -> re-capture at the next launch
            ids, _ = osc.export()
            add, rem = synth.scene_update_batch(rng, boxes, ids)
            ctx.update_scene(add, rem)
            osc.update(add, rem)
        qn = q + rng.normal(0, 0.05, q.shape).astype(np.float32) * (it > 0)
        qd.copy_(torch.from_numpy(qn))
        go = g.launch()
        d = (ctx.detect_active_set_partitioned(qd, radius, DELTA, tau) if radius > 0
             else ctx.detect_active_set(qd, DELTA, tau))
        assert go["n"] == d["n"] > 0
        n = d["n"]
        assert torch.equal(go["records"][:n], d["records"][:n])
        for k in ("wp_offsets", "wp_min", "wp_argmin"):
            assert torch.equal(go[k], d[k]), k
    g.close()

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
    ex = m.eval(pts[psel], Q, want_kappa=True, want_hash=True)
    oz = oracle.project(ex["f"], ex["g"], Q, minv)
    gz = qz[:, ids[psel]]
    if prec == 0:   # fp32 path: allclose on pairs away from ReLU kinks
        ok = ex["kappa"] > 1e-4
        d = np.abs(gz - oz)[ok]
        assert np.all(d <= 1e-4 * (np.abs(oz[ok]) + np.abs((ex["f"][..., None] * minv * ex["g"]))[ok]) + 1e-5)
    else:
        # tensor path, element by element.  (i) vs the oracle's EMU_FP16 projection (the same
        # operand rounding): every component of every pair whose GPU gradient took the
        # emulation's ReLU branches (gate 1 of tests/test_gpu_tensor.py), >= 99 % of pairs
        em = m.eval(pts[psel], Q, flags=oracle.EMU_FP16, want_kappa=True, want_hash=True)
        oze = oracle.project(em["f"], em["g"], Q, minv)
        g_gpu = g2[:, ids[psel]].astype(np.float64)
        same = (np.linalg.norm(g_gpu - em["g"], axis=-1) <= 1e-2 * np.maximum(1.0, np.linalg.norm(em["g"], axis=-1)))
        assert same.mean() >= 0.99, same.mean()
        scale_e = np.abs(oze) + np.abs(em["f"][..., None] * minv * em["g"])
        err_e = np.abs(gz - oze)
        bound_e = 1e-2 * np.abs(em["f"][..., None] * minv) * np.maximum(1.0, np.linalg.norm(em["g"], axis=-1))[..., None] \
            + 1e-5 * scale_e + 1e-3 * minv * np.abs(em["g"]) + 1e-5
        assert np.all((err_e <= bound_e)[same]), (err_e - bound_e)[same].max()
        # (ii) vs the exact oracle: every component of every kink-free pair (exact ReLU masks =
        # emulated masks, the GPU on the emulation's branch) within the value tolerance 2e-2
        # times |M^-1 grad| plus |f| M^-1 times the gradient tolerance 5e-2
        kf = (ex["mask_hash"] == em["mask_hash"]) & (em["kappa"] > 1e-3) & same
        bound_x = minv * (2e-2 * np.abs(ex["g"]) + 5e-2 * np.abs(ex["f"])[..., None]) + 1e-5 * np.abs(oz) + 1e-5
        err_x = np.abs(gz - oz)
        assert kf.mean() > 0.5, kf.mean()
        assert np.all((err_x <= bound_x)[kf]), (err_x - bound_x)[kf].max()


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


def _same_detect(a, b):
    assert a["n"] == b["n"] > 0
    n = a["n"]
    assert torch.equal(a["records"][:n], b["records"][:n])
    for k in ("wp_offsets", "wp_min", "wp_argmin"):
        assert torch.equal(a[k], b[k]), k


def test_detect_graph_recaptures_after_weight_reload():
    """A captured detect holds the output row, the bias and the chosen kernel by value: after
    gcdf_load_weights the next launch re-captures and equals the direct call with the new
    weights (dense and partitioned graphs; the second network has another activation, so
    another kernel)."""
    cfg = synth.get_config("C2")
    pts, _ = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg)[:, :8]
    tau = 2.0  # f - delta <= 2 holds for a large share of the pairs of all three networks
    ctx = _ctx(cfg, 2)
    ctx.update_scene(pts)
    qd = torch.from_numpy(q).cuda()
    graphs = {r: ctx.detect_graph(qd, DELTA, tau, radius=r) for r in (0.0, 1.8)}
    for path in (synth.weights_path(cfg.H, seed=8), synth.weights_path(cfg.H, act=2)):
        ctx.load_weights(path)
        for r, g in graphs.items():
            go = g.launch()
            d = ctx.detect_active_set_partitioned(qd, r, DELTA, tau) if r > 0 else ctx.detect_active_set(qd, DELTA, tau)
            _same_detect(go, d)
    for g in graphs.values():
        g.close()


def test_partitioned_graph_after_call_at_another_radius():
    """A direct partitioned call at another radius rebuilds the partition grid; the graph
    captured at r = 1.8 must still replay the r = 1.8 partition (the grid is rebuilt at the
    graph's radius before the replay)."""
    cfg = synth.get_config("C2")
    pts, _ = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg)[:, :8]
    tau = synth.load_tau(cfg.name)
    ctx = _ctx(cfg, 2)
    ctx.update_scene(pts)
    qd = torch.from_numpy(q).cuda()
    g = ctx.detect_graph(qd, DELTA, tau, radius=1.8)
    ref = {k: (v.clone() if torch.is_tensor(v) else v) for k, v in g.launch().items()}
    for r in (3.0, 0.9, 1.8, 3.0):
        other = ctx.detect_active_set_partitioned(qd, r, DELTA, tau)
        go = g.launch()
        _same_detect(go, ref)
        if r != 1.8:
            assert other["n"] != ref["n"]
    g.close()


def test_detect_graph_rejects_a_converted_q():
    """The graph replays the captured q pointer: a q that needs a dtype / layout conversion
    (a private copy) is refused instead of being silently frozen."""
    cfg = synth.get_config("C1")
    pts, _ = synth.make_scene_points(cfg)
    ctx = _ctx(cfg, 0)
    ctx.update_scene(pts)
    q64 = torch.from_numpy(synth.make_waypoints(cfg)).double().cuda()
    with pytest.raises(ValueError):
        ctx.detect_graph(q64, DELTA, 0.5)

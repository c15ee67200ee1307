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
    """Softplus runs on GCDF_FP32 and on GCDF_FP16 in the translation frame; the bf16 and
    split-fp16 paths and the SE(2) tensor path refuse it (DIM_MISMATCH) instead of silently
    evaluating ReLU."""
    from paper_2601_18548_b200 import BF16, FP16, FP16X3, FRAME_SE2, Context, GcdfError
    for prec, kw in ((BF16, {}), (FP16X3, {}), (FP16, {"frame": FRAME_SE2})):
        ctx = Context(0, precision=prec, scene_capacity=1024, max_waypoints=16, max_active=1024, **kw)
        with pytest.raises(GcdfError) as e:
            ctx.load_weights(synth.weights_path(128, act=2))
        assert e.value.name == "DIM_MISMATCH"


# ------------------------------------------------------------------ tensor-core path (K2s)
# Gates (R17 / R26): vs the oracle's EMU_FP16 mode (same rounding points: 16-bit A operands,
# sigma' of layers 1..5 from the rounded activation) median |df| at fp32 noise, max |df| <=
# 5e-3 and ||dg|| <= 1e-2 max(1, ||g||) on every pair; vs the exact oracle the north-star tensor-path tolerances
# |df| <= 2e-2 and | ||g|| - ||g_exact|| | <= 5e-2 -- on every pair, since the softplus
# field has no kinks.
TC_EMU_VAL_MAX, TC_EMU_GREL, TC_VAL, TC_GNORM = 5e-3, 1e-2, 2e-2, 5e-2


def _tc_gates(v, g, exact, emu, what):
    dv_emu = np.abs(v - emu["f"])
    dg_emu = np.linalg.norm(g - emu["g"], axis=-1)
    gn_emu = np.linalg.norm(emu["g"], axis=-1)
    dv = np.abs(v - exact["f"])
    dgn = np.abs(np.linalg.norm(g, axis=-1) - np.linalg.norm(exact["g"], axis=-1))
    print(f"{what}: |df| vs EMU median {np.median(dv_emu):.2e} p99 {np.quantile(dv_emu, 0.99):.2e} max "
          f"{dv_emu.max():.2e}; vs exact max {dv.max():.2e}; ||dg|| vs EMU median {np.median(dg_emu):.2e} max "
          f"{dg_emu.max():.2e}; gnorm diff vs exact max {dgn.max():.2e}")
    # same rounding points: fp32 noise in the median; the tail is where the MUFU-approximated
    # softplus lands on the other side of a 16-bit rounding boundary than the f64 one
    assert np.median(dv_emu) <= 1e-6 and dv_emu.max() <= TC_EMU_VAL_MAX, what
    assert np.median(dg_emu) <= 1e-5 and np.all(dg_emu <= TC_EMU_GREL * np.maximum(1.0, gn_emu)), what
    assert dv.max() <= TC_VAL, (what, dv.max())
    assert dgn.max() <= TC_GNORM, (what, dgn.max())


@pytest.fixture(scope="module")
def c2_tc():
    cfg, pts, q, m, full = _case("C2", 8)
    emu = m.eval(pts, q.reshape(-1, 9), flags=oracle.EMU_FP16, nthreads=NT)
    return cfg, pts, q, m, full, emu


def test_softplus_query_dense_tensor(c2_tc):
    from paper_2601_18548_b200 import FP16
    cfg, pts, q, m, full, emu = c2_tc
    ctx = _ctx(cfg, precision=FP16)
    ctx.update_scene(pts)
    v, g = ctx.query_values_grads(torch.from_numpy(q))
    torch.cuda.synchronize()
    vt, gt = v.cpu().numpy(), g.cpu().numpy()
    M = len(pts)
    assert np.all(np.isinf(vt[:, M:])) and np.all(gt[:, M:] == 0)  # dead tail slots
    _tc_gates(vt[:, :M], gt[:, :M], full, emu, "C2/8 dense fp16 softplus")


def test_softplus_detect_tensor(c2_tc):
    from paper_2601_18548_b200 import FP16
    cfg, pts, q, m, full, emu = c2_tc
    tau = float(np.quantile(full["f"], 0.01)) - DELTA
    ctx = _ctx(cfg, precision=FP16)
    ids = ctx.update_scene(pts)
    qt = torch.from_numpy(q)
    out = ctx.detect_active_set(qt, DELTA, tau)
    v, g = ctx.query_values_grads(qt)
    torch.cuda.synchronize()
    gpu = records_np(out)
    orc = oracle_detect(m, pts, ids, q.reshape(-1, 9), tau, nthreads=NT)

    def gchk(gg, og, kap):
        assert np.all(np.abs(np.linalg.norm(gg, axis=-1) - np.linalg.norm(og, axis=-1)) <= TC_GNORM)

    nd, nc = compare_active_sets(gpu, orc, full["f"], ids, BAND_FP32 + TC_VAL, val_atol=TC_VAL, grad_check=gchk,
                                 what="C2/8 detect fp16 softplus")
    assert nc > 0
    # the fused detect's records are the dense query's values and gradients, bit for bit
    vn, gn = v.cpu().numpy(), g.cpu().numpy()
    assert np.array_equal(gpu["value"], vn[gpu["wp"], gpu["pt"]])
    assert np.array_equal(gpu["grad"], gn[gpu["wp"], gpu["pt"]])
    assert np.all(np.abs(out["wp_min"].cpu().numpy() - orc["wp_min"]) <= TC_VAL)


def test_softplus_tensor_c1_shape_and_partition():
    """Ragged tails on the tensor path: C1 points (256 = 2 tiles) under the H = 128
    softplus network, dense and range-partitioned detect vs the EMU oracle."""
    from paper_2601_18548_b200 import FP16
    cfg = synth.get_config("C1")
    pts, _ = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg)
    m = oracle.MLP(synth.weights_path(128, act=2))
    full = m.eval(pts, q.reshape(-1, 9), nthreads=NT)
    emu = m.eval(pts, q.reshape(-1, 9), flags=oracle.EMU_FP16, nthreads=NT)
    from paper_2601_18548_b200 import Context
    ctx = Context(0, precision=FP16, scene_capacity=4096, max_waypoints=64, max_active=1 << 16,
                  max_candidates=1 << 16)
    ctx.load_weights(synth.weights_path(128, act=2))
    ids = ctx.update_scene(pts[:200])  # 200 live points: a ragged second tile
    v, g = ctx.query_values_grads(torch.from_numpy(q))
    torch.cuda.synchronize()
    sub = {k: full[k][:, :200] for k in ("f", "g")}
    esub = {k: emu[k][:, :200] for k in ("f", "g")}
    _tc_gates(v.cpu().numpy()[:, :200], g.cpu().numpy()[:, :200], sub, esub, "C1 dense fp16 softplus")
    tau = float(np.quantile(sub["f"], 0.2)) - DELTA
    part = ctx.detect_active_set_partitioned(torch.from_numpy(q), 3.0, DELTA, tau)
    torch.cuda.synchronize()
    gp = records_np(part)
    orc = m.detect(pts[:200], ids, q.reshape(-1, 9), DELTA, tau, nthreads=NT, radius=3.0)
    orc["_tau"] = tau
    nd, nc = compare_active_sets(gp, orc, sub["f"], ids, BAND_FP32 + TC_VAL, val_atol=TC_VAL,
                                 what="C1 partitioned fp16 softplus")
    assert nc > 0


def test_softplus_c5_full_size_sampled():
    """The bench configuration of the variant (python bench.py --activation softplus: C5,
    256 waypoints x 1M points, fp16 K2s, full-size detect): sampled pairs against the EMU and
    exact oracles one by one, sampled active-set memberships, and the per-waypoint min."""
    from paper_2601_18548_b200 import FP16
    cfg = synth.get_config("C5")
    pts, _ = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg)
    tau = synth.load_tau("C5", 2)
    ctx = _ctx(cfg, precision=FP16)
    ids = ctx.update_scene(pts)
    out = ctx.detect_active_set(torch.from_numpy(q), DELTA, tau)
    torch.cuda.synchronize()
    gpu = records_np(out)
    m = oracle.MLP(synth.weights_path(cfg.H, act=2))
    Q = q.reshape(-1, 9)
    rng = np.random.default_rng(2025)
    wsel = np.sort(rng.choice(Q.shape[0], 3, replace=False))
    psel = np.sort(rng.choice(len(pts), 4096, replace=False))
    ex = m.eval(pts[psel], Q[wsel], nthreads=NT)
    em = m.eval(pts[psel], Q[wsel], flags=oracle.EMU_FP16, nthreads=NT)
    v, g = ctx.query_values_grads(torch.from_numpy(Q[wsel].reshape(1, -1, 9)))
    _tc_gates(v.cpu().numpy()[:, psel], g.cpu().numpy()[:, psel], ex, em, "C5 sampled fp16 softplus")
    recset = set(zip(gpu["wp"].tolist(), gpu["pt"].tolist()))
    thr = tau + DELTA
    checked = 0
    for wi, w in enumerate(wsel):
        for pj, pid in enumerate(psel):
            f = ex["f"][wi, pj]
            if abs(f - thr) > BAND_FP32 + TC_VAL:
                assert ((int(w), int(ids[pid])) in recset) == (f <= thr), (w, pid, f)
                checked += 1
    assert checked > 0.9 * len(wsel) * len(psel)
    assert np.all(out["wp_min"].cpu().numpy()[wsel] <= ex["f"].min(axis=1) + TC_VAL)
    frac = out["n"] / (len(pts) * Q.shape[0])
    assert 0.001 < frac < 0.05, frac

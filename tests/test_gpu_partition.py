"""NEXT-1 range-partitioned detect (R23) on the GPU:
against the float64 oracle's partitioned detect, and against the GPU's own unpartitioned
detect filtered by distance (bit-identical values: each pair's arithmetic is independent
of which tile carries it)."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import BAND_FP32, BF16_VAL_ATOL, DELTA, fp32_close, oracle_mlp, records_np

pytestmark = pytest.mark.gpu
NT = max(1, min(os.cpu_count() or 1, 64))
R = 1.8                      # SPEC.md part_radius
DIST_BAND = 1e-4             # membership may differ within 1e-4 m of the circle (fp32 test, R23)


def _ctx(cfg, precision, max_candidates=None, extra=4096):
    from paper_2601_18548_b200 import Context
    ctx = Context(0, precision=precision, scene_capacity=cfg.M + extra, max_waypoints=cfg.B * cfg.N,
                  max_active=min(cfg.pairs, 1 << 22),
                  max_candidates=max_candidates if max_candidates is not None else cfg.pairs)
    ctx.load_weights(synth.weights_path(cfg.H))
    return ctx


def _dist(pts, q):
    return np.sqrt((pts[None, :, 0] - q[:, None, 0]) ** 2 + (pts[None, :, 1] - q[:, None, 1]) ** 2)


@pytest.fixture(scope="module")
def c2():
    cfg = synth.get_config("C2")
    pts, boxes = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg)[:, :24]
    return cfg, pts, boxes, q


@pytest.mark.parametrize("prec", [0, 2])
def test_partitioned_vs_oracle(c2, prec):
    cfg, pts, _, q = c2
    tau = synth.load_tau(cfg.name)
    ctx = _ctx(cfg, prec)
    ids = ctx.update_scene(pts)
    Q = q.reshape(-1, 9)
    out = ctx.detect_active_set_partitioned(torch.from_numpy(q), R, DELTA, tau)
    gpu = records_np(out)
    m = oracle_mlp(cfg)
    od = m.detect(pts, ids, Q, DELTA, tau, radius=R, nthreads=NT)
    d = _dist(pts.astype(np.float64), Q)
    border = np.abs(d - R) <= DIST_BAND
    psz = out["part_sizes"].cpu().numpy()
    assert np.all(np.abs(psz - od["part_sizes"]) <= border.sum(axis=1))
    val_atol = 1e-5 if prec == 0 else BF16_VAL_ATOL
    band = BAND_FP32 if prec == 0 else BAND_FP32 + BF16_VAL_ATOL
    F = m.eval(pts, Q, want_grad=False, nthreads=NT)["f"]
    pos = {int(i): j for j, i in enumerate(ids)}
    g = set(zip(gpu["wp"].tolist(), gpu["pt"].tolist()))
    o = set(zip(od["wp"].tolist(), od["pt"].tolist()))
    for (w, p) in g ^ o:
        j = pos[p]
        assert border[w, j] or abs(F[w, j] - DELTA - tau) <= band, (w, p)
    # matched records: values (and for fp32, gradients) vs the oracle
    ok = [(k, pos[p]) for k, (w, p) in enumerate(zip(gpu["wp"], gpu["pt"])) if (int(w), int(p)) in o]
    ks = np.array([k for k, _ in ok])
    js = np.array([j for _, j in ok])
    fo = F[gpu["wp"][ks], js]
    if prec == 0:
        assert np.all(fp32_close(gpu["value"][ks], fo))
    else:
        assert np.all(np.abs(gpu["value"][ks] - fo) <= val_atol)
    # per-step minimum over the partition
    wmin = out["wp_min"].cpu().numpy()
    for w in range(Q.shape[0]):
        inside = d[w] <= R
        if inside.any() and not border[w].any():
            assert abs(wmin[w] - F[w, inside].min()) <= val_atol + 1e-4 * abs(F[w, inside].min())
    frac = out["n"] / max(psz.sum(), 1)
    print(f"\npartition r={R}: {psz.sum()} of {len(pts) * Q.shape[0]} pairs "
          f"({psz.sum() / (len(pts) * Q.shape[0]):.2%}), {out['n']} active ({frac:.2%} of the partition pairs)")


def _in_fp32(xyz, Q, w, r):
    """The kernel's membership test, replicated in float32 (RN, no FMA)."""
    ex = np.float32(xyz[0]) - np.float32(Q[w, 0])
    ey = np.float32(xyz[1]) - np.float32(Q[w, 1])
    rr = np.float32(r) * np.float32(r)
    return np.float32(ex * ex) + np.float32(ey * ey) <= rr


@pytest.mark.parametrize("prec", [0, 2])
def test_partitioned_equals_filtered_unpartitioned(c2, prec):
    """Bit-identical records to the unpartitioned detect restricted to the partition pairs
    (membership replicated in fp32); a radius covering the scene reproduces the
    unpartitioned detect exactly; the grid is rebuilt after scene updates and radius
    changes (three rounds of 200 removes + 200 adds)."""
    cfg, pts, boxes, q = c2
    tau = synth.load_tau(cfg.name)
    ctx = _ctx(cfg, prec)
    osc = oracle.Scene(cfg.M + 4096)
    assert np.array_equal(ctx.update_scene(pts), osc.update(pts))
    qt = torch.from_numpy(q)
    Q = q.reshape(-1, 9)
    rng = np.random.default_rng(77)
    for step in range(3):
        ids, xyz = osc.export()
        pos = {int(i): j for j, i in enumerate(ids)}
        full = records_np(ctx.detect_active_set(qt, DELTA, tau))
        for r in (R, 3.0):
            part = records_np(ctx.detect_active_set_partitioned(qt, r, DELTA, tau))
            keep = np.array([_in_fp32(xyz[pos[int(p)]], Q, int(w), r) for w, p in zip(full["wp"], full["pt"])],
                            dtype=bool)
            for k in ("wp", "pt", "value", "grad"):
                np.testing.assert_array_equal(part[k], full[k][keep], err_msg=f"{k} r={r} step={step}")
        big = ctx.detect_active_set_partitioned(qt, 1e4, DELTA, tau)
        b = records_np(big)
        for k in ("wp", "pt", "value", "grad"):
            np.testing.assert_array_equal(b[k], full[k])
        fo = ctx.detect_active_set(qt, DELTA, tau)
        assert torch.equal(big["wp_min"], fo["wp_min"]) and torch.equal(big["wp_argmin"], fo["wp_argmin"])
        assert int(big["part_sizes"].sum().item()) == len(ids) * Q.shape[0]
        add, rem = synth.scene_update_batch(rng, boxes, ids)
        assert np.array_equal(ctx.update_scene(add, rem), osc.update(add, rem))


def test_partition_capacity_and_arguments(c2):
    from paper_2601_18548_b200 import GcdfError
    cfg, pts, _, q = c2
    tau = synth.load_tau(cfg.name)
    qt = torch.from_numpy(q)
    small = _ctx(cfg, 2, max_candidates=1000)
    small.update_scene(pts)
    with pytest.raises(GcdfError) as e:
        small.detect_active_set_partitioned(qt, R, DELTA, tau)
    assert e.value.name == "CAPACITY"
    assert int(small.detect_active_set(qt, DELTA, tau)["n"]) > 0  # the context stays usable
    off = _ctx(cfg, 2, max_candidates=0)
    off.update_scene(pts)
    with pytest.raises(GcdfError) as e:
        off.detect_active_set_partitioned(qt, R, DELTA, tau)
    assert e.value.name == "INVALID_ARG"
    for bad in (0.0, -1.0, float("inf"), float("nan")):
        with pytest.raises(GcdfError):
            small.detect_active_set_partitioned(qt, bad, DELTA, tau)

"""GPU parity of the fp32 path (GCDF_FP32) against the float64 oracle, through the C ABI.

Sizes: C1 in full (H = 32, 4,096 pairs, ragged tail: 256 = 2 tiles), C2 on 16 of its 64
waypoints (160,000 pairs, 79 tiles per waypoint with a ragged last tile of 16 points).
"""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import (BAND_FP32, DELTA, KINK_FP32, check_fp32_dense, compare_active_sets, fp32_close,
                      oracle_detect, oracle_mlp, records_np)

pytestmark = pytest.mark.gpu
NT = max(1, min(os.cpu_count() or 1, 64))


def _ctx(cfg, precision=0, extra_cap=4096, **kw):
    from paper_2601_18548_b200 import Context
    ctx = Context(0, precision=precision, scene_capacity=cfg.M + extra_cap, max_waypoints=cfg.B * cfg.N,
                  max_active=min(cfg.pairs, 1 << 22), **kw)
    ctx.load_weights(synth.weights_path(cfg.H))
    return ctx


@pytest.fixture(scope="module")
def c1():
    cfg = synth.get_config("C1")
    pts, _ = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg)
    m = oracle_mlp(cfg)
    full = m.eval(pts, q.reshape(-1, 9), want_kappa=True, nthreads=NT)
    return cfg, pts, q, m, full


@pytest.fixture(scope="module")
def c2():
    cfg = synth.get_config("C2")
    pts, _ = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg)[:, :16]
    m = oracle_mlp(cfg)
    full = m.eval(pts, q.reshape(-1, 9), want_kappa=True, nthreads=NT)
    return cfg, pts, q, m, full


@pytest.mark.parametrize("which", ["c1", "c2"])
def test_query_dense_fp32(which, request):
    cfg, pts, q, m, full = request.getfixturevalue(which)
    ctx = _ctx(cfg)
    ids = ctx.update_scene(pts)
    assert np.array_equal(ids, np.arange(len(pts)))
    info = ctx.scene_info()
    assert info["n_live"] == len(pts) and info["local_bound"] % 128 == 0
    v, g = ctx.query_values_grads(torch.from_numpy(q))
    torch.cuda.synchronize()
    v = v.cpu().numpy()[:, : len(pts)]
    g = g.cpu().numpy()[:, : len(pts)]
    nk = check_fp32_dense(v, g, full["f"], full["g"], full["kappa"], what=which)
    # dead tail slots: +INF value, zero gradient
    vt, gt = ctx.query_values_grads(torch.from_numpy(q))
    vt = vt.cpu().numpy()[:, len(pts):]
    assert np.all(np.isinf(vt) & (vt > 0)) and np.all(gt.cpu().numpy()[:, len(pts):] == 0)
    print(f"{which}: {v.size} pairs, {nk} gradients differ within {KINK_FP32} of a ReLU kink")


@pytest.mark.parametrize("which", ["c1", "c2"])
def test_detect_fp32(which, request):
    cfg, pts, q, m, full = request.getfixturevalue(which)
    tau = synth.load_tau(cfg.name)
    ctx = _ctx(cfg)
    ids = ctx.update_scene(pts)
    out = ctx.detect_active_set(torch.from_numpy(q), DELTA, tau)
    torch.cuda.synchronize()
    gpu = records_np(out)
    orc = oracle_detect(m, pts, ids, q.reshape(-1, 9), tau, nthreads=NT)

    def gchk(gg, og, kap):
        bad = ~np.all(fp32_close(gg, og), axis=-1)
        assert not (bad & (kap > KINK_FP32)).any()

    nd, nc = compare_active_sets(gpu, orc, full["f"], ids, BAND_FP32, grad_check=gchk, kappa_full=full["kappa"],
                                 what=which)
    assert nc > 0 and nd <= 0.01 * nc + 2
    # per-waypoint min / argmin (union = min)
    wmin = out["wp_min"].cpu().numpy()
    warg = out["wp_argmin"].cpu().numpy()
    assert np.all(fp32_close(wmin, orc["wp_min"]))
    F = full["f"]
    srt = np.sort(F, axis=1)
    clear = (srt[:, 1] - srt[:, 0]) > 1e-4  # argmin unique beyond fp32 error
    assert np.array_equal(warg[clear], orc["wp_argmin"][clear])
    # offsets are the per-waypoint block structure of the GPU's own records
    offs = out["wp_offsets"].cpu().numpy()
    assert offs[0] == 0 and offs[-1] == out["n"] and np.all(np.diff(offs) >= 0)
    assert np.array_equal(np.searchsorted(gpu["wp"], np.arange(len(offs)), side="left"), offs)


def test_compaction_exact_vs_own_values(c2):
    """T2: K3 over the GPU's own dense values equals a brute-force filter of those values,
    bit for bit and in order; the fused detect produces the identical record stream."""
    cfg, pts, q, m, full = c2
    tau = synth.load_tau(cfg.name)
    ctx = _ctx(cfg)
    ctx.update_scene(pts)
    qt = torch.from_numpy(q)
    v, g = ctx.query_values_grads(qt)
    dense = ctx.compact_dense(v, g, DELTA, tau)
    fused = ctx.detect_active_set(qt, DELTA, tau)
    torch.cuda.synchronize()
    vn, gn = v.cpu().numpy(), g.cpu().numpy()
    W, lb = vn.shape
    live = np.zeros(lb, bool)
    live[: len(pts)] = True
    act = (vn - np.float32(DELTA) <= np.float32(tau)) & live[None, :]
    w_idx, s_idx = np.nonzero(act)
    a = records_np(dense)
    assert dense["n"] == len(w_idx)
    assert np.array_equal(a["wp"], w_idx) and np.array_equal(a["pt"], s_idx)
    assert np.array_equal(a["value"], vn[w_idx, s_idx]) and np.array_equal(a["grad"], gn[w_idx, s_idx])
    b = records_np(fused)
    for k in ("wp", "pt", "value", "grad"):
        assert np.array_equal(a[k], b[k]), k
    vm = np.where(live[None, :], vn, np.inf)
    assert np.array_equal(dense["wp_min"].cpu().numpy(), vm.min(1))
    assert np.array_equal(dense["wp_argmin"].cpu().numpy(), vm.argmin(1))
    assert np.array_equal(fused["wp_min"].cpu().numpy(), vm.min(1))


@pytest.mark.parametrize("frac", [0.3, 1.0])
def test_compaction_dense_activity(c2, frac):
    """K3 with a large active fraction (hundreds of actives per 8-tile unit, thousands per
    32-unit emit batch, so the emit kernel's record list fills and drains in pieces): bit-exact
    against a filter of the same values, offsets included; an output capacity below the count
    gives CAPACITY with the first `capacity` records still exact."""
    from paper_2601_18548_b200 import GcdfError
    cfg, pts, q, m, full = c2
    ctx = _ctx(cfg)
    ctx.update_scene(pts)
    v, g = ctx.query_values_grads(torch.from_numpy(q))
    torch.cuda.synchronize()
    vn, gn = v.cpu().numpy(), g.cpu().numpy()
    W, lb = vn.shape
    live = np.zeros(lb, bool)
    live[: len(pts)] = True
    tau = float(np.quantile(vn[:, : len(pts)], frac)) if frac < 1 else 1e30
    act = (vn - np.float32(DELTA) <= np.float32(tau)) & live[None, :]
    w_idx, s_idx = np.nonzero(act)
    assert len(w_idx) > 0.25 * W * len(pts) * min(frac, 1.0)
    dense = ctx.compact_dense(v, g, DELTA, tau)
    a = records_np(dense)
    assert dense["n"] == len(w_idx)
    assert np.array_equal(a["wp"], w_idx) and np.array_equal(a["pt"], s_idx)
    assert np.array_equal(a["value"], vn[w_idx, s_idx]) and np.array_equal(a["grad"], gn[w_idx, s_idx])
    assert np.array_equal(dense["wp_offsets"].cpu().numpy(), np.searchsorted(w_idx, np.arange(W + 1), side="left"))
    cap = len(w_idx) // 3 + 7
    o = ctx.alloc_detect_outputs(W, cap)
    with pytest.raises(GcdfError):
        ctx.compact_dense(v, g, DELTA, tau, outputs=o)
    b = records_np({"records": o["records"], "n": cap, "capacity": cap})
    assert np.array_equal(b["wp"], w_idx[:cap]) and np.array_equal(b["pt"], s_idx[:cap])
    assert np.array_equal(b["value"], vn[w_idx[:cap], s_idx[:cap]])


def test_pairgen_transform(c1):
    """A2 standalone: p' = fl32(p - q_xy) exactly (one fp32 rounding of the f64 difference)."""
    cfg, pts, q, m, full = c1
    ctx = _ctx(cfg)
    ctx.update_scene(pts)
    out = ctx.pairgen_transform(torch.from_numpy(q)).cpu().numpy()
    qq = q.reshape(-1, 9).astype(np.float64)
    M = len(pts)
    ex = pts[None, :, 0].astype(np.float64) - qq[:, None, 0]
    ey = pts[None, :, 1].astype(np.float64) - qq[:, None, 1]
    assert np.array_equal(out[:, :M, 0], ex.astype(np.float32))
    assert np.array_equal(out[:, :M, 1], ey.astype(np.float32))
    assert np.array_equal(out[:, :M, 2], np.broadcast_to(pts[:, 2], (qq.shape[0], M)))
    assert np.all(out[:, :M, 3] == 1.0) and np.all(out[:, M:, 3] == 0.0)


def test_scene_updates_match_oracle_replay(c1):
    """T3 / P5: random add/remove script; ids equal the oracle's replay of the id rule and
    detect equals the oracle on the replayed id -> xyz map after every step."""
    cfg, pts, q, m, full = c1
    tau = synth.load_tau(cfg.name)
    ctx = _ctx(cfg, extra_cap=384)
    osc = oracle.Scene(cfg.M + 384)
    assert np.array_equal(ctx.update_scene(pts), osc.update(pts))
    _, boxes = synth.make_scene_points(cfg)
    rng = np.random.default_rng(77)
    qt = torch.from_numpy(q)
    for step in range(4):
        live, _ = osc.export()
        add, rem = synth.scene_update_batch(rng, boxes, live, n_remove=40 + 20 * step, n_add=50)
        gids = ctx.update_scene(add, rem)
        oids = osc.update(add, rem)
        assert np.array_equal(gids, oids), step
        oi, oxyz = osc.export()
        info = ctx.scene_info()
        assert info["n_live"] == len(oi)
        out = ctx.detect_active_set(qt, DELTA, tau)
        torch.cuda.synchronize()
        gpu = records_np(out)
        orc = oracle_detect(m, oxyz, oi, q.reshape(-1, 9), tau, nthreads=NT)
        ff = m.eval(oxyz, q.reshape(-1, 9), want_grad=False, nthreads=NT)["f"]
        compare_active_sets(gpu, orc, ff, oi, BAND_FP32, what=f"step {step}")
        assert np.all(fp32_close(out["wp_min"].cpu().numpy(), orc["wp_min"]))


def test_errors_are_atomic(c1):
    from paper_2601_18548_b200 import GcdfError
    cfg, pts, q, m, full = c1
    ctx = _ctx(cfg, extra_cap=0)
    ctx.update_scene(pts[:100])
    with pytest.raises(GcdfError) as e:
        ctx.update_scene(pts[:5], remove_ids=[3, 3])
    assert e.value.name == "UNKNOWN_ID"
    with pytest.raises(GcdfError) as e:
        ctx.update_scene(pts[:5], remove_ids=[100])
    assert e.value.name == "UNKNOWN_ID"
    bad = pts[:2].copy()
    bad[1, 2] = np.nan
    with pytest.raises(GcdfError) as e:
        ctx.update_scene(bad)
    assert e.value.name == "NONFINITE"
    assert ctx.scene_info()["n_live"] == 100
    with pytest.raises(GcdfError) as e:  # capacity (cfg.M + 0 slots... rounded up to 256)
        ctx.update_scene(np.zeros((10_000, 3), np.float32))
    assert e.value.name == "CAPACITY"
    with pytest.raises(GcdfError) as e:
        ctx.detect_active_set(torch.zeros((2, cfg.N, 9)), DELTA, 0.0)  # B*N > max_waypoints
    assert e.value.name == "CAPACITY"
    with pytest.raises(GcdfError) as e:
        ctx.load_weights("/nonexistent.mlpw")
    assert e.value.name == "IO"
    # detect output capacity: count stays exact, CAPACITY reported
    tau = synth.load_tau(cfg.name)
    with pytest.raises(GcdfError) as e:
        ctx.detect_active_set(torch.from_numpy(q), DELTA, tau + 10.0, capacity=7)
    assert e.value.name == "CAPACITY"
    ok = ctx.detect_active_set(torch.from_numpy(q), DELTA, tau + 10.0, capacity=100 * cfg.N)
    assert ok["n"] == 100 * cfg.N  # every live pair active


def test_empty_scene(c1):
    cfg, pts, q, m, full = c1
    ctx = _ctx(cfg)
    out = ctx.detect_active_set(torch.from_numpy(q), DELTA, 0.0)
    assert out["n"] == 0
    assert torch.all(torch.isinf(out["wp_min"])) and torch.all(out["wp_argmin"] == -1)
    assert torch.all(out["wp_offsets"] == 0)
    ids = ctx.update_scene(pts[:3])
    ctx.update_scene(remove_ids=ids)
    out = ctx.detect_active_set(torch.from_numpy(q), DELTA, 100.0)
    assert out["n"] == 0 and torch.all(out["wp_argmin"] == -1)


def test_virtual_ranks_merge_bitexact(c2):
    """T4f: the obstacle points sharded over 2 and 3 'virtual ranks' on one GPU; per-rank
    detect + device gather (concatenation) + merge kernel == the 1-rank result, bit for bit."""
    cfg, pts, q, m, full = c2
    tau = synth.load_tau(cfg.name)
    qt = torch.from_numpy(q)
    ref = _ctx(cfg)
    ref.update_scene(pts)
    r1 = ref.detect_active_set(qt, DELTA, tau)
    a = records_np(r1)
    for world in (2, 3):
        ctxs = [_ctx(cfg, rank=r, world=world) for r in range(world)]
        outs = []
        for c in ctxs:
            assert np.array_equal(c.update_scene(pts), np.arange(len(pts)))
            outs.append(c.detect_active_set(qt, DELTA, tau))
        stride = max(o["n"] for o in outs)
        recs = torch.cat([o["records"][:stride] if o["records"].shape[0] >= stride else
                          torch.cat([o["records"], o["records"].new_zeros((stride - o["records"].shape[0], 48))])
                          for o in outs])
        offs = torch.cat([o["wp_offsets"] for o in outs])
        key = torch.stack([o["wp_key"] for o in outs]).min(0).values
        mg = ctxs[0].merge_active_sets(world, q.shape[0] * q.shape[1], recs, stride, offs, key, r1["capacity"])
        torch.cuda.synchronize()
        assert int(mg["count"].item()) == r1["n"]
        mg["n"] = r1["n"]
        b = records_np(mg)
        for k in ("wp", "pt", "value", "grad"):
            assert np.array_equal(a[k], b[k]), (world, k)
        assert torch.equal(mg["wp_offsets"], r1["wp_offsets"])
        assert torch.equal(mg["wp_min"], r1["wp_min"]) and torch.equal(mg["wp_argmin"], r1["wp_argmin"])


@pytest.mark.parametrize("prec", [0, 2])
def test_detect_host_buffers_match_device_call(c2, prec):
    """The end-to-end host-buffer call (q and results in host memory, copies inside the
    library) returns exactly what the device call returns, on fp32 and fp16 contexts;
    a too-small host capacity reports CAPACITY with the exact count."""
    from paper_2601_18548_b200 import GcdfError
    cfg, pts, q, m, full = c2
    tau = synth.load_tau(cfg.name)
    ctx = _ctx(cfg, precision=prec)
    ctx.update_scene(pts)
    qt = torch.from_numpy(q)
    dev = ctx.detect_active_set(qt, DELTA, tau)
    n = int(dev["n"])
    assert n > 0
    for pinned in (True, False):
        ho = ctx.alloc_host_outputs(q.shape[0] * q.shape[1], n + 5, pinned=pinned)
        h = ctx.detect_active_set_host(qt, DELTA, tau, ho)
        assert h["n"] == n
        assert torch.equal(h["records"][:n], dev["records"][:n].cpu())
        for k in ("wp_offsets", "wp_min", "wp_argmin"):
            assert torch.equal(h[k], dev[k].cpu()), k
    small = ctx.alloc_host_outputs(q.shape[0] * q.shape[1], max(n // 2, 1), pinned=True)
    with pytest.raises(GcdfError):
        ctx.detect_active_set_host(qt, DELTA, tau, small)

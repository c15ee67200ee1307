"""GPU parity of the tcgen05 tensor-core path (GCDF_FP16 default, GCDF_BF16) vs the oracle.

Gates (R17, R28), at the paper's gradient scale (R11: median ||grad_q f|| ~ 1):
  (1) same rounding points: vs the oracle's EMU mode for the operand type (fp16 / bf16
      rounding of exactly the MMA operands) the median value error is fp32 noise (<= 1e-6)
      and the p99 small (the tail differs only where fp32 accumulation order moves a value
      across a 16-bit rounding boundary or a ReLU kink);
  (2) vs the exact oracle, values on every pair: |df| <= 2e-2 (north star);
  (3a) vs the exact oracle, | ||g_gpu|| - ||g_exact|| | <= 5e-2 (north star) on every pair
      whose exact ReLU masks equal the emulated ones (kink-free under 16-bit operands);
  (3b) on all pairs, the fraction within 5e-2 is >= min(0.99, f_emu - 0.005), f_emu = the
      same fraction of the EMU oracle alone (no GPU involved): a ReLU mask flipped by 16-bit
      operand rounding moves the gradient by ~10 % of its norm, so at unit gradient scale
      the operand type itself leaves ~2 % (fp16) / ~18 % (bf16) of pairs outside 5e-2
      (R28, EMU-only numbers in DESIGN.md).
Where the operand type alone exceeds (2) (bf16 at this scale: EMU-only max |df| ~ 8e-2),
the GPU is held to the EMU's own error + 5e-3 and the shortfall is reported; the bf16
contract (2e-2 / 5e-2) is met by the fp16 default on every gate; the fp32-accurate split path is
GCDF_FP16X3 (tests/test_gpu_fp16x3.py).
"""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import BF16_GNORM_ATOL, BF16_VAL_ATOL, DELTA, compare_active_sets, oracle_detect, oracle_mlp, records_np

pytestmark = pytest.mark.gpu
NT = max(1, min(os.cpu_count() or 1, 64))
KINK_EMU = 1e-3
PRECS = {"fp16": (2, oracle.EMU_FP16), "bf16": (1, oracle.EMU_BF16)}


def _ctx(cfg, prec, **kw):
    from paper_2601_18548_b200 import Context
    ctx = Context(0, precision=PRECS[prec][0], scene_capacity=cfg.M + 4096, max_waypoints=cfg.B * cfg.N,
                  max_active=min(cfg.pairs, 1 << 22), **kw)
    ctx.load_weights(synth.weights_path(cfg.H))
    return ctx


def _round(x, prec):
    return x.to(torch.float16 if prec == "fp16" else torch.bfloat16).to(torch.float64)


@pytest.mark.parametrize("prec", ["fp16", "bf16"])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_selftest_umma(mode, prec):
    """One UMMA block: K-major B (forward), MN-major B (backward), N = 16 (last GEMM)."""
    from paper_2601_18548_b200.gcdf import selftest_umma
    g = torch.Generator().manual_seed(mode)
    A = torch.randn(128, 128, generator=g)
    B = torch.randn(16 if mode == 2 else 128, 128, generator=g)
    D = selftest_umma(mode | (4 if prec == "fp16" else 0), A.cuda(), B.cuda()).cpu().double()
    ref = _round(A, prec) @ (_round(B, prec) if mode == 1 else _round(B, prec).T)
    n = ref.shape[1]
    err = (D[:, :n] - ref).abs().max().item()
    assert err <= 1e-4 * max(1.0, ref.abs().max().item()), err


def stats_and_gates(v, g, exact, emu, prec, what="", agree_min=0.85, kink_emu=KINK_EMU):
    dv = np.abs(v - emu["f"])
    de = np.abs(v - exact["f"])
    gn_exact = np.linalg.norm(exact["g"], axis=-1)
    gd = np.abs(np.linalg.norm(g, axis=-1) - gn_exact)
    dg_emu = np.linalg.norm(g - emu["g"], axis=-1) / np.maximum(1.0, np.linalg.norm(emu["g"], axis=-1))
    # kink-free (R17): the exact ReLU masks equal the emulated ones, no emulated pre-activation
    # within kink_emu of zero, and the GPU took the emulation's branches (its gradient agrees
    # with the emulation's to 1e-2 max(1, ||g||); a flip moves it by ~10 %).  The last clause
    # drops the pairs where fp32 accumulation order moved a 16-bit rounding boundary upstream
    # of a kink (<= 1 % by gate 1; counted as "gpu_branch_differs")
    same_branch = dg_emu <= 1e-2
    kink_free = (exact["mask_hash"] == emu["mask_hash"]) & (emu["kappa"] > kink_emu) & same_branch
    # the operand type's own error (EMU oracle vs exact oracle, no GPU involved)
    emu_de = np.abs(emu["f"] - exact["f"])
    emu_gd = np.abs(np.linalg.norm(emu["g"], axis=-1) - gn_exact)
    st = {"emu_val_agree_1e-5": float(np.mean(dv <= 1e-5)), "emu_val_max": float(dv.max()),
          "emu_val_p50": float(np.median(dv)), "emu_val_p99": float(np.percentile(dv, 99)),
          "emu_grad_agree_1e-4": float(np.mean(dg_emu <= 1e-4)), "emu_grad_p99": float(np.percentile(dg_emu, 99)),
          "exact_val_max": float(de.max()), "exact_val_p99": float(np.percentile(de, 99)),
          "gnorm_within_5e-2": float(np.mean(gd <= BF16_GNORM_ATOL)), "gnorm_p99": float(np.percentile(gd, 99)),
          "gnorm_max_kink_free": float(gd[kink_free].max()) if kink_free.any() else 0.0,
          "kink_free_frac": float(kink_free.mean()), "gnorm_median_exact": float(np.median(gn_exact)),
          "gpu_branch_differs": float(1.0 - same_branch.mean()),
          "type_only_val_max": float(emu_de.max()), "type_only_gnorm_within_5e-2": float(np.mean(emu_gd <= BF16_GNORM_ATOL))}
    print(f"\n[{prec}] {what}: {st}", flush=True)
    # gate 1: the bulk agrees with the emulation to fp32-accumulation noise; the tail is
    # 16-bit rounding-boundary / ReLU-kink flips (8x more frequent but 8x smaller for fp16)
    assert st["emu_val_p50"] <= 1e-6, st
    assert st["emu_val_agree_1e-5"] >= agree_min, st
    # fp16: fixed bounds; bf16 (R28): the GPU may differ from the emulation by no more than the
    # operand type itself differs from the exact network (layer 1 runs on split bf16 operands,
    # ~16-bit effective precision, not the EMU model's exact layer 1, which moves more kinks)
    if prec == "fp16":
        assert st["emu_val_max"] <= 1e-2, st
        assert st["emu_grad_p99"] <= 1e-2, st
    else:
        type_grad_p99 = float(np.percentile(np.linalg.norm(emu["g"] - exact["g"], axis=-1)
                                            / np.maximum(1.0, gn_exact), 99))
        st["type_only_grad_p99"] = type_grad_p99
        assert st["emu_val_max"] <= st["type_only_val_max"], st
        assert st["emu_grad_p99"] <= type_grad_p99, st
    assert st["gpu_branch_differs"] <= (0.01 if prec == "fp16" else 0.05), st
    # gate 2: the north-star value tolerance where the operand type can meet it (fp16);
    # otherwise (bf16) the type's own error + 5e-3 (R28)
    if st["type_only_val_max"] <= BF16_VAL_ATOL:
        assert st["exact_val_max"] <= BF16_VAL_ATOL, st
    else:
        assert st["exact_val_max"] <= st["type_only_val_max"] + 5e-3, st
    # gate 3a / 3b (R17, R28)
    # 3a per kink-free pair: 5e-2, or -- where the operand type's own deviation on that pair
    # already exceeds it (SE(2): d f / d theta scales with the point's distance, up to 14 m) --
    # that deviation + 1e-2 max(1, ||g||)
    lim = np.maximum(BF16_GNORM_ATOL, emu_gd + 1e-2 * np.maximum(1.0, gn_exact))
    bad = kink_free & (gd > lim)
    assert not bad.any(), (int(bad.sum()), st)
    assert st["gnorm_within_5e-2"] >= min(0.99, st["type_only_gnorm_within_5e-2"] - 0.005), st
    return st


@pytest.fixture(scope="module")
def c2():
    cfg = synth.get_config("C2")
    pts, _ = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg)[:, :12]
    m = oracle_mlp(cfg)
    Q = q.reshape(-1, 9)
    exact = m.eval(pts, Q, want_kappa=True, want_hash=True, nthreads=NT)
    emu = {p: m.eval(pts, Q, flags=PRECS[p][1], want_kappa=True, want_hash=True, nthreads=NT) for p in PRECS}
    return cfg, pts, q, m, exact, emu


@pytest.mark.parametrize("prec", ["fp16", "bf16"])
def test_query_dense(c2, prec):
    cfg, pts, q, m, exact, emu = c2
    ctx = _ctx(cfg, prec)
    ctx.update_scene(pts)
    v, g = ctx.query_values_grads(torch.from_numpy(q))
    torch.cuda.synchronize()
    M = len(pts)
    vn, gnp = v.cpu().numpy(), g.cpu().numpy()
    stats_and_gates(vn[:, :M], gnp[:, :M], exact, emu[prec], prec, "C2 dense (120k pairs)")
    assert np.all(np.isinf(vn[:, M:])) and np.all(gnp[:, M:] == 0)


@pytest.mark.parametrize("prec", ["fp16", "bf16"])
def test_detect(c2, prec):
    cfg, pts, q, m, exact, emu = c2
    tau = synth.load_tau(cfg.name)
    ctx = _ctx(cfg, prec)
    ids = ctx.update_scene(pts)
    out = ctx.detect_active_set(torch.from_numpy(q), DELTA, tau)
    torch.cuda.synchronize()
    gpu = records_np(out)
    Q = q.reshape(-1, 9)
    # bf16 at the paper's scale: the operand type's own value error (EMU oracle, no GPU)
    # exceeds the north-star 2e-2, so its band and value tolerance are that error + 5e-3 (R28)
    tol = BF16_VAL_ATOL if prec == "fp16" else float(np.abs(emu[prec]["f"] - exact["f"]).max()) + 5e-3
    orc = oracle_detect(m, pts, ids, Q, tau, nthreads=NT)
    nd, nc = compare_active_sets(gpu, orc, exact["f"], ids, 1e-3 + tol, val_atol=tol, what="vs exact")
    assert nc > 0
    assert np.all(np.abs(out["wp_min"].cpu().numpy() - orc["wp_min"]) <= tol)
    print(f"\n[{prec}] detect C2: {out['n']} active, oracle {orc['count']}, {nd} differ (all within the band)")


@pytest.mark.parametrize("prec", ["fp16", "bf16"])
def test_fused_equals_dense_plus_compact(c2, prec):
    cfg, pts, q, m, exact, emu = c2
    tau = synth.load_tau(cfg.name)
    ctx = _ctx(cfg, prec)
    ctx.update_scene(pts)
    qt = torch.from_numpy(q)
    v, g = ctx.query_values_grads(qt)
    a = records_np(ctx.compact_dense(v, g, DELTA, tau))
    b = records_np(ctx.detect_active_set(qt, DELTA, tau))
    for k in ("wp", "pt", "value", "grad"):
        assert np.array_equal(a[k], b[k]), k


def test_qchannel_mode_fp16(c2):
    """TGRAD_QCHANNEL: the translational gradient is the network's q^t input channel (R3)."""
    from paper_2601_18548_b200 import TGRAD_QCHANNEL
    cfg, pts, q, m, exact, emu = c2
    ctx = _ctx(cfg, "fp16", tgrad_mode=TGRAD_QCHANNEL)
    ctx.update_scene(pts[:2000])
    v, g = ctx.query_values_grads(torch.from_numpy(q[:, :2]))
    ex = m.eval(pts[:2000], q[:, :2].reshape(-1, 9), flags=oracle.TGRAD_QCHANNEL)
    em = m.eval(pts[:2000], q[:, :2].reshape(-1, 9), flags=oracle.TGRAD_QCHANNEL | oracle.EMU_FP16)
    gn = g.cpu().numpy()[:, :2000]
    ne = np.linalg.norm(ex["g"], axis=-1)
    d = np.abs(np.linalg.norm(gn, axis=-1) - ne)
    d_type = np.abs(np.linalg.norm(em["g"], axis=-1) - ne)  # the operand type alone (R28)
    assert np.mean(d <= BF16_GNORM_ATOL) >= min(0.99, np.mean(d_type <= BF16_GNORM_ATOL) - 0.005)
    assert np.abs(v.cpu().numpy()[:, :2000] - ex["f"]).max() <= BF16_VAL_ATOL


def test_c5_full_size_sampled():
    """The bench configuration (C5: 256 waypoints x 1M points, fp16, full-size detect):
    sampled pairs against the oracle one by one, plus the per-waypoint min property."""
    cfg = synth.get_config("C5")
    pts, _ = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg)
    tau = synth.load_tau(cfg.name)
    ctx = _ctx(cfg, "fp16")
    ids = ctx.update_scene(pts)
    out = ctx.detect_active_set(torch.from_numpy(q), DELTA, tau)
    torch.cuda.synchronize()
    gpu = records_np(out)
    rng = np.random.default_rng(2024)
    m = oracle_mlp(cfg)
    Q = q.reshape(-1, 9)
    wsel = np.sort(rng.choice(Q.shape[0], 3, replace=False))
    psel = np.sort(rng.choice(len(pts), 4096, replace=False))
    ex = m.eval(pts[psel], Q[wsel], want_kappa=True, want_hash=True, nthreads=NT)
    em = m.eval(pts[psel], Q[wsel], flags=oracle.EMU_FP16, want_kappa=True, want_hash=True, nthreads=NT)
    v, g = ctx.query_values_grads(torch.from_numpy(Q[wsel].reshape(1, -1, 9)))
    stats_and_gates(v.cpu().numpy()[:, psel], g.cpu().numpy()[:, psel], ex, em, "fp16", "C5 sampled")
    recset = set(zip(gpu["wp"].tolist(), gpu["pt"].tolist()))
    thr = tau + DELTA
    checked = 0
    for wi, w in enumerate(wsel):
        for pj, pid in enumerate(psel):
            f = ex["f"][wi, pj]
            if abs(f - thr) > 1e-3 + BF16_VAL_ATOL:
                assert ((int(w), int(ids[pid])) in recset) == (f <= thr), (w, pid, f)
                checked += 1
    assert checked > 0.9 * len(wsel) * len(psel)
    wmin = out["wp_min"].cpu().numpy()[wsel]
    assert np.all(wmin <= ex["f"].min(axis=1) + BF16_VAL_ATOL)
    offs = out["wp_offsets"].cpu().numpy()
    assert offs[-1] == out["n"] and np.all(np.diff(offs) >= 0)
    frac = out["n"] / (len(pts) * Q.shape[0])
    assert 0.001 < frac < 0.05
    print(f"\nC5: {out['n']} active ({frac:.4%}), {checked} sampled memberships checked")


def test_c4_batched_replanning_with_updates():
    """C4 (128 trajectories x 64 waypoints x 20k points, fp16) after 3 rounds of the scene
    dynamics (200 removes + 200 adds on a moved box): ids equal the oracle's replay of the id
    rule; sampled pairs and the per-waypoint minimum match the oracle on the replayed scene."""
    cfg = synth.get_config("C4")
    pts, boxes = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg)
    tau = synth.load_tau(cfg.name)
    ctx = _ctx(cfg, "fp16")
    osc = oracle.Scene(cfg.M + 4096)
    assert np.array_equal(ctx.update_scene(pts), osc.update(pts))
    rng = np.random.default_rng(404)
    for _ in range(3):
        live, _ = osc.export()
        add, rem = synth.scene_update_batch(rng, boxes, live)
        assert np.array_equal(ctx.update_scene(add, rem), osc.update(add, rem))
    ids, xyz = osc.export()
    out = ctx.detect_active_set(torch.from_numpy(q), DELTA, tau)
    torch.cuda.synchronize()
    gpu = records_np(out)
    Q = q.reshape(-1, 9)
    m = oracle_mlp(cfg)
    wsel = np.sort(rng.choice(Q.shape[0], 4, replace=False))
    psel = np.sort(rng.choice(len(ids), 2048, replace=False))
    ex = m.eval(xyz[psel], Q[wsel], want_grad=False)
    recset = set(zip(gpu["wp"].tolist(), gpu["pt"].tolist()))
    thr = tau + DELTA
    for wi, w in enumerate(wsel):
        for pj, pi in enumerate(psel):
            f = ex["f"][wi, pj]
            if abs(f - thr) > 1e-3 + BF16_VAL_ATOL:
                assert ((int(w), int(ids[pi])) in recset) == (f <= thr)
    # exact per-waypoint minimum on the sampled waypoints, over the whole replayed scene
    full = m.eval(xyz, Q[wsel], want_grad=False, nthreads=NT)["f"]
    wmin = out["wp_min"].cpu().numpy()[wsel]
    assert np.all(np.abs(wmin - full.min(axis=1)) <= BF16_VAL_ATOL)
    # values of the records of the sampled waypoints vs the oracle
    pos = {int(i): j for j, i in enumerate(ids)}
    sel = np.isin(gpu["wp"], wsel)
    wrow = {int(w): k for k, w in enumerate(wsel)}
    fo = np.array([full[wrow[int(w)], pos[int(p)]] for w, p in zip(gpu["wp"][sel], gpu["pt"][sel])])
    assert len(fo) > 0 and np.all(np.abs(gpu["value"][sel] - fo) <= BF16_VAL_ATOL)


def test_c3_dense_scene_full_rows():
    """C3 (100 waypoints x 100k points of the dense 120-box scene, fp16): for 4 sampled
    waypoints, the whole row against the oracle (values of every pair, exact active-set
    membership outside the tolerance band, per-waypoint min / argmin), plus the record
    order and offsets invariants of the full result."""
    cfg = synth.get_config("C3")
    pts, _ = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg)
    tau = synth.load_tau(cfg.name)
    ctx = _ctx(cfg, "fp16")
    ids = ctx.update_scene(pts)
    out = ctx.detect_active_set(torch.from_numpy(q), DELTA, tau)
    torch.cuda.synchronize()
    gpu = records_np(out)
    n = int(out["n"])
    key = gpu["wp"].astype(np.int64) * (1 << 32) + gpu["pt"].astype(np.int64)
    assert np.all(np.diff(key) > 0), "records not in strict (wp, pt) order"
    offs = out["wp_offsets"].cpu().numpy()
    assert offs[0] == 0 and offs[-1] == n and np.all(np.diff(offs) >= 0)
    assert np.array_equal(np.repeat(np.arange(len(offs) - 1), np.diff(offs)), gpu["wp"])
    Q = q.reshape(-1, 9)
    rng = np.random.default_rng(303)
    wsel = np.sort(rng.choice(Q.shape[0], 4, replace=False))
    m = oracle_mlp(cfg)
    full = m.eval(pts, Q[wsel], want_grad=False, nthreads=NT)["f"]
    v, _ = ctx.query_values_grads(torch.from_numpy(Q[wsel].reshape(1, -1, 9)), want_grads=False)
    v = v.cpu().numpy()[:, ids]
    assert np.abs(v - full).max() <= BF16_VAL_ATOL
    thr = tau + DELTA
    wmin = out["wp_min"].cpu().numpy()[wsel]
    warg = out["wp_argmin"].cpu().numpy()[wsel]
    assert np.all(np.abs(wmin - full.min(axis=1)) <= BF16_VAL_ATOL)
    for k, w in enumerate(wsel):
        rec = set(gpu["pt"][offs[w]:offs[w + 1]].tolist())
        orc = set(ids[full[k] <= thr].tolist())
        band = set(ids[np.abs(full[k] - thr) <= 1e-3 + BF16_VAL_ATOL].tolist())
        assert (rec ^ orc) <= band, (w, len(rec ^ orc), len(band))
        assert int(warg[k]) in set(ids[full[k] <= full[k].min() + 2 * BF16_VAL_ATOL].tolist())
    frac = n / (len(pts) * Q.shape[0])
    print(f"\nC3: {n} active ({frac:.4%})")


@pytest.mark.parametrize("n_wp,n_pts", [(1, 100), (1, 128), (1, 300), (2, 200), (3, 129), (4, 257), (5, 700),
                                        (7, 1000)])
def test_tile_count_edge_cases(c2, n_wp, n_pts):
    """Tile counts below / around the three tiles a CTA keeps in flight (K2b): one tile, a
    ragged last tile, CTAs whose second / third slot has no tile (passed turns), and the
    last-round tail.  Dense values and gradients vs the EMU oracle (same rounding points),
    and the fused detect bit-identical to dense query + standalone compaction."""
    cfg, pts, q, m, exact, emu = c2
    P = pts[:n_pts]
    qq = q[:, :n_wp]
    ctx = _ctx(cfg, "fp16")
    ctx.update_scene(P)
    qt = torch.from_numpy(qq)
    v, g = ctx.query_values_grads(qt)
    torch.cuda.synchronize()
    vn, gn = v.cpu().numpy()[:, :n_pts], g.cpu().numpy()[:, :n_pts]
    em = m.eval(P, qq.reshape(-1, 9), flags=oracle.EMU_FP16)
    # gate 1 of stats_and_gates (fp16): fp32-noise median, rounding-boundary / kink flips in the tail
    dv = np.abs(vn - em["f"])
    assert np.median(dv) <= 1e-6 and dv.max() <= 1e-2, (np.median(dv), dv.max())
    dg = np.linalg.norm(gn - em["g"], axis=-1) / np.maximum(1.0, np.linalg.norm(em["g"], axis=-1))
    assert np.percentile(dg, 99) <= 1e-2, np.percentile(dg, 99)
    assert np.all(np.isinf(v.cpu().numpy()[:, n_pts:]))
    # threshold at the sample's own median so that every case has actives and inactives
    tau = float(np.median(em["f"])) - DELTA
    a = records_np(ctx.compact_dense(v, g, DELTA, tau))
    b = records_np(ctx.detect_active_set(qt, DELTA, tau))
    assert len(b["wp"]) > 0
    for k in ("wp", "pt", "value", "grad"):
        assert np.array_equal(a[k], b[k]), k


def test_staging_overflow_reports_capacity(c2):
    """More actives than the staging capacity (max_active): the tiles that no longer fit are
    dropped by the detect warp's allocation, the call reports CAPACITY, and a retry with a
    context of sufficient capacity returns the full canonical set."""
    from paper_2601_18548_b200 import Context, GcdfError
    cfg, pts, q, m, exact, emu = c2
    qt = torch.from_numpy(q[:, :4])
    tau = float(np.median(emu["fp16"]["f"])) - DELTA  # ~half of the pairs active
    small = Context(0, precision=2, scene_capacity=cfg.M + 4096, max_waypoints=64, max_active=1024)
    small.load_weights(synth.weights_path(cfg.H))
    small.update_scene(pts)
    with pytest.raises(GcdfError) as e:
        small.detect_active_set(qt, DELTA, tau, capacity=1024)
    assert e.value.name == "CAPACITY"
    big = _ctx(cfg, "fp16")
    big.update_scene(pts)
    full = records_np(big.detect_active_set(qt, DELTA, tau))
    assert len(full["wp"]) > 1024
    assert np.all(np.diff(full["wp"].astype(np.int64) * (1 << 32) + full["pt"]) > 0)  # canonical order

"""Pins of the float64 oracle against things other than itself.

Each test names what fixes the expected value: a hand-worked example, a closed form,
an invariant implied by the paper's construction, finite differences, brute force,
or an independent second differentiation (torch autograd).  CPU only.
"""
import json
import struct
from pathlib import Path

import numpy as np
import pytest

import oracle
import synth

GOLD = Path(__file__).resolve().parent / "golden"
DELTA = 0.10


def _write(tmp_path, name, act, dims, layers):
    p = tmp_path / name
    synth.write_mlpw(p, act, dims, layers)
    return p


def _rand_inputs(rng, M, W, dyadic=False):
    pts = np.stack([rng.uniform(-7, 7, M), rng.uniform(-7, 7, M), rng.uniform(0, 2, M)], 1)
    q = np.concatenate([rng.uniform(-5, 5, (W, 2)), rng.uniform(-np.pi, np.pi, (W, 7))], 1)
    if dyadic:
        pts = np.round(pts * 1024) / 1024
        q = np.round(q * 1024) / 1024
    return pts, q


@pytest.fixture(scope="module")
def mlp32(tmp_path_factory):
    act, dims, layers = synth.make_weights(32, seed=11)
    p = tmp_path_factory.mktemp("w") / "h32.mlpw"
    synth.write_mlpw(p, act, dims, layers)
    return oracle.MLP(p), (act, dims, layers)


# ------------------------------------------------------------------ O1: weights file
def test_mlpw_errors(tmp_path):
    act, dims, layers = synth.make_weights(32, seed=1)
    good = _write(tmp_path, "g.mlpw", act, dims, layers)
    m = oracle.MLP(good)
    assert m.dims == [12] + [32] * 6 + [1] and m.L == 7 and m.act == 1
    raw = good.read_bytes()
    cases = {
        "bad_magic": (b"MLPX" + raw[4:], "BAD_MAGIC"),
        "version": (raw[:4] + struct.pack("<I", 2) + raw[8:], "VERSION"),
        "truncated": (raw[:-8], "IO"),
        "trailing": (raw + b"\0" * 8, "DIM_MISMATCH"),
    }
    for name, (blob, err) in cases.items():
        p = tmp_path / (name + ".mlpw")
        p.write_bytes(blob)
        with pytest.raises(oracle.OracleError) as ei:
            oracle.MLP(p)
        assert ei.value.name == err, name
    # input width must be 3 + n = 12
    bad_dims = [13] + [32] * 6 + [1]
    rng = np.random.default_rng(0)
    bl = [(rng.normal(size=(bad_dims[i + 1], bad_dims[i])), np.zeros(bad_dims[i + 1])) for i in range(7)]
    with pytest.raises(oracle.OracleError) as ei:
        oracle.MLP(_write(tmp_path, "d.mlpw", 1, bad_dims, bl))
    assert ei.value.name == "DIM_MISMATCH"


# ------------------------------------------------------------------ hand-worked golden example
def test_hand_worked_example(tmp_path):
    g = json.loads((GOLD / "hand_example.json").read_text())
    for ni, net in enumerate(g["networks"]):
        layers = [(np.array(l["W"], float), np.array(l["b"], float)) for l in net["layers"]]
        dims = [12] + [1] * 6 + [1]
        m = oracle.MLP(_write(tmp_path, "hand%d.mlpw" % ni, 1, dims, layers))
        for case in net["cases"]:
            out = m.eval(np.array([case["p"]]), np.array([case["q"]]))
            assert abs(out["f"][0, 0] - case["f"]) <= 1e-12
            np.testing.assert_allclose(out["g"][0, 0], case["grad"], rtol=0, atol=1e-12)


# ------------------------------------------------------------------ closed forms
def test_identity_activation_closed_form(tmp_path):
    """Identity activation: f = (W7...W1) x_in + b_eff; grad = mapped rows of the product."""
    rng = np.random.default_rng(5)
    dims = [12, 9, 7, 8, 6, 5, 4, 1]
    layers = [(rng.normal(size=(dims[i + 1], dims[i])), rng.normal(size=dims[i + 1])) for i in range(7)]
    m = oracle.MLP(_write(tmp_path, "id.mlpw", 0, dims, layers))
    A = np.eye(12)
    c = np.zeros(12)
    for W, b in layers:  # affine composition x -> W (A x + c) + b
        A, c = W @ A, W @ c + b
    pts, q = _rand_inputs(rng, 13, 5)
    out = m.eval(pts, q)
    out_qc = m.eval(pts, q, flags=oracle.TGRAD_QCHANNEL)
    for w in range(q.shape[0]):
        for j in range(pts.shape[0]):
            x = np.concatenate([[pts[j, 0] - q[w, 0], pts[j, 1] - q[w, 1], pts[j, 2], 0, 0], q[w, 2:]])
            f = (A @ x + c)[0]
            assert abs(out["f"][w, j] - f) <= 1e-10 * max(1, abs(f))
            row = A[0]
            want = np.concatenate([[-row[0], -row[1]], row[5:]])
            np.testing.assert_allclose(out["g"][w, j], want, rtol=1e-11, atol=1e-11)
            want_qc = np.concatenate([[row[3], row[4]], row[5:]])
            np.testing.assert_allclose(out_qc["g"][w, j], want_qc, rtol=1e-11, atol=1e-11)


def test_zero_head_constant(tmp_path):
    """Zero output layer -> f == b7 and grad == 0 for every input."""
    act, dims, layers = synth.make_weights(32, seed=2)
    layers[-1] = (np.zeros_like(layers[-1][0]), np.array([0.731]))
    m = oracle.MLP(_write(tmp_path, "z.mlpw", act, dims, layers))
    pts, q = _rand_inputs(np.random.default_rng(1), 20, 4)
    out = m.eval(pts, q)
    assert np.all(out["f"] == 0.731)
    assert np.all(out["g"] == 0.0)


# ------------------------------------------------------------------ second implementation
def test_torch_autograd_float64(mlp32):
    """Independent differentiation: torch float64 autograd of the same network."""
    torch = pytest.importorskip("torch")
    m, (act, dims, layers) = mlp32
    rng = np.random.default_rng(9)
    pts, q = _rand_inputs(rng, 64, 6)
    out = m.eval(pts, q, want_kappa=True)
    Ws = [(torch.tensor(W), torch.tensor(b)) for W, b in layers]
    P = torch.tensor(pts)
    for w in range(q.shape[0]):
        qt = torch.tensor(q[w]).repeat(P.shape[0], 1).requires_grad_(True)
        pq = torch.cat([P[:, :2] - qt[:, :2], P[:, 2:3], torch.zeros(P.shape[0], 2, dtype=torch.float64),
                        qt[:, 2:]], 1)
        h = pq
        for li, (W, b) in enumerate(Ws):
            h = h @ W.T + b
            if li < len(Ws) - 1:
                h = torch.relu(h)
        f = h[:, 0]
        (gq,) = torch.autograd.grad(f.sum(), qt)
        np.testing.assert_allclose(out["f"][w], f.detach().numpy(), rtol=1e-12, atol=1e-12)
        ok = out["kappa"][w] > 1e-9
        np.testing.assert_allclose(out["g"][w][ok], gq.numpy()[ok], rtol=1e-10, atol=1e-12)


# ------------------------------------------------------------------ finite differences
def test_central_fd_all_components(mlp32):
    """P3: central FD of the oracle's own forward, all 9 q components, rel <= 1e-6."""
    m, _ = mlp32
    rng = np.random.default_rng(3)
    pts, q = _rand_inputs(rng, 40, 5)
    base = m.eval(pts, q, want_hash=True)
    checked = skipped = 0
    for k in range(9):
        h = 1e-6 * np.maximum(1.0, np.abs(q[:, k]))
        qp, qm = q.copy(), q.copy()
        qp[:, k] += h
        qm[:, k] -= h
        op = m.eval(pts, qp, want_grad=False, want_hash=True)
        om = m.eval(pts, qm, want_grad=False, want_hash=True)
        fd = (op["f"] - om["f"]) / (2 * h[:, None])
        same = (op["mask_hash"] == base["mask_hash"]) & (om["mask_hash"] == base["mask_hash"])
        g = base["g"][:, :, k]
        err = np.abs(fd - g) / np.maximum(1.0, np.abs(g))
        assert np.all(err[same] <= 1e-6), (k, err[same].max())
        checked += same.sum()
        skipped += (~same).sum()
    assert skipped <= 0.01 * (checked + skipped)


def test_chain_rule_translation_equals_minus_point_gradient(mlp32):
    """dF/dq_x = -dF/dp_x (FD on p)."""
    m, _ = mlp32
    rng = np.random.default_rng(4)
    pts, q = _rand_inputs(rng, 30, 3)
    base = m.eval(pts, q, want_hash=True)
    for ax in (0, 1):
        h = 1e-6 * np.maximum(1.0, np.abs(pts[:, ax]))
        pp, pm = pts.copy(), pts.copy()
        pp[:, ax] += h
        pm[:, ax] -= h
        op = m.eval(pp, q, want_grad=False, want_hash=True)
        om = m.eval(pm, q, want_grad=False, want_hash=True)
        fd_p = (op["f"] - om["f"]) / (2 * h[None, :])
        same = (op["mask_hash"] == base["mask_hash"]) & (om["mask_hash"] == base["mask_hash"])
        g = base["g"][:, :, ax]
        assert np.all(np.abs(-fd_p - g)[same] <= 1e-6 * np.maximum(1, np.abs(g[same])))


# ------------------------------------------------------------------ invariants
def test_base_translation_invariance_bitexact(mlp32):
    """P1: moving the base and the point rigidly together leaves value and gradient
    unchanged (BASELINE north_star).  Dyadic inputs make the f64
    subtraction exact, so the result is bit-identical."""
    m, _ = mlp32
    rng = np.random.default_rng(6)
    pts, q = _rand_inputs(rng, 50, 4, dyadic=True)
    a = m.eval(pts, q)
    for t in ([3.5, -2.25], [-6.0009765625, 0.5]):
        p2, q2 = pts.copy(), q.copy()
        p2[:, :2] += t
        q2[:, :2] += t
        b = m.eval(p2, q2)
        assert np.array_equal(a["f"], b["f"]) and np.array_equal(a["g"], b["g"])
    # general inputs: <= 1e-12 relative
    pts, q = _rand_inputs(rng, 50, 4)
    a = m.eval(pts, q)
    t = np.array([1.2345, -0.987])
    p2, q2 = pts.copy(), q.copy()
    p2[:, :2] += t
    q2[:, :2] += t
    b = m.eval(p2, q2, want_kappa=True)
    np.testing.assert_allclose(a["f"], b["f"], rtol=1e-12, atol=1e-12)
    ok = b["kappa"] > 1e-9
    np.testing.assert_allclose(a["g"][ok], b["g"][ok], rtol=1e-9, atol=1e-12)


def test_point_above_base_and_batch_consistency(mlp32):
    """P1b: p_xy = q_xy gives the same value as the point at the origin with the base at
    the origin.  P2(iv): a batch row equals the single-pair evaluation bit for bit."""
    m, _ = mlp32
    rng = np.random.default_rng(7)
    pts, q = _rand_inputs(rng, 17, 3)
    for w in range(3):
        p = np.array([[q[w, 0], q[w, 1], 0.7]])
        q0 = q[w].copy()
        q0[:2] = 0.0
        a = m.eval(p, q[w:w + 1])
        b = m.eval(np.array([[0.0, 0.0, 0.7]]), q0[None])
        assert a["f"][0, 0] == b["f"][0, 0]
        np.testing.assert_array_equal(a["g"], b["g"])
    full = m.eval(pts, q)
    for w in range(3):
        for j in (0, 5, 16):
            one = m.eval(pts[j:j + 1], q[w:w + 1])
            assert one["f"][0, 0] == full["f"][w, j]
            np.testing.assert_array_equal(one["g"][0, 0], full["g"][w, j])
    multi = m.eval(pts, q, nthreads=3)
    np.testing.assert_array_equal(multi["f"], full["f"])
    np.testing.assert_array_equal(multi["g"], full["g"])


# ------------------------------------------------------------------ brute-force active set
def test_detect_bruteforce_C1(tmp_path):
    """P4: enumerate all pairs, filter, sort by (wp, pt), min per waypoint (smallest id on
    ties), compare with the oracle's loop-order output exactly."""
    cfg = synth.get_config("C1")
    pts, _ = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg).reshape(-1, 9)
    m = oracle.MLP(synth.weights_path(cfg.H))
    # a scene with holes: ids are not 0..M-1
    ids = np.arange(pts.shape[0], dtype=np.int64) * 3 + 1
    # exact ties: duplicate each waypoint's nearest point under the next id, so the
    # argmin must pick the smaller id and both copies appear in order
    pre = m.eval(pts, q, want_grad=False)["f"]
    dup = np.unique(np.argmin(pre, axis=1))
    order = np.argsort(np.concatenate([ids, ids[dup] + 1]), kind="stable")
    pts = np.concatenate([pts, pts[dup]])[order]
    ids = np.concatenate([ids, ids[dup] + 1])[order]
    tau = synth.load_tau("C1")
    d = m.detect(pts, ids, q, DELTA, tau)
    full = m.eval(pts, q)
    F = full["f"]
    pairs = sorted((w, int(ids[j])) for w in range(q.shape[0]) for j in range(len(ids))
                   if F[w, j] - DELTA <= tau)
    assert d["count"] == len(pairs)
    assert [(int(a), int(b)) for a, b in zip(d["wp"], d["pt"])] == pairs
    pos = {int(i): j for j, i in enumerate(ids)}
    for k, (w, pt) in enumerate(pairs):
        assert d["value"][k] == F[w, pos[pt]]
        np.testing.assert_array_equal(d["grad"][k], full["g"][w, pos[pt]])
    for w in range(q.shape[0]):
        best = min(range(len(ids)), key=lambda j: (F[w, j], ids[j]))
        assert d["wp_min"][w] == F[w, best] and d["wp_argmin"][w] == ids[best]
        assert d["wp_offsets"][w] == sum(1 for a, _ in pairs if a < w)
    assert d["wp_offsets"][-1] == len(pairs)
    # sparsity sits near the calibrated 5% target
    assert 0.02 <= len(pairs) / F.size <= 0.10
    # every record satisfies the predicate, every non-record violates it
    assert np.all(d["value"] - DELTA <= tau)
    # empty scene: +inf / -1 / zero records
    e = m.detect(np.zeros((0, 3)), np.zeros(0, np.int64), q, DELTA, tau)
    assert e["count"] == 0 and np.all(np.isinf(e["wp_min"])) and np.all(e["wp_argmin"] == -1)


# ------------------------------------------------------------------ EMU_BF16 self-consistency
def test_emu_bf16_consistency(tmp_path):
    """P6(i): bf16-representable weights + weight rounding only == exact, bit for bit.
    P6(ii): full emulation stays within the bf16 error scale of the exact result."""
    act, dims, layers = synth.make_weights(32, seed=3)

    def to_bf16(a):
        u = np.asarray(a, np.float32).view(np.uint32).astype(np.uint64)
        u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
        return u.astype(np.uint32).view(np.float32).astype(np.float64)

    rl = [(to_bf16(W), b) for W, b in layers]
    m = oracle.MLP(_write(tmp_path, "bf.mlpw", act, dims, rl))
    pts, q = _rand_inputs(np.random.default_rng(8), 64, 4)
    a = m.eval(pts, q)
    b = m.eval(pts, q, flags=oracle.EMU_W)
    assert np.array_equal(a["f"], b["f"]) and np.array_equal(a["g"], b["g"])
    c = m.eval(pts, q, flags=oracle.EMU_BF16, want_hash=True)
    d = m.eval(pts, q, want_hash=True)
    assert np.max(np.abs(c["f"] - d["f"])) <= 2e-2 * max(1.0, np.abs(d["f"]).max())
    same = c["mask_hash"] == d["mask_hash"]
    gn = np.linalg.norm(d["g"], axis=-1)
    dg = np.linalg.norm(c["g"] - d["g"], axis=-1)
    assert np.all(dg[same] <= 2e-2 * np.maximum(1.0, gn[same]))


# ------------------------------------------------------------------ scene replay (O2)
def test_scene_id_rule():
    s = oracle.Scene(10)
    ids = s.update(np.arange(18, dtype=np.float32).reshape(6, 3))
    assert list(ids) == [0, 1, 2, 3, 4, 5]
    ids2 = s.update(np.ones((3, 3), np.float32), remove_ids=[1, 4])
    assert list(ids2) == [6, 7, 8]          # freed ids are not reused in the same call
    ids3 = s.update(np.ones((2, 3), np.float32))
    assert list(ids3) == [1, 4]             # ... but are in the next one
    live, xyz = s.export()
    assert list(live) == [0, 1, 2, 3, 4, 5, 6, 7, 8]
    with pytest.raises(oracle.OracleError):
        s.update(remove_ids=[9])            # unknown id: atomic failure
    assert list(s.export()[0]) == list(live)
    with pytest.raises(oracle.OracleError):
        s.update(np.ones((2, 3), np.float32))   # capacity


def test_emu_rounding_points_hand_example(tmp_path):
    """O8 pinned by hand: which quantities are rounded to bf16 (golden emu_network)."""
    g = json.loads((GOLD / "hand_example.json").read_text())["emu_network"]
    layers = [(np.array(l["W"], float), np.array(l["b"], float)) for l in g["layers"]]
    m = oracle.MLP(_write(tmp_path, "emu.mlpw", 1, [12] + [1] * 6 + [1], layers))
    P, Q = np.array([g["p"]]), np.array([g["q"]])
    for flags, key in ((0, "exact"), (oracle.EMU_W, "exact"), (oracle.EMU_A, "emu_a"),
                       (oracle.EMU_BF16, "emu_a")):
        out = m.eval(P, Q, flags=flags)
        assert out["f"][0, 0] == g[key]["f"], (flags, out["f"][0, 0])
        np.testing.assert_array_equal(out["g"][0, 0], g[key]["grad"])


def test_threshold_inclusive_hand_example(tmp_path):
    g = json.loads((GOLD / "hand_example.json").read_text())["networks"][1]
    layers = [(np.array(l["W"], float), np.array(l["b"], float)) for l in g["layers"]]
    m = oracle.MLP(_write(tmp_path, "thr.mlpw", 1, [12] + [1] * 6 + [1], layers))
    # both cases share q_xy = (1, 0) after re-basing their points: p = (1, 0) -> f = 21, p = (2, 0) -> f = 25
    pts = np.array([[1.0, 0.0, 0.3], [2.0, 0.0, 0.0]])
    q = np.array([[1.0, 0.0, 0, 0, 0, 0, 0, 0, 0]])
    tau = 25.0 - 0.1
    d = m.detect(pts, np.array([4, 9]), q, 0.1, tau)
    assert list(d["pt"]) == [4, 9] and list(d["value"]) == [21.0, 25.0]
    d = m.detect(pts, np.array([4, 9]), q, 0.1, np.nextafter(tau, -np.inf))
    assert list(d["pt"]) == [4]
    assert d["wp_min"][0] == 21.0 and d["wp_argmin"][0] == 4


def test_emu_weight_rounding_hand_example(tmp_path):
    g = json.loads((GOLD / "hand_example.json").read_text())["emu_w_network"]
    layers = [(np.array(l["W"], float), np.array(l["b"], float)) for l in g["layers"]]
    m = oracle.MLP(_write(tmp_path, "emuw.mlpw", 1, [12] + [1] * 6 + [1], layers))
    P, Q = np.array([g["p"]]), np.array([g["q"]])
    for flags, key in ((0, "exact"), (oracle.EMU_W, "emu_w"), (oracle.EMU_BF16, "emu_bf16")):
        out = m.eval(P, Q, flags=flags)
        assert out["f"][0, 0] == g[key]["f"], flags
        np.testing.assert_array_equal(out["g"][0, 0], g[key]["grad"])


def test_emu_fp16_vs_bf16_hand_example(tmp_path):
    """O8 for the fp16 operand type: hand-derived fp16 vs bf16 rounding (with a tie)."""
    g = json.loads((GOLD / "hand_example.json").read_text())["emu16_network"]
    layers = [(np.array(l["W"], float), np.array(l["b"], float)) for l in g["layers"]]
    m = oracle.MLP(_write(tmp_path, "emu16.mlpw", 1, [12] + [1] * 6 + [1], layers))
    P, Q = np.array([g["p"]]), np.array([g["q"]])
    for flags, key in ((0, "exact"), (oracle.EMU_FP16, "emu_fp16"), (oracle.EMU_BF16, "emu_bf16")):
        out = m.eval(P, Q, flags=flags)
        assert out["f"][0, 0] == g[key]["f"], (flags, out["f"][0, 0])
        np.testing.assert_array_equal(out["g"][0, 0], g[key]["grad"])


def test_emu_fp16_subnormal_and_range(tmp_path):
    """fp16 rounding of tiny backward deltas keeps subnormals (cvt.rn.f16 semantics):
    a zero-head-like network with w7 = 2^-20 must give a gradient of exactly 2^-20 * W1
    under EMU_FP16 (2^-20 is an fp16 subnormal: 2^-24 * 16)."""
    g = json.loads((GOLD / "hand_example.json").read_text())["networks"][1]
    layers = [(np.array(l["W"], float), np.array(l["b"], float)) for l in g["layers"]]
    layers[-1] = (np.array([[2.0 ** -20]]), np.array([1.0]))
    m = oracle.MLP(_write(tmp_path, "sub.mlpw", 1, [12] + [1] * 6 + [1], layers))
    out = m.eval(np.array([[2.0, 0.0, 0.0]]), np.array([[1.0, 0, 0, 0, 0, 0, 0, 0, 0]]), flags=oracle.EMU_FP16)
    assert out["g"][0, 0, 0] == -(2.0 ** -20) and out["g"][0, 0, 2] == 0.5 * 2.0 ** -20


def test_range_partition_bruteforce_C1():
    """NEXT-1 pin: the partitioned detect equals brute force over
    the pairs whose point lies within `radius` (planar distance, inclusive) of the step's
    base position; partition sizes are brute-force counts; radius <= 0 / +inf reproduce
    the unpartitioned detect exactly; a point placed exactly on the circle is included."""
    cfg = synth.get_config("C1")
    pts, _ = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg).reshape(-1, 9)
    m = oracle.MLP(synth.weights_path(cfg.H))
    ids = np.arange(pts.shape[0], dtype=np.int64) * 2 + 5
    tau = synth.load_tau("C1")
    full = m.detect(pts, ids, q, DELTA, tau)
    for r in (0.0, np.inf):
        d = m.detect(pts, ids, q, DELTA, tau, radius=r)
        for k in ("value", "grad", "wp", "pt", "wp_offsets", "wp_min", "wp_argmin"):
            np.testing.assert_array_equal(d[k], full[k])
    # boundary point: exactly radius 2.5 from waypoint 3's base (a 3-4-5 triangle, exact in f64)
    r = 2.5
    qb = q.copy()
    qb[3, 0:2] = [1.0, -2.0]
    pts_b = np.concatenate([pts, [[1.0 + 1.5, -2.0 + 2.0, 0.7]]])
    ids_b = np.concatenate([ids, [ids[-1] + 7]])
    d = m.detect(pts_b, ids_b, qb, DELTA, 1e9, radius=r)   # tau huge: every partition pair is active
    F = m.eval(pts_b, qb, want_grad=False)["f"]
    inside = ((pts_b[None, :, 0] - qb[:, None, 0]) ** 2 + (pts_b[None, :, 1] - qb[:, None, 1]) ** 2) <= r * r
    assert inside[3, -1]
    np.testing.assert_array_equal(d["part_sizes"], inside.sum(axis=1))
    pairs = [(w, int(ids_b[j])) for w in range(qb.shape[0]) for j in range(len(ids_b)) if inside[w, j]]
    assert d["count"] == len(pairs) and [(int(a), int(b)) for a, b in zip(d["wp"], d["pt"])] == pairs
    for w in range(qb.shape[0]):
        js = np.flatnonzero(inside[w])
        if js.size == 0:
            assert np.isinf(d["wp_min"][w]) and d["wp_argmin"][w] == -1
        else:
            j = js[np.argmin(F[w, js])]
            assert d["wp_min"][w] == F[w, j] and d["wp_argmin"][w] == ids_b[j]
    # the real threshold: records = brute force on the partition pairs
    d = m.detect(pts, ids, q, DELTA, tau, radius=1.8)
    F = m.eval(pts, q, want_grad=False)["f"]
    inside = ((pts[None, :, 0] - q[:, None, 0]) ** 2 + (pts[None, :, 1] - q[:, None, 1]) ** 2) <= 1.8 ** 2
    pairs = [(w, int(ids[j])) for w in range(q.shape[0]) for j in range(len(ids))
             if inside[w, j] and F[w, j] - DELTA <= tau]
    assert d["count"] == len(pairs) and [(int(a), int(b)) for a, b in zip(d["wp"], d["pt"])] == pairs
    assert 0 < d["part_sizes"].sum() < inside.size


def test_sparse_jacobian_equals_projection_products():
    """NEXT-2 pin (Eq. 17-19, reading R18): the CSR rows placed by direct
    memory operations equal the stacked dense products grad_{q_i} c_{q_i} P_i with
    (P_i)_{r,c} = 1 iff c = r + 2n(i-1) (1-based i), per trajectory block of 2Nn columns;
    c = f - delta in the records' (step-major, Eq. 14) order."""
    cfg = synth.get_config("C1")
    pts, _ = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg).reshape(-1, 9)
    m = oracle.MLP(synth.weights_path(cfg.H))
    ids = np.arange(pts.shape[0], dtype=np.int64)
    tau = synth.load_tau("C1")
    d = m.detect(pts, ids, q, DELTA, tau)
    n = 9
    for B in (1, 2):                       # the 16 steps as 1 x 16 or 2 trajectories x 8
        N = q.shape[0] // B
        sj = oracle.sparse_jacobian(d, DELTA)
        K = d["count"]
        dense = np.zeros((K, 2 * B * N * n))
        for k in range(K):
            for t in range(sj["row_ptr"][k], sj["row_ptr"][k + 1]):
                dense[k, sj["col"][t]] = sj["val"][t]
        # the paper's construction, trajectory by trajectory
        ref = np.zeros_like(dense)
        for b in range(B):
            for i in range(1, N + 1):              # 1-based step index as in Eq. 19
                wp = b * N + (i - 1)
                rows = np.flatnonzero(d["wp"] == wp)
                P = np.zeros((n, 2 * N * n))
                for r in range(n):
                    P[r, r + 2 * n * (i - 1)] = 1.0
                block = d["grad"][rows] @ P        # grad_{q_i} c_{q_i} P_i
                ref[rows, b * 2 * N * n:(b + 1) * 2 * N * n] = block
        np.testing.assert_array_equal(dense, ref)
        np.testing.assert_array_equal(sj["c"], d["value"] - DELTA)
        assert np.array_equal(sj["row_ptr"], np.arange(K + 1) * n)
        # Eq. 14 order: rows grouped by step, steps ascending
        assert np.all(np.diff(d["wp"]) >= 0)


def test_single_step_projection_reaches_zero_level_set(tmp_path):
    """NEXT-3 pin (Theorem 1.2): for a field satisfying the weighted eikonal
    equation ||grad_q f||_{M^-1} = 1 -- here a linear (identity-activation) network whose
    output layer is scaled to unit M^-1-norm gradient -- one step q_z = q - f M^-1 grad f
    lands on the zero level set: f(p, q_z) = 0.  With M = I and a unit gradient the step is
    q - f grad f; the projection is the plain formula on random fields too."""
    rng = np.random.default_rng(9)
    dims = [12, 9, 7, 8, 6, 5, 4, 1]
    layers = [(rng.normal(size=(dims[i + 1], dims[i])), rng.normal(size=dims[i + 1])) for i in range(7)]
    minv = rng.uniform(0.2, 3.0, 9)
    for mv in (minv, np.ones(9)):
        m0 = oracle.MLP(_write(tmp_path, "lin0.mlpw", 0, dims, layers))
        pts, q = _rand_inputs(rng, 7, 5)
        g = m0.eval(pts, q)["g"][0, 0]                    # constant gradient of a linear field
        s = 1.0 / np.sqrt(g @ (mv * g))                  # ||s g||_{M^-1} = 1
        scaled = layers[:-1] + [(layers[-1][0] * s, layers[-1][1] * s)]
        m = oracle.MLP(_write(tmp_path, "lin.mlpw", 0, dims, scaled))
        out = m.eval(pts, q)
        np.testing.assert_allclose(np.einsum("wjt,t,wjt->wj", out["g"], mv, out["g"]), 1.0, rtol=1e-12)
        qz = oracle.project(out["f"], out["g"], q, mv)
        for w in range(q.shape[0]):
            fz = m.eval(pts, qz[w])["f"]                  # f(p_j, q_z[w, j]) on the diagonal
            np.testing.assert_allclose(np.diag(fz), 0.0, atol=1e-10)
    # random ReLU field: the formula itself, component by component
    act, dims2, layers2 = synth.make_weights(32, seed=4)
    m2 = oracle.MLP(_write(tmp_path, "r.mlpw", act, dims2, layers2))
    pts, q = _rand_inputs(rng, 6, 3)
    out = m2.eval(pts, q)
    qz = oracle.project(out["f"], out["g"], q, minv)
    for w in range(q.shape[0]):
        for j in range(pts.shape[0]):
            for t in range(9):
                assert qz[w, j, t] == q[w, t] - out["f"][w, j] * (minv[t] * out["g"][w, j, t])


def test_se2_frame_variant(mlp32):
    """NEXT-4 SE(2) frame pins (reading R24): (i) rigid-motion invariance -- rotating every
    point and the base about an arbitrary centre by phi and adding phi to theta leaves f
    unchanged, rotates the translational gradient by phi and keeps d f/d theta and the
    joint gradients; (ii) central FD of the variant's forward, all 9 components; (iii) at
    theta = 0 the variant equals the translation-only frame (R(0) = I, theta channel 0)."""
    m, _ = mlp32
    S = oracle.FRAME_SE2
    rng = np.random.default_rng(21)
    pts, q = _rand_inputs(rng, 30, 6)
    base = m.eval(pts, q, flags=S, want_hash=True)
    for phi, ctr in ((0.7, np.array([1.3, -2.1])), (-2.4, np.array([-3.0, 0.5]))):
        c, s = np.cos(phi), np.sin(phi)
        R = np.array([[c, -s], [s, c]])
        pts2 = pts.copy()
        pts2[:, :2] = (pts[:, :2] - ctr) @ R.T + ctr
        q2 = q.copy()
        q2[:, :2] = (q[:, :2] - ctr) @ R.T + ctr
        q2[:, 2] = q[:, 2] + phi
        o2 = m.eval(pts2, q2, flags=S)
        np.testing.assert_allclose(o2["f"], base["f"], rtol=1e-11, atol=1e-11)
        np.testing.assert_allclose(o2["g"][..., :2], base["g"][..., :2] @ R.T, rtol=1e-9, atol=1e-10)
        np.testing.assert_allclose(o2["g"][..., 2:], base["g"][..., 2:], rtol=1e-9, atol=1e-10)
    checked = skipped = 0
    for k in range(9):
        h = 1e-6 * np.maximum(1.0, np.abs(q[:, k]))
        qp, qm = q.copy(), q.copy()
        qp[:, k] += h
        qm[:, k] -= h
        op = m.eval(pts, qp, flags=S, want_grad=False, want_hash=True)
        om = m.eval(pts, qm, flags=S, want_grad=False, want_hash=True)
        fd = (op["f"] - om["f"]) / (2 * h[:, None])
        same = (op["mask_hash"] == base["mask_hash"]) & (om["mask_hash"] == base["mask_hash"])
        g = base["g"][:, :, k]
        err = np.abs(fd - g) / np.maximum(1.0, np.abs(g))
        assert np.all(err[same] <= 1e-6), (k, err[same].max())
        checked += same.sum()
        skipped += (~same).sum()
    assert skipped <= 0.02 * (checked + skipped)
    q0 = q.copy()
    q0[:, 2] = 0.0
    a0 = m.eval(pts, q0, flags=S)
    b0 = m.eval(pts, q0)
    np.testing.assert_array_equal(a0["f"], b0["f"])
    np.testing.assert_array_equal(a0["g"][..., [0, 1, 3, 4, 5, 6, 7, 8]], b0["g"][..., [0, 1, 3, 4, 5, 6, 7, 8]])
    with pytest.raises(oracle.OracleError):
        m.eval(pts, q, flags=S | oracle.TGRAD_QCHANNEL)


# ------------------------------------------------------------------ softplus variant (NEXT-4, R26)
@pytest.fixture(scope="module")
def mlp32_softplus(tmp_path_factory):
    _, dims, layers = synth.make_weights(32, seed=12)
    p = tmp_path_factory.mktemp("w") / "h32sp.mlpw"
    synth.write_mlpw(p, 2, dims, layers)
    return oracle.MLP(p), (2, dims, layers)


def test_softplus_hand_worked_example(tmp_path):
    """Hand-worked softplus network (tests/golden/softplus_hand_example.json): every
    softplus / sigmoid value along the path is ln 2, ln 3, 1/2, 3/4, 2/3 or 1/4."""
    g = json.loads((GOLD / "softplus_hand_example.json").read_text())
    layers = [(np.array(l["W"], float), np.array(l["b"], float)) for l in g["layers"]]
    m = oracle.MLP(_write(tmp_path, "sphand.mlpw", 2, [12] + [1] * 6 + [1], layers))
    assert m.act == 2
    for case in g["cases"]:
        out = m.eval(np.array([case["p"]]), np.array([case["q"]]))
        assert abs(out["f"][0, 0] - case["f"]) <= 1e-12
        np.testing.assert_allclose(out["g"][0, 0], case["grad"], rtol=0, atol=1e-12)


def test_softplus_emu_hand_worked(tmp_path):
    """The softplus EMU_FP16 mode (R26 rounding points: h1..h5 rounded as A operands,
    sigma' of layers 1..5 recovered as 1 - e^-h~ from the rounded activation, sigma'6 =
    sigmoid(z6) unrounded, every backward delta rounded) on the hand-worked network with
    W7 = 1.313, against the step-by-step derivation in softplus_hand_example.json
    ["emu_fp16"] (tools/golden_softplus_emu.py: math + numpy float16, no oracle).  The
    golden also lists six mis-placed rounding points (e.g. sigma'6 from the rounded h6),
    each of which changes f or the gradient, so each would fail this pin."""
    g = json.loads((GOLD / "softplus_hand_example.json").read_text())
    e = g["emu_fp16"]
    layers = [(np.array(l["W"], float), np.array(l["b"], float)) for l in e["layers"]]
    m = oracle.MLP(_write(tmp_path, "spemu.mlpw", 2, [12] + [1] * 6 + [1], layers))
    for case in g["cases"]:
        out = m.eval(np.array([case["p"]]), np.array([case["q"]]), flags=oracle.EMU_FP16)
        assert abs(out["f"][0, 0] - e["f"]) <= 1e-12
        np.testing.assert_allclose(out["g"][0, 0], e["grad"], rtol=0, atol=1e-15)
        for name, mu in e["_mutants"].items():
            assert abs(out["f"][0, 0] - mu["f"]) > 1e-12 or abs(out["g"][0, 0][0] - mu["grad0"]) > 1e-12, name


def test_softplus_saturated_is_affine_closed_form(tmp_path):
    """Every pre-activation >= 40: softplus(z) = z + log1p(e^-z) = z (1 + O(1e-19)) and
    sigmoid(z) = 1 - O(1e-18), so the network equals the affine composition and the
    gradient the mapped row of the product (same closed form as the identity activation)."""
    rng = np.random.default_rng(21)
    dims = [12, 9, 7, 8, 6, 5, 4, 1]
    layers = [(rng.uniform(0.0, 0.05, (dims[i + 1], dims[i])), np.full(dims[i + 1], 60.0)) for i in range(7)]
    m = oracle.MLP(_write(tmp_path, "spsat.mlpw", 2, dims, layers))
    A, c = np.eye(12), np.zeros(12)
    for W, b in layers:
        A, c = W @ A, W @ c + b
    pts = np.stack([rng.uniform(0, 3, 11), rng.uniform(0, 3, 11), rng.uniform(0, 2, 11)], 1)
    q = np.concatenate([rng.uniform(-3, 0, (4, 2)), rng.uniform(0, 1, (4, 7))], 1)
    out = m.eval(pts, q)
    for w in range(q.shape[0]):
        for j in range(pts.shape[0]):
            x = np.concatenate([[pts[j, 0] - q[w, 0], pts[j, 1] - q[w, 1], pts[j, 2], 0, 0], q[w, 2:]])
            f = (A @ x + c)[0]
            assert abs(out["f"][w, j] - f) <= 1e-12 * abs(f)
            row = A[0]
            np.testing.assert_allclose(out["g"][w, j], np.concatenate([[-row[0], -row[1]], row[5:]]),
                                       rtol=1e-12, atol=1e-15)


def test_softplus_cutoff_is_constant(tmp_path):
    """Every first-layer pre-activation <= -745 (e^z underflows to 0 in f64): h1 = 0 exactly
    and sigma'(z1) = 0, so f is the network evaluated on h1 = 0 (independent of the input)
    and the gradient vanishes."""
    rng = np.random.default_rng(22)
    _, dims, layers = synth.make_weights(8, seed=4)
    layers[0] = (np.zeros_like(layers[0][0]), np.full(8, -800.0))
    m = oracle.MLP(_write(tmp_path, "spcut.mlpw", 2, dims, layers))
    pts, q = _rand_inputs(rng, 9, 3)
    out = m.eval(pts, q)
    assert np.all(out["f"] == out["f"][0, 0])
    assert np.all(out["g"] == 0.0)
    # the constant: softplus network on h1 = 0, written with numpy (log1p(exp)) layer by layer
    h = np.zeros(8)
    for W, b in layers[1:-1]:
        z = W @ h + b
        h = np.log1p(np.exp(z))
    f = (layers[-1][0] @ h + layers[-1][1])[0]
    assert abs(out["f"][0, 0] - f) <= 1e-12 * max(1, abs(f))


def test_softplus_torch_autograd_float64(mlp32_softplus):
    """Independent differentiation: torch float64 autograd with torch's softplus (threshold
    raised to 50 so it never switches to the identity)."""
    torch = pytest.importorskip("torch")
    m, (_, dims, layers) = mlp32_softplus
    rng = np.random.default_rng(23)
    pts, q = _rand_inputs(rng, 64, 5)
    out = m.eval(pts, q)
    Ws = [(torch.tensor(W), torch.tensor(b)) for W, b in layers]
    P = torch.tensor(pts)
    for w in range(q.shape[0]):
        qt = torch.tensor(q[w]).repeat(P.shape[0], 1).requires_grad_(True)
        h = torch.cat([P[:, :2] - qt[:, :2], P[:, 2:3], torch.zeros(P.shape[0], 2, dtype=torch.float64),
                       qt[:, 2:]], 1)
        for li, (W, b) in enumerate(Ws):
            h = h @ W.T + b
            if li < len(Ws) - 1:
                h = torch.nn.functional.softplus(h, beta=1.0, threshold=50.0)
        f = h[:, 0]
        (gq,) = torch.autograd.grad(f.sum(), qt)
        np.testing.assert_allclose(out["f"][w], f.detach().numpy(), rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(out["g"][w], gq.numpy(), rtol=1e-10, atol=1e-12)


def test_softplus_central_fd_and_invariance(mlp32_softplus):
    """Central FD of all 9 components (smooth network: nothing skipped) and base-translation
    invariance (bit-identical on dyadic inputs)."""
    m, _ = mlp32_softplus
    rng = np.random.default_rng(24)
    pts, q = _rand_inputs(rng, 40, 5)
    base = m.eval(pts, q)
    for k in range(9):
        h = 1e-5 * np.maximum(1.0, np.abs(q[:, k]))
        qp, qm = q.copy(), q.copy()
        qp[:, k] += h
        qm[:, k] -= h
        fd = (m.eval(pts, qp, want_grad=False)["f"] - m.eval(pts, qm, want_grad=False)["f"]) / (2 * h[:, None])
        g = base["g"][:, :, k]
        assert np.all(np.abs(fd - g) <= 1e-7 * np.maximum(1.0, np.abs(g))), k
    pts, q = _rand_inputs(rng, 30, 3, dyadic=True)
    a = m.eval(pts, q)
    p2, q2 = pts.copy(), q.copy()
    p2[:, :2] += [2.75, -4.5]
    q2[:, :2] += [2.75, -4.5]
    b = m.eval(p2, q2)
    assert np.array_equal(a["f"], b["f"]) and np.array_equal(a["g"], b["g"])


def test_softplus_emu_consistency(mlp32_softplus):
    """EMU_FP16 (tensor-path rounding points, R26: 16-bit A operands, sigma' of layers 1..5
    recovered as 1 - exp(-h~) from the rounded activation) stays within the 16-bit error
    scale of the exact result (the recovery is exact for unrounded h: 1 - e^-softplus(z) =
    sigmoid(z))."""
    m, _ = mlp32_softplus
    pts, q = _rand_inputs(np.random.default_rng(25), 64, 4)
    d = m.eval(pts, q)
    c = m.eval(pts, q, flags=oracle.EMU_FP16)
    assert np.max(np.abs(c["f"] - d["f"])) <= 5e-3 * max(1.0, np.abs(d["f"]).max())
    gn = np.linalg.norm(d["g"], axis=-1)
    assert np.all(np.linalg.norm(c["g"] - d["g"], axis=-1) <= 1e-2 * np.maximum(1.0, gn))


# ------------------------------------------------------------------ randomized brute force
def test_detect_equals_bruteforce_randomized(tmp_path):
    """Property check on many tiny random problems (hypothesis): the oracle's detect (O6, O7)
    equals enumerate-filter-sort-min over its own pairwise evaluation, for random widths,
    activations, ids with holes, duplicated points (exact value ties), thresholds (incl. one
    that hits a value exactly) and range partitions."""
    hyp = pytest.importorskip("hypothesis")
    st = hyp.strategies

    @hyp.settings(max_examples=40, deadline=None, derandomize=True)
    @hyp.given(seed=st.integers(0, 2**31 - 1), act=st.sampled_from([1, 2]), H=st.sampled_from([2, 5, 8]),
               M=st.integers(0, 12), W=st.integers(1, 4), radius=st.sampled_from([0.0, 2.5, 6.0]))
    def check(seed, act, H, M, W, radius):
        rng = np.random.default_rng(seed)
        _, dims, layers = synth.make_weights(H, seed=seed % 1000)
        path = tmp_path / f"r{seed}_{act}_{H}.mlpw"
        synth.write_mlpw(path, act, dims, layers)
        m = oracle.MLP(path)
        pts, q = _rand_inputs(rng, M, W)
        if M >= 2:
            pts[M - 1] = pts[0]  # a duplicated point: equal values, smaller id must win
        ids = np.sort(rng.choice(10 * M + 1, size=M, replace=False)).astype(np.int64)
        full = m.eval(pts, q)
        f = full["f"]
        tau = float(f.ravel()[rng.integers(f.size)]) - DELTA if f.size else 0.5  # hits a value exactly
        d = m.detect(pts, ids, q, DELTA, tau, radius=radius)
        inr = np.ones((W, M), bool)
        if radius > 0:
            inr = (pts[None, :, 0] - q[:, None, 0]) ** 2 + (pts[None, :, 1] - q[:, None, 1]) ** 2 <= radius ** 2
        want = [(w, ids[j]) for w in range(W) for j in range(M) if inr[w, j] and f[w, j] - DELTA <= tau]
        want.sort()
        got = list(zip(d["wp"].tolist(), d["pt"].tolist()))
        assert got == [(int(a), int(b)) for a, b in want]
        assert d["count"] == len(want)
        for w in range(W):
            cand = [(f[w, j], ids[j]) for j in range(M) if inr[w, j]]
            if cand:
                fm, im = min(cand)
                assert d["wp_min"][w] == fm and d["wp_argmin"][w] == im
            else:
                assert np.isinf(d["wp_min"][w]) and d["wp_argmin"][w] == -1
        assert np.array_equal(np.diff(d["wp_offsets"]), np.bincount(d["wp"], minlength=W)[:W] if len(want) else
                              np.zeros(W, np.int64))

    check()

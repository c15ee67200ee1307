"""Shared helpers of the GPU parity tests (the CUDA path vs the float64 oracle)."""
from __future__ import annotations

import numpy as np

import oracle
import synth

DELTA = synth.inputs.DELTA

# fp32 path, BASELINE north_star: 1e-4 relative / 1e-5 absolute (allclose form, R17)
FP32_RTOL, FP32_ATOL = 1e-4, 1e-5
# gradient of a ReLU net is discontinuous at kinks: a pair may differ only if some
# hidden pre-activation is within KINK of zero.  fp32 rounding of z is ~1e-6 at the R11
# scale: 1e-5 passes every fp32-tolerance suite, 1e-6 fails four (R17); round 1 used 1e-4
KINK_FP32 = 1e-5
BAND_FP32 = 1e-3          # active-set parity band around the threshold (north_star)
# bf16 tensor-core path (R17)
BF16_VAL_ATOL = 2e-2      # value vs exact oracle
BF16_GNORM_ATOL = 5e-2    # | ||g_gpu|| - ||g_oracle|| |
BF16_EMU_VAL_ATOL = 1e-3  # value vs EMU_BF16 oracle
BF16_EMU_GREL = 1e-2      # ||dg|| <= 1e-2 max(1, ||g||) vs EMU_BF16
BAND_BF16 = BAND_FP32 + BF16_VAL_ATOL


def scene_for(cfg, ctx=None):
    pts, boxes = synth.make_scene_points(cfg)
    ids = None
    if ctx is not None:
        ids = ctx.update_scene(pts)
    return pts, boxes, ids


def fp32_close(a, o):
    return np.abs(a - o) <= FP32_ATOL + FP32_RTOL * np.abs(o)


def check_fp32_dense(gv, gg, ov, og, kappa, what=""):
    """values: every pair; gradients: every pair except <0.1% within KINK of a ReLU kink."""
    bad_v = ~fp32_close(gv, ov)
    assert not bad_v.any(), f"{what}: {bad_v.sum()} values out of tolerance, max err {np.abs(gv - ov).max():.3e}"
    bad_g = ~np.all(fp32_close(gg, og), axis=-1)
    near = kappa <= KINK_FP32
    assert not (bad_g & ~near).any(), f"{what}: {(bad_g & ~near).sum()} kink-free gradients out of tolerance"
    assert bad_g.sum() <= 1e-3 * bad_g.size + 1, f"{what}: {bad_g.sum()} gradients differ near kinks"
    return int(bad_g.sum())


def records_np(out):
    from paper_2601_18548_b200 import records_to_dict
    n = int(out["n"]) if "n" in out else int(out["count"].item())
    n = min(n, int(out["capacity"]))
    d = records_to_dict(out["records"], n)
    return {k: v.cpu().numpy() for k, v in d.items()}


def compare_active_sets(gpu, orc, full_f, ids, band, val_atol=None, grad_check=None, kappa_full=None, what=""):
    """gpu: records dict (value, grad, wp, pt); orc: oracle detect dict; full_f [W, M] oracle
    values with ids [M] for the band test.  Sets must match except pairs within `band`
    of the threshold; matched records are checked by val_atol / grad_check."""
    pos = {int(i): j for j, i in enumerate(ids)}
    g_keys = list(zip(gpu["wp"].tolist(), gpu["pt"].tolist()))
    o_keys = list(zip(orc["wp"].tolist(), orc["pt"].tolist()))
    assert g_keys == sorted(g_keys), f"{what}: GPU records not in canonical (wp, pt) order"
    gs, os_ = set(g_keys), set(o_keys)
    diff = gs ^ os_
    tau_eff = orc["_tau"] + DELTA
    for (w, pt) in diff:
        f = full_f[w, pos[pt]]
        assert abs(f - tau_eff) <= band, f"{what}: pair ({w},{pt}) f={f} differs but is {abs(f - tau_eff):.3e} from threshold"
    gi = {k: i for i, k in enumerate(g_keys)}
    oi = {k: i for i, k in enumerate(o_keys)}
    common = sorted(gs & os_)
    ga = np.array([gi[k] for k in common], dtype=np.int64)
    oa = np.array([oi[k] for k in common], dtype=np.int64)
    if len(common):
        if val_atol is None:
            assert np.all(fp32_close(gpu["value"][ga], orc["value"][oa])), what
        else:
            assert np.all(np.abs(gpu["value"][ga] - orc["value"][oa]) <= val_atol), what
        if grad_check is not None:
            kap = None if kappa_full is None else np.array([kappa_full[w, pos[pt]] for (w, pt) in common])
            grad_check(gpu["grad"][ga], orc["grad"][oa], kap)
    return len(diff), len(common)


def oracle_detect(m, pts, ids, q, tau, flags=0, nthreads=8):
    d = m.detect(pts, ids, q, DELTA, tau, flags=flags, nthreads=nthreads)
    d["_tau"] = tau
    return d


def oracle_mlp(cfg):
    return oracle.MLP(synth.weights_path(cfg.H))

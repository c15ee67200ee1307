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

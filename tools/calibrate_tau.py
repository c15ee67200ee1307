"""Freeze the activation margin tau per config (R12) -> configs/tau.json.

tau = (quantile_q of f over a seeded subsample of the config's pairs) - delta, so that
about a fraction q of pairs is active.  f comes ONLY from the float64 oracle
(oracle/), never from the CUDA path; this script is the provenance of every tau.
Usage: python tools/calibrate_tau.py [--threads T]
"""
import argparse
import dataclasses
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
import synth   # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--wp", type=int, default=16)
    ap.add_argument("--pts", type=int, default=16384)
    a = ap.parse_args()
    out = {}
    # act 1: the ReLU network (R9); act 2: the same weights under softplus (NEXT-4, R26),
    # stored as "<config>_softplus"; hidden 256: the wide network (NEXT-4, R27), "<config>_H256"
    for act, hidden in ((1, None), (2, None), (1, 256)):
        for name, cfg in synth.CONFIGS.items():
            if hidden is not None:
                if cfg.H != 128:
                    continue
                cfg = dataclasses.replace(cfg, H=hidden)
            pts, _ = synth.make_scene_points(cfg)
            q = synth.make_waypoints(cfg).reshape(-1, 9)
            rng = np.random.default_rng([cfg.seed, 99])
            wsel = np.sort(rng.choice(q.shape[0], size=min(a.wp, q.shape[0]), replace=False))
            psel = np.sort(rng.choice(pts.shape[0], size=min(a.pts, pts.shape[0]), replace=False))
            m = oracle.MLP(synth.weights_path(cfg.H, act=act))
            f = m.eval(pts[psel], q[wsel], want_grad=False, nthreads=a.threads)["f"].ravel()
            quant = float(np.quantile(f, cfg.quantile))
            tau = quant - synth.inputs.DELTA
            frac = float(np.mean(f - synth.inputs.DELTA <= tau))
            key = synth.tau_key(name, act, hidden)
            out[key] = {"tau": tau, "quantile": cfg.quantile, "sample_pairs": int(f.size),
                        "sample_active_fraction": frac, "f_mean": float(f.mean()), "f_std": float(f.std())}
            print(key, out[key], flush=True)
    out["_provenance"] = ("written by tools/calibrate_tau.py from oracle/ float64 values on a seeded "
                          "subsample (rng seed [cfg.seed, 99]); delta = %.2f" % synth.inputs.DELTA)
    (ROOT / "configs").mkdir(exist_ok=True)
    (ROOT / "configs" / "tau.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()

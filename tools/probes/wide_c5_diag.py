"""Diagnostics for the H = 256 C5 sampled parity: the pairs with the largest gradient-norm
error vs the exact oracle among the kink-free ones (dev tool)."""
import os
import sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np
import torch

import oracle
import synth
from paper_2601_18548_b200 import FP16, Context

H = 256
cfg = synth.get_config("C5")
pts, _ = synth.make_scene_points(cfg)
q = synth.make_waypoints(cfg)
ctx = Context(0, precision=FP16, scene_capacity=cfg.M + 4096, max_waypoints=256, max_active=1 << 22)
ctx.load_weights(synth.weights_path(H))
ctx.update_scene(pts)
m = oracle.MLP(synth.weights_path(H))
Q = q.reshape(-1, 9)
rng = np.random.default_rng(2026)
wsel = np.sort(rng.choice(Q.shape[0], 2, replace=False))
psel = np.sort(rng.choice(len(pts), 2048, replace=False))
NT = os.cpu_count()
ex = m.eval(pts[psel], Q[wsel], want_kappa=True, want_hash=True, nthreads=NT)
em = m.eval(pts[psel], Q[wsel], flags=oracle.EMU_FP16, want_kappa=True, want_hash=True, nthreads=NT)
v, g = ctx.query_values_grads(torch.from_numpy(Q[wsel].reshape(1, -1, 9)))
g = g.cpu().numpy()[:, psel]
gn = np.linalg.norm(g, axis=-1)
ge = np.linalg.norm(ex["g"], axis=-1)
gm = np.linalg.norm(em["g"], axis=-1)
kf = (ex["mask_hash"] == em["mask_hash"]) & (em["kappa"] > 1e-3)
gd = np.abs(gn - ge)
order = np.argsort(-(gd * kf).ravel())[:8]
for o in order:
    w, j = np.unravel_index(o, gd.shape)
    print(f"w={wsel[w]} pt={psel[j]} |g| gpu {gn[w, j]:.5f} emu {gm[w, j]:.5f} exact {ge[w, j]:.5f} "
          f"kappa_emu {em['kappa'][w, j]:.2e} kappa_ex {ex['kappa'][w, j]:.2e} |dg_emu| "
          f"{np.linalg.norm(g[w, j] - em['g'][w, j]):.2e}")
# the same pairs on a small scene holding only the sampled points (K2w tiles of a different shape)
ctx2 = Context(0, precision=FP16, scene_capacity=4096, max_waypoints=256, max_active=1 << 16)
ctx2.load_weights(synth.weights_path(H))
ctx2.update_scene(pts[psel])
v2, g2 = ctx2.query_values_grads(torch.from_numpy(Q[wsel].reshape(1, -1, 9)))
g2 = g2.cpu().numpy()[:, : len(psel)]
print("small-scene vs full-scene gradient max diff", np.abs(g2 - g).max())

"""Seeded synthetic workloads shaped like the paper's randomized-clutter benchmark.

Everything here is random-number drawing and file writing; none of the method's
arithmetic lives here (see synth/__init__.py).  Recipe:

* Map: 14 x 14 m, rectangular obstacles "with varying heights", 80/100/120 of them
  (Sec. V-C "randomized cluttered environments").  Box sizes are not
  given in the paper; half-extents U(0.1, 0.6) m follow SPEC.md:489's planar sizes.
* Obstacle points: area-uniform on the six faces of each box, fp32, exact count.
  Points within 0.5 m (xy) of the start base are redrawn.
* Waypoints: start at the map centre with the arm at zero, goal >= 3 m away
  (PAPER.md:527), base linearly interpolated (naive init) plus
  jitter so the arm joints are exercised.  q = [x, y, theta, j1..j6] (PAPER.md:350-352,
  n = 9 for the 6-DoF Kinova Gen3 on a planar base).
* Weights: the paper's "7-layer MLP" on [p, q] in R^{3+n} with
  random init (no trained weights are available): He-normal N(0, 2/fan_in)
  on every layer including the output row, b ~ U(-0.1, 0.1), output bias 1.0.  With the
  He-normal output row the median ||grad_q f||_2 is ~1 (0.99 at C2, H = 128), the scale
  Theorem 1 fixes for a GCDF's gradient, so the north-star's absolute
  tolerances are read at the paper's scale (R11).  Written as MLPW v1.
"""
from __future__ import annotations

import json
import os
import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
N_DOF = 9          # [x, y, theta, j1..j6]
N_IN = 3 + N_DOF   # MLP input width, "(3+n)"
MAP_HALF = 7.0     # 14 x 14 m map


@dataclass(frozen=True)
class Config:
    name: str
    B: int            # parallel trajectories
    N: int            # waypoints per trajectory
    M: int            # obstacle points
    H: int            # hidden width
    boxes: int
    seed: int
    quantile: float   # target active fraction used to calibrate tau (configs/tau.json)
    dynamic: bool = False
    desc: str = ""

    @property
    def pairs(self) -> int:
        return self.B * self.N * self.M


# BASELINE.json "configs" C1..C5.
CONFIGS = {
    "C1": Config("C1", 1, 16, 256, 32, 100, 101, 0.05, desc="1 traj x 16 wp x 256 pts, small MLP"),
    "C2": Config("C2", 1, 64, 10_000, 128, 100, 102, 0.01, desc="1 traj x 64 wp x 10k pts"),
    "C3": Config("C3", 1, 100, 100_000, 128, 120, 103, 0.01, desc="dense clutter, 100 wp x 100k pts"),
    "C4": Config("C4", 128, 64, 20_000, 128, 100, 104, 0.01, dynamic=True,
                 desc="128 traj x 64 wp x 20k pts, incremental scene updates"),
    "C5": Config("C5", 1, 256, 1_000_000, 128, 120, 105, 0.01, desc="256 wp x 1M pts (8-GPU config)"),
}

DELTA = 0.10  # safety threshold delta; the paper never gives it; SPEC.md:455 uses 0.10


def get_config(name: str) -> Config:
    return CONFIGS[name]


def tau_key(name: str, act: int = 1, hidden=None) -> str:
    """configs/tau.json key: "<name>", "<name>_softplus" (act 2, R26) or "<name>_H256" (R27)."""
    if hidden is not None and hidden != get_config(name).H:
        return f"{name}_H{hidden}"
    return name if act == 1 else name + "_softplus"


def load_tau(name: str, act: int = 1, hidden=None) -> float:
    """tau frozen by tools/calibrate_tau.py (which calls only oracle/)."""
    with open(REPO / "configs" / "tau.json") as fh:
        return float(json.load(fh)[tau_key(name, act, hidden)]["tau"])


# ----------------------------------------------------------------------------- scene
def make_boxes(rng: np.random.Generator, n_boxes: int) -> np.ndarray:
    """[n_boxes, 7] = cx, cy, half_x, half_y, yaw, z_bottom, height."""
    cx = rng.uniform(-MAP_HALF, MAP_HALF, n_boxes)
    cy = rng.uniform(-MAP_HALF, MAP_HALF, n_boxes)
    hx = rng.uniform(0.1, 0.6, n_boxes)
    hy = rng.uniform(0.1, 0.6, n_boxes)
    yaw = rng.uniform(0.0, np.pi, n_boxes)
    z0 = rng.uniform(0.0, 1.2, n_boxes)
    h = rng.uniform(0.1, 0.8, n_boxes)
    return np.stack([cx, cy, hx, hy, yaw, z0, h], axis=1)


def _sample_on_boxes(rng: np.random.Generator, boxes: np.ndarray, n: int) -> np.ndarray:
    """n points area-uniform over all faces of all boxes (float64)."""
    cx, cy, hx, hy, yaw, z0, h = boxes.T
    # face areas: top, bottom, +x, -x, +y, -y
    a_tb = 4.0 * hx * hy
    a_x = 2.0 * hy * h
    a_y = 2.0 * hx * h
    areas = np.stack([a_tb, a_tb, a_x, a_x, a_y, a_y], axis=1).reshape(-1)
    face = rng.choice(areas.size, size=n, p=areas / areas.sum())
    b = face // 6
    f = face % 6
    u = rng.uniform(-1.0, 1.0, n)
    v = rng.uniform(0.0, 1.0, n)
    w = rng.uniform(-1.0, 1.0, n)
    lx = np.empty(n); ly = np.empty(n); lz = np.empty(n)
    # top / bottom
    m = f < 2
    lx[m] = u[m] * hx[b[m]]; ly[m] = w[m] * hy[b[m]]
    lz[m] = np.where(f[m] == 0, h[b[m]], 0.0)
    # +x / -x
    m = (f == 2) | (f == 3)
    lx[m] = np.where(f[m] == 2, hx[b[m]], -hx[b[m]]); ly[m] = u[m] * hy[b[m]]; lz[m] = v[m] * h[b[m]]
    # +y / -y
    m = f >= 4
    ly[m] = np.where(f[m] == 4, hy[b[m]], -hy[b[m]]); lx[m] = u[m] * hx[b[m]]; lz[m] = v[m] * h[b[m]]
    c, s = np.cos(yaw[b]), np.sin(yaw[b])
    x = cx[b] + c * lx - s * ly
    y = cy[b] + s * lx + c * ly
    z = z0[b] + lz
    return np.stack([x, y, z], axis=1)


def make_scene_points(cfg: Config, start_clear: float = 0.5):
    """Returns (points fp32 [M,3], boxes [nb,7]).  Deterministic from cfg.seed."""
    rng = np.random.default_rng([cfg.seed, 1])
    boxes = make_boxes(rng, cfg.boxes)
    pts = _sample_on_boxes(rng, boxes, cfg.M)
    while True:  # redraw points too close to the start base (the robot stands there)
        bad = np.hypot(pts[:, 0], pts[:, 1]) < start_clear
        if not bad.any():
            break
        pts[bad] = _sample_on_boxes(rng, boxes, int(bad.sum()))
    return pts.astype(np.float32), boxes


def make_waypoints(cfg: Config, mode: str = "interp") -> np.ndarray:
    """q fp32 [B, N, 9]: straight-line base interpolation start->goal plus jitter."""
    rng = np.random.default_rng([cfg.seed, 2])
    q = np.zeros((cfg.B, cfg.N, N_DOF))
    s = np.linspace(0.0, 1.0, cfg.N)[:, None]
    for b in range(cfg.B):
        r = rng.uniform(3.0, 6.5)
        bearing = rng.uniform(-np.pi, np.pi)
        goal = np.zeros(N_DOF)
        goal[0], goal[1], goal[2] = r * np.cos(bearing), r * np.sin(bearing), bearing
        if mode != "naive":
            goal[3:] = rng.uniform(-np.pi / 2, np.pi / 2, 6)
        traj = s * goal[None, :]
        jit = np.zeros((cfg.N, N_DOF))
        jit[:, 0:2] = rng.normal(0.0, 0.1, (cfg.N, 2))
        jit[:, 2] = rng.normal(0.0, 0.3, cfg.N)
        if mode != "naive":
            jit[:, 3:] = rng.normal(0.0, 0.3, (cfg.N, 6))
        q[b] = traj + jit
    return q.astype(np.float32)


def scene_update_batch(rng: np.random.Generator, boxes: np.ndarray, live_ids: np.ndarray,
                       n_remove: int = 200, n_add: int = 200):
    """C4 dynamics: remove n_remove random live ids; add n_add points on one box moved by
    U(-0.3, 0.3)^2 m.  Returns (add_xyz fp32 [n_add,3], remove_ids int64 [n_remove])."""
    rem = np.sort(rng.choice(live_ids, size=min(n_remove, live_ids.size), replace=False)).astype(np.int64)
    return _moved_box_points(rng, boxes, n_add), rem


def scene_update_batch_mask(rng: np.random.Generator, boxes: np.ndarray, alive: np.ndarray,
                            n_remove: int = 200, n_add: int = 200):
    """Same dynamics as scene_update_batch for a large scene given as a boolean alive[id]
    mask (O(n_remove) rejection sampling instead of O(M) work per step)."""
    picked = set()
    while len(picked) < n_remove:
        i = int(rng.integers(0, alive.size))
        if alive[i]:
            picked.add(i)
    rem = np.array(sorted(picked), dtype=np.int64)
    return _moved_box_points(rng, boxes, n_add), rem


def _moved_box_points(rng, boxes, n_add):
    box = boxes[rng.integers(0, boxes.shape[0])].copy()
    box[0:2] += rng.uniform(-0.3, 0.3, 2)
    return _sample_on_boxes(rng, box[None, :], n_add).astype(np.float32)


# ----------------------------------------------------------------------------- weights
def make_weights(H: int, seed: int = 7, n_hidden_layers: int = 6, act: int = 1):
    """Random-init weights of the paper's network shape [12, H x 6, 1].

    Returns (act, dims, [(W[out][in] f64, b[out] f64), ...])."""
    rng = np.random.default_rng([seed, H, 3])
    dims = [N_IN] + [H] * n_hidden_layers + [1]
    layers = []
    for li in range(len(dims) - 1):
        fan_in, fan_out = dims[li], dims[li + 1]
        W = rng.normal(0.0, np.sqrt(2.0 / fan_in), (fan_out, fan_in))
        if li < len(dims) - 2:
            b = rng.uniform(-0.1, 0.1, fan_out)
        else:
            b = np.ones(fan_out)
        layers.append((W, b))
    return act, dims, layers


def write_mlpw(path, act: int, dims, layers) -> None:
    """MLPW v1: "MLPW", u32 version=1, u32 activation, u32 L, u32 dims[L+1],
    then per layer f64 W row-major [out][in], f64 b[out]; little-endian."""
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    with open(path, "wb") as fh:
        fh.write(b"MLPW")
        fh.write(struct.pack("<III", 1, act, len(dims) - 1))
        fh.write(struct.pack("<%dI" % len(dims), *dims))
        for W, b in layers:
            fh.write(np.ascontiguousarray(W, dtype="<f8").tobytes())
            fh.write(np.ascontiguousarray(b, dtype="<f8").tobytes())


def read_mlpw_raw(path):
    """Plain reader for tests (returns act, dims, layers)."""
    data = Path(path).read_bytes()
    assert data[:4] == b"MLPW"
    ver, act, L = struct.unpack_from("<III", data, 4)
    dims = list(struct.unpack_from("<%dI" % (L + 1), data, 16))
    off = 16 + 4 * (L + 1)
    layers = []
    for li in range(L):
        n_w = dims[li + 1] * dims[li]
        W = np.frombuffer(data, "<f8", n_w, off).reshape(dims[li + 1], dims[li]); off += 8 * n_w
        b = np.frombuffer(data, "<f8", dims[li + 1], off); off += 8 * dims[li + 1]
        layers.append((W.copy(), b.copy()))
    return act, dims, layers


def weights_path(H: int, seed: int = 7, act: int = 1) -> str:
    """Deterministic weights file for hidden width H (generated on first use).  act = 2: the
    same random-init weights under the softplus activation (NEXT-4 variant, R26)."""
    # "_r2": recipe revision 2 (He-normal output row, R11); a stale cached file of
    # the round-1 recipe (output row N(0, 1/(5H))) is never picked up
    name = f"gcdf_H{H}_s{seed}_r2.mlpw" if act == 1 else f"gcdf_H{H}_s{seed}_r2_act{act}.mlpw"
    p = REPO / "build" / "inputs" / name
    if not p.exists():
        _, dims, layers = make_weights(H, seed)
        tmp = p.with_suffix(".tmp%d" % os.getpid())
        write_mlpw(tmp, act, dims, layers)
        os.replace(tmp, p)
    return str(p)

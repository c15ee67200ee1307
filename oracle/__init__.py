"""TEST INFRASTRUCTURE ONLY -- float64 CPU oracle of the GCDF hot path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this package.  It shares no code with paper_2601_18548_b200/ (the
CUDA path) and never imports it.  The arithmetic lives in gcdf_oracle.c (plain C,
float64, no BLAS, no -ffast-math, no FMA contraction); this file only marshals
numpy arrays.  See the header of gcdf_oracle.c for the step list and citations.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "gcdf_oracle.c"
_LIB = _HERE / "liboracle.so"

EMU_W = 1
EMU_A = 2
EMU_BF16 = EMU_W | EMU_A
TGRAD_QCHANNEL = 4
EMU_FP16_FLAG = 8
EMU_FP16 = EMU_W | EMU_A | EMU_FP16_FLAG
FRAME_SE2 = 16   # NEXT-4 variant: points rotated into the base frame (R24)

ERRORS = {0: "OK", -1: "INVALID", -2: "IO", -3: "BAD_MAGIC", -4: "VERSION", -5: "DIM_MISMATCH",
          -7: "CAPACITY", -12: "NOMEM"}


class OracleError(RuntimeError):
    def __init__(self, code, what=""):
        super().__init__(f"oracle {what}: {ERRORS.get(code, code)}")
        self.code = code
        self.name = ERRORS.get(code, str(code))


def build(force: bool = False) -> str:
    """gcc the oracle (the checker is built, not used, by __graft_entry__.build())."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(".so.tmp%d" % os.getpid())
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-pthread", "-o", str(tmp), str(_SRC), "-lm"])
        os.replace(tmp, _LIB)
    return str(_LIB)


_lib = None


def _L():
    global _lib
    if _lib is None:
        lib = C.CDLL(build())
        P, I64, D, I = C.c_void_p, C.c_int64, C.c_double, C.c_int
        lib.or_load.argtypes = [C.c_char_p, C.POINTER(P)]
        lib.or_free.argtypes = [P]
        lib.or_free.restype = None
        lib.or_info.argtypes = [P, C.POINTER(I), C.POINTER(I), C.POINTER(I)]
        lib.or_eval.argtypes = [P, P, I64, P, I64, I, P, P, P, P, I]
        lib.or_detect.argtypes = [P, P, P, I64, P, I64, I, D, D, P, P, P, P, I64, C.POINTER(I64),
                                  P, P, P, I]
        lib.or_sparse_jacobian.argtypes = [P, P, P, I64, D, P, P, P, P]
        lib.or_project.argtypes = [P, P, P, P, I64, I64, P]
        lib.or_detect_part.argtypes = [P, P, P, I64, P, I64, I, D, D, D, P, P, P, P, I64, C.POINTER(I64),
                                       P, P, P, P, I]
        lib.or_scene_new.argtypes = [I64, C.POINTER(P)]
        lib.or_scene_free.argtypes = [P]
        lib.or_scene_free.restype = None
        lib.or_scene_update.argtypes = [P, P, I64, P, P, I64]
        lib.or_scene_export.argtypes = [P, P, P]
        lib.or_scene_export.restype = I64
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class MLP:
    """O1: an MLPW v1 file loaded by the oracle's own parser."""

    def __init__(self, path):
        h = C.c_void_p()
        rc = _L().or_load(str(path).encode(), C.byref(h))
        if rc:
            raise OracleError(rc, f"load {path}")
        self._h = h
        act, L = C.c_int(), C.c_int()
        dims = (C.c_int * 17)()
        _L().or_info(h, C.byref(act), C.byref(L), dims)
        self.act, self.L = act.value, L.value
        self.dims = [dims[i] for i in range(self.L + 1)]

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.or_free(self._h)
            self._h = None

    def eval(self, pts, q, flags: int = 0, nthreads: int = 1, want_grad=True, want_kappa=False,
             want_hash=False):
        """pts [M,3], q [W,9] -> f [W,M] (+ g [W,M,9], kappa [W,M], mask_hash [W,M])."""
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        q = np.ascontiguousarray(q, dtype=np.float64).reshape(-1, 9)
        M, W = pts.shape[0], q.shape[0]
        f = np.empty((W, M))
        g = np.empty((W, M, 9)) if want_grad else None
        k = np.empty((W, M)) if want_kappa else None
        hsh = np.empty((W, M), dtype=np.uint64) if want_hash else None
        rc = _L().or_eval(self._h, _p(pts), M, _p(q), W, flags, _p(f), _p(g), _p(k), _p(hsh),
                          int(nthreads))
        if rc:
            raise OracleError(rc, "eval")
        out = {"f": f}
        if want_grad:
            out["g"] = g
        if want_kappa:
            out["kappa"] = k
        if want_hash:
            out["mask_hash"] = hsh
        return out

    def detect(self, pts, ids, q, delta, tau, flags: int = 0, cap=None, nthreads: int = 1, radius: float = 0.0):
        """O6-O7 over the live scene (ids ascending) and W = B*N waypoint rows; radius > 0
        restricts step i to its range partition I_{M,i} (NEXT-1, gcdf_oracle.c)."""
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        q = np.ascontiguousarray(q, dtype=np.float64).reshape(-1, 9)
        M, W = pts.shape[0], q.shape[0]
        if cap is None:
            cap = W * M
        cap = max(int(cap), 1)
        rf = np.empty(cap)
        rg = np.empty((cap, 9))
        rwp = np.empty(cap, dtype=np.int64)
        rpt = np.empty(cap, dtype=np.int64)
        cnt = C.c_int64()
        off = np.empty(W + 1, dtype=np.int64)
        wmin = np.empty(W)
        warg = np.empty(W, dtype=np.int64)
        psz = np.empty(W, dtype=np.int64)
        rc = _L().or_detect_part(self._h, _p(pts), _p(ids), M, _p(q), W, flags, float(radius), float(delta),
                                 float(tau), _p(rf), _p(rg), _p(rwp), _p(rpt), cap, C.byref(cnt), _p(off),
                                 _p(wmin), _p(warg), _p(psz), int(nthreads))
        if rc:
            raise OracleError(rc, "detect")
        n = cnt.value
        s = min(n, cap)
        return {"count": n, "value": rf[:s], "grad": rg[:s], "wp": rwp[:s], "pt": rpt[:s],
                "wp_offsets": off, "wp_min": wmin, "wp_argmin": warg, "part_sizes": psz}


def project(f, g, q, minv):
    """NEXT-3 (Theorem 1.2): q_z = q - f M^{-1} grad_q f for f [W, M], g [W, M, 9], q [W, 9],
    minv [9] (the diagonal of M^{-1})."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    W, M = f.shape
    g = np.ascontiguousarray(g, dtype=np.float64).reshape(W, M, 9)
    q = np.ascontiguousarray(q, dtype=np.float64).reshape(W, 9)
    minv = np.ascontiguousarray(minv, dtype=np.float64).reshape(9)
    qz = np.empty((W, M, 9))
    rc = _L().or_project(_p(f), _p(g), _p(q), _p(minv), W, M, _p(qz))
    if rc:
        raise OracleError(rc, "project")
    return qz


def sparse_jacobian(rec: dict, delta: float):
    """NEXT-2 (Eq. 14-19): constraint vector c = f - delta and the CSR sparse Jacobian of
    the active records (rec: value [K], grad [K, 9], wp [K] in (wp, pt) order)."""
    f = np.ascontiguousarray(rec["value"], dtype=np.float64)
    g = np.ascontiguousarray(rec["grad"], dtype=np.float64).reshape(-1, 9)
    wp = np.ascontiguousarray(rec["wp"], dtype=np.int64)
    K = f.shape[0]
    c = np.empty(K)
    row_ptr = np.empty(K + 1, dtype=np.int64)
    col = np.empty(K * 9, dtype=np.int64)
    val = np.empty(K * 9)
    rc = _L().or_sparse_jacobian(_p(f), _p(g), _p(wp), K, float(delta), _p(c), _p(row_ptr), _p(col), _p(val))
    if rc:
        raise OracleError(rc, "sparse_jacobian")
    return {"c": c, "row_ptr": row_ptr, "col": col, "val": val}


class Scene:
    """O2: the oracle's own id -> xyz map, replaying gcdf_update_scene's id rule."""

    def __init__(self, capacity: int):
        h = C.c_void_p()
        rc = _L().or_scene_new(int(capacity), C.byref(h))
        if rc:
            raise OracleError(rc, "scene")
        self._h = h
        self.capacity = int(capacity)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.or_scene_free(self._h)
            self._h = None

    def update(self, add_xyz=None, remove_ids=None):
        add = np.ascontiguousarray(np.zeros((0, 3)) if add_xyz is None else add_xyz,
                                   dtype=np.float32).reshape(-1, 3)
        rem = np.ascontiguousarray(np.zeros(0) if remove_ids is None else remove_ids, dtype=np.int64)
        out = np.empty(add.shape[0], dtype=np.int64)
        rc = _L().or_scene_update(self._h, _p(add), add.shape[0], _p(out), _p(rem), rem.shape[0])
        if rc:
            raise OracleError(rc, "scene update")
        return out

    def export(self):
        n = _L().or_scene_export(self._h, None, None)
        ids = np.empty(n, dtype=np.int64)
        xyz = np.empty((n, 3))
        _L().or_scene_export(self._h, _p(ids), _p(xyz))
        return ids, xyz

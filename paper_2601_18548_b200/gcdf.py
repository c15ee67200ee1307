"""Thin ctypes binding of libgcdf (include/gcdf.h).  Argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; torch supplies device
memory (output tensors, the workspace) and the current CUDA stream.  There is no CPU
path: if libgcdf.so is missing or no B200 is present, construction raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np
import torch

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libgcdf.so"  # the in-tree build (python -m paper_2601_18548_b200.build); no override

FP32, BF16, FP16, FP16X3, BF16X3 = 0, 1, 2, 3, 4  # FP16X3 / BF16X3: 3-term split tensor-core paths (R25, R29)
TGRAD_CHAINRULE, TGRAD_QCHANNEL = 0, 1
FRAME_TRANSLATE, FRAME_SE2 = 0, 1  # gcdf_frame (include/gcdf.h; R24)
STATUS = {0: "OK", -1: "INVALID_ARG", -2: "IO", -3: "BAD_MAGIC", -4: "VERSION", -5: "DIM_MISMATCH",
          -6: "NOT_LOADED", -7: "CAPACITY", -8: "UNKNOWN_ID", -9: "NONFINITE", -10: "CUDA",
          -11: "UNSUPPORTED", -12: "NCCL"}
REC_BYTES = 48  # sizeof(gcdf_active_t)

EXPORTED = ["gcdf_default_options", "gcdf_create", "gcdf_destroy", "gcdf_last_error", "gcdf_has_tcgen05",
            "gcdf_workspace_bytes", "gcdf_bind_workspace", "gcdf_load_weights", "gcdf_update_scene",
            "gcdf_scene_info", "gcdf_pairgen_transform", "gcdf_query_values_grads", "gcdf_detect_active_set",
            "gcdf_detect_active_set_partitioned", "gcdf_detect_active_set_host", "gcdf_sparse_jacobian",
            "gcdf_project_dense", "gcdf_graph_create_detect", "gcdf_graph_launch", "gcdf_graph_destroy", "gcdf_compact_dense", "gcdf_merge_active_sets", "gcdf_launch_count", "gcdf_profile_enable",
            "gcdf_profile_read", "gcdf_profile_read_exchange", "gcdf_selftest_umma", "gcdf_debug_trace",
            "gcdf_nccl_unique_id", "gcdf_dist_init", "gcdf_dist_init_host", "gcdf_dist_info",
            "gcdf_broadcast_waypoints"]
COMM_KINDS = {0: "none", 1: "nccl", 2: "host"}
# gcdf_host_allgather_fn (include/gcdf.h): the test backend's blocking host all-gather
HOST_ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)


class GcdfError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = code
        self.name = STATUS.get(code, str(code))
        super().__init__(f"gcdf {self.name}: {msg}")


class Options(C.Structure):
    _fields_ = [("precision", C.c_int32), ("tgrad_mode", C.c_int32), ("scene_capacity", C.c_int64),
                ("max_waypoints", C.c_int32), ("max_active", C.c_int64), ("rank", C.c_int32),
                ("world", C.c_int32), ("max_candidates", C.c_int64), ("frame", C.c_int32), ("exchange", C.c_int32)]


_lib = None


def load_library(path: str | Path = LIB_PATH):
    """Load libgcdf.so (raises if it has not been built: no fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not Path(path).exists():
        raise ImportError(f"{path} not built: run `python -m paper_2601_18548_b200.build` (nvcc, sm_100a)")
    lib = C.CDLL(str(path))
    P, I32, I64, F = C.c_void_p, C.c_int32, C.c_int64, C.c_float
    PI64 = C.POINTER(C.c_int64)
    lib.gcdf_default_options.argtypes = [C.POINTER(Options)]
    lib.gcdf_default_options.restype = None
    lib.gcdf_create.argtypes = [C.c_int, C.POINTER(Options), C.POINTER(P)]
    lib.gcdf_destroy.argtypes = [P]
    lib.gcdf_last_error.argtypes = [P]
    lib.gcdf_last_error.restype = C.c_char_p
    lib.gcdf_has_tcgen05.argtypes = []
    lib.gcdf_workspace_bytes.argtypes = [P, PI64]
    lib.gcdf_bind_workspace.argtypes = [P, P, I64]
    lib.gcdf_load_weights.argtypes = [P, C.c_char_p, P]
    lib.gcdf_update_scene.argtypes = [P, P, I64, P, P, I64, P]
    lib.gcdf_scene_info.argtypes = [P, PI64, PI64, PI64]
    lib.gcdf_pairgen_transform.argtypes = [P, P, I32, I32, P, P]
    lib.gcdf_query_values_grads.argtypes = [P, P, I32, I32, P, P, P]
    lib.gcdf_detect_active_set.argtypes = [P, P, I32, I32, F, F, P, I64, P, P, P, P, P, P, P]
    lib.gcdf_detect_active_set_host.argtypes = [P, P, I32, I32, F, F, P, I64, P, P, P, P, P]
    lib.gcdf_sparse_jacobian.argtypes = [P, P, P, I64, F, P, P, P, P, P]
    lib.gcdf_project_dense.argtypes = [P, P, I32, I32, P, P, P, P]
    lib.gcdf_graph_create_detect.argtypes = [P, P, I32, I32, F, F, F, P, I64, P, P, P, P, P, P, C.POINTER(P)]
    lib.gcdf_graph_launch.argtypes = [P, P, P]
    lib.gcdf_graph_destroy.argtypes = [P]
    lib.gcdf_detect_active_set_partitioned.argtypes = [P, P, I32, I32, F, F, F, P, I64, P, P, P, P, P, P, P, P]
    lib.gcdf_compact_dense.argtypes = [P, P, P, I32, I64, F, F, P, I64, P, P, P, P, P, P, P]
    lib.gcdf_merge_active_sets.argtypes = [P, I32, I32, P, I64, P, P, P, I64, P, P, P, P, P]
    lib.gcdf_launch_count.argtypes = [P]
    lib.gcdf_launch_count.restype = I64
    lib.gcdf_profile_enable.argtypes = [P, C.c_int]
    lib.gcdf_profile_read.argtypes = [P, C.POINTER(C.c_double), PI64, C.c_int]
    lib.gcdf_profile_read_exchange.argtypes = [P, C.POINTER(C.c_double), PI64, C.c_int]
    lib.gcdf_nccl_unique_id.argtypes = [C.c_char_p]
    lib.gcdf_dist_init.argtypes = [P, C.c_char_p, I32, I32]
    lib.gcdf_dist_init_host.argtypes = [P, HOST_ALLGATHER_FN, P]
    lib.gcdf_dist_info.argtypes = [P, C.POINTER(I32), C.POINTER(I32)]
    lib.gcdf_broadcast_waypoints.argtypes = [P, P, I32, I32, P]
    lib.gcdf_selftest_umma.argtypes = [C.c_int, C.c_int, P, P, P, P]
    lib.gcdf_debug_trace.argtypes = [P, P]
    _lib = lib
    return lib


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(device):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class DetectGraph:
    """A captured detect (gcdf_graph_*); keeps its q and output tensors alive."""

    def __init__(self, ctx: "Context", q: torch.Tensor, delta: float, tau: float, radius: float = 0.0,
                 capacity: int | None = None):
        q0 = q
        q, B, N = ctx._q(q)
        if q.data_ptr() != q0.data_ptr():
            # the graph replays with the captured pointer: a private copy (dtype / device /
            # layout conversion) would make refills of the caller's tensor invisible
            raise ValueError("DetectGraph: q must be a contiguous float32 [B, N, 9] tensor on the context's device")
        self.ctx, self.q = ctx, q
        self.outputs = ctx.alloc_detect_outputs(B * N, capacity if capacity is not None else ctx.max_active)
        o = self.outputs
        o["part_sizes"] = torch.empty(B * N, dtype=torch.int64, device=ctx.device) if radius > 0 else None
        h = C.c_void_p()
        ctx._check(ctx.lib.gcdf_graph_create_detect(
            ctx._h, _ptr(q), B, N, float(radius), float(delta), float(tau), _ptr(o["records"]), int(o["capacity"]),
            _ptr(o["wp_offsets"]), _ptr(o["wp_min"]), _ptr(o["wp_argmin"]), _ptr(o["wp_key"]), _ptr(o["part_sizes"]),
            _ptr(o["count"]), C.byref(h)))
        self._g = h

    def launch(self, sync_count: bool = True):
        nh = C.c_int64(-1)
        self.ctx._check(self.ctx.lib.gcdf_graph_launch(self._g, C.byref(nh) if sync_count else None,
                                                       _stream(self.ctx.device)))
        if sync_count:
            self.outputs["n"] = nh.value
        return self.outputs

    def close(self):
        if getattr(self, "_g", None) is not None and _lib is not None:
            _lib.gcdf_graph_destroy(self._g)
            self._g = None

    def __del__(self):
        self.close()


def records_to_dict(rec: torch.Tensor, n: int) -> dict:
    """View [n] gcdf_active_t records (uint8 [cap, 48]) as value / grad / wp / pt tensors."""
    r = rec[:n].view(torch.int32).view(n, 12) if n > 0 else rec.new_zeros((0, 12), dtype=torch.int32)
    f = r.view(torch.float32)
    return {"value": f[:, 0], "grad": f[:, 1:10], "wp": r[:, 10].to(torch.int64) & 0xFFFFFFFF,
            "pt": r[:, 11].to(torch.int64) & 0xFFFFFFFF}


def selftest_umma(mode: int, A: torch.Tensor, B: torch.Tensor) -> torch.Tensor:
    """Diagnostics: one tcgen05 UMMA block (see gcdf_selftest_umma)."""
    lib = load_library()
    A = A.to(torch.float32).contiguous()
    B = B.to(device=A.device, dtype=torch.float32).contiguous()
    D = torch.zeros((128, 128), dtype=torch.float32, device=A.device)
    rc = lib.gcdf_selftest_umma(A.device.index or 0, mode, _ptr(A), _ptr(B), _ptr(D), _stream(A.device))
    if rc:
        raise GcdfError(rc, "selftest_umma")
    return D


class Context:
    """One libgcdf context on one CUDA device (one rank)."""

    def __init__(self, device: int = 0, precision: int = FP16, tgrad_mode: int = TGRAD_CHAINRULE,
                 scene_capacity: int = 1 << 20, max_waypoints: int = 256, max_active: int = 1 << 22,
                 rank: int = 0, world: int = 1, max_candidates: int = 0, frame: int = 0, exchange: bool = False):
        self.lib = load_library()
        if not torch.cuda.is_available():
            raise RuntimeError("libgcdf needs a CUDA device (B200); no CPU path exists")
        self.device = torch.device("cuda", device)
        o = Options()
        self.lib.gcdf_default_options(C.byref(o))
        o.precision, o.tgrad_mode, o.scene_capacity = precision, tgrad_mode, scene_capacity
        o.max_waypoints, o.max_active, o.rank, o.world = max_waypoints, max_active, rank, world
        o.max_candidates, o.frame, o.exchange = max_candidates, frame, int(exchange)
        self.opts = o
        h = C.c_void_p()
        rc = self.lib.gcdf_create(device, C.byref(o), C.byref(h))
        if rc:
            raise GcdfError(rc, "gcdf_create failed (needs an sm_100 device; bf16 needs the tcgen05 build)")
        self._h = h
        nb = C.c_int64()
        self._check(self.lib.gcdf_workspace_bytes(h, C.byref(nb)))
        self.workspace = torch.empty(int(nb.value), dtype=torch.uint8, device=self.device)
        self._check(self.lib.gcdf_bind_workspace(h, _ptr(self.workspace), int(nb.value)))
        self.max_active = max_active
        self.rank, self.world = rank, world

    def close(self):
        """Destroy the library context and release its workspace (idempotent)."""
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            try:  # (at interpreter shutdown torch.cuda may already be torn down)
                torch.cuda.synchronize(self.device)
            except Exception:
                pass
            _lib.gcdf_destroy(h)
            self._h = None
        self.workspace = None

    def __del__(self):
        self.close()

    def _check(self, rc):
        if rc:
            raise GcdfError(rc, self.lib.gcdf_last_error(self._h).decode(errors="replace"))
        return rc

    @property
    def launches(self) -> int:
        return int(self.lib.gcdf_launch_count(self._h))

    def debug_trace(self, buf: torch.Tensor | None) -> None:
        """Diagnostics: pipeline clock64 trace of CTA 0 (int64 [18*4*13*4] on the device) or None."""
        self._check(self.lib.gcdf_debug_trace(self._h, _ptr(buf)))

    def profile_enable(self, on: bool = True) -> None:
        self._check(self.lib.gcdf_profile_enable(self._h, int(on)))

    def profile_read(self, reset: bool = True):
        ms, n = C.c_double(), C.c_int64()
        self._check(self.lib.gcdf_profile_read(self._h, C.byref(ms), C.byref(n), int(reset)))
        return ms.value, n.value

    def profile_read_exchange(self, reset: bool = True):
        ms, n = C.c_double(), C.c_int64()
        self._check(self.lib.gcdf_profile_read_exchange(self._h, C.byref(ms), C.byref(n), int(reset)))
        return ms.value, n.value

    # -------------------------------------------------------------- sharded scene
    def dist_init(self, group=None) -> None:
        """NCCL communicator of the sharded detect (gcdf_dist_init): rank 0 draws the NCCL
        unique id in the library, the 128 bytes travel through the torch.distributed group
        (plumbing), every rank creates its communicator."""
        import torch.distributed as dist
        buf = C.create_string_buffer(128)
        if self.rank == 0:
            rc = self.lib.gcdf_nccl_unique_id(buf)
            if rc:
                raise GcdfError(rc, "gcdf_nccl_unique_id")
        obj = [buf.raw if self.rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        self._check(self.lib.gcdf_dist_init(self._h, obj[0], self.rank, self.world))

    def dist_init_local_nccl(self) -> None:
        """world == 1 with the exchange buffers (exchange=True): a one-rank NCCL communicator,
        so the whole exchange path (all-gather group + merge kernel) runs on one GPU."""
        buf = C.create_string_buffer(128)
        rc = self.lib.gcdf_nccl_unique_id(buf)
        if rc:
            raise GcdfError(rc, "gcdf_nccl_unique_id")
        self._check(self.lib.gcdf_dist_init(self._h, buf.raw, self.rank, self.world))

    def dist_init_host(self, allgather) -> None:
        """TEST BACKEND (gcdf_dist_init_host): allgather(send: bytes-like numpy uint8 [n],
        recv: numpy uint8 [world * n]) -> None, a blocking host all-gather (e.g. gloo)."""
        world = self.world

        def _cb(send, recv, nbytes, user):
            try:
                s = np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_uint8)), shape=(max(int(nbytes), 1),))
                r = np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_uint8)), shape=(max(world * int(nbytes), 1),))
                allgather(s[: int(nbytes)], r[: world * int(nbytes)])
                return 0
            except Exception:  # noqa: BLE001 -- reported to the library as a failed exchange
                import traceback
                traceback.print_exc()
                return 1
        self._host_cb = HOST_ALLGATHER_FN(_cb)  # kept alive with the context
        self._check(self.lib.gcdf_dist_init_host(self._h, self._host_cb, None))

    def broadcast_waypoints(self, q: torch.Tensor) -> torch.Tensor:
        """gcdf_broadcast_waypoints: rank 0's waypoints to every rank, in place (q: [B, N, 9]
        float32 contiguous on this context's device)."""
        if q.dtype != torch.float32 or not q.is_contiguous() or q.device != self.device or q.dim() != 3:
            raise ValueError("broadcast_waypoints: q must be a contiguous float32 [B, N, 9] tensor on the context's device")
        self._check(self.lib.gcdf_broadcast_waypoints(self._h, C.c_void_p(q.data_ptr()), int(q.shape[0]),
                                                      int(q.shape[1]), _stream(self.device)))
        return q

    def dist_info(self):
        k, v = C.c_int32(), C.c_int32()
        self._check(self.lib.gcdf_dist_info(self._h, C.byref(k), C.byref(v)))
        return {"kind": COMM_KINDS.get(k.value, k.value), "nccl_version": v.value}

    # -------------------------------------------------------------- weights / scene
    def load_weights(self, path) -> None:
        self._check(self.lib.gcdf_load_weights(self._h, str(path).encode(), _stream(self.device)))

    def update_scene(self, add_xyz=None, remove_ids=None) -> np.ndarray:
        add = np.ascontiguousarray(np.zeros((0, 3)) if add_xyz is None else add_xyz, dtype=np.float32).reshape(-1, 3)
        rem = np.ascontiguousarray(np.zeros(0) if remove_ids is None else remove_ids, dtype=np.int64).ravel()
        ids = np.empty(add.shape[0], dtype=np.int64)
        self._check(self.lib.gcdf_update_scene(self._h, add.ctypes.data_as(C.c_void_p), add.shape[0],
                                               ids.ctypes.data_as(C.c_void_p), rem.ctypes.data_as(C.c_void_p),
                                               rem.shape[0], _stream(self.device)))
        return ids

    def scene_info(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(self.lib.gcdf_scene_info(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return {"n_live": a.value, "id_bound": b.value, "local_bound": c.value}

    def local_to_global(self, slots: torch.Tensor) -> torch.Tensor:
        return ((slots // 128) * self.world + self.rank) * 128 + slots % 128

    # -------------------------------------------------------------- hot path
    def _q(self, q: torch.Tensor):
        if q.dim() != 3 or q.shape[2] != 9:
            raise ValueError("q must be [B, N, 9]")
        q = q.to(device=self.device, dtype=torch.float32).contiguous()
        return q, int(q.shape[0]), int(q.shape[1])

    def pairgen_transform(self, q: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        q, B, N = self._q(q)
        lb = self.scene_info()["local_bound"]
        if out is None:
            out = torch.empty((B * N, lb, 4), dtype=torch.float32, device=self.device)
        self._check(self.lib.gcdf_pairgen_transform(self._h, _ptr(q), B, N, _ptr(out), _stream(self.device)))
        return out

    def query_values_grads(self, q: torch.Tensor, want_grads: bool = True, values=None, grads=None):
        q, B, N = self._q(q)
        lb = self.scene_info()["local_bound"]
        if values is None:
            values = torch.empty((B * N, lb), dtype=torch.float32, device=self.device)
        if want_grads and grads is None:
            grads = torch.empty((B * N, lb, 9), dtype=torch.float32, device=self.device)
        self._check(self.lib.gcdf_query_values_grads(self._h, _ptr(q), B, N, _ptr(values),
                                                     _ptr(grads) if want_grads else None, _stream(self.device)))
        return values, (grads if want_grads else None)

    def alloc_detect_outputs(self, n_wp: int, capacity: int):
        d = self.device
        return {"records": torch.empty((max(capacity, 1), REC_BYTES), dtype=torch.uint8, device=d),
                "wp_offsets": torch.empty(n_wp + 1, dtype=torch.int64, device=d),
                "wp_min": torch.empty(n_wp, dtype=torch.float32, device=d),
                "wp_argmin": torch.empty(n_wp, dtype=torch.int64, device=d),
                "wp_key": torch.empty(n_wp, dtype=torch.int64, device=d),
                "count": torch.empty(1, dtype=torch.int64, device=d), "capacity": capacity}

    def detect_active_set(self, q: torch.Tensor, delta: float, tau: float, capacity: int | None = None,
                          outputs: dict | None = None, sync_count: bool = True):
        """Fused detect.  Returns the output dict (+ 'n' = host count when sync_count)."""
        q, B, N = self._q(q)
        if outputs is None:
            outputs = self.alloc_detect_outputs(B * N, capacity if capacity is not None else self.max_active)
        o = outputs
        nh = C.c_int64(-1)
        self._check(self.lib.gcdf_detect_active_set(
            self._h, _ptr(q), B, N, float(delta), float(tau), _ptr(o["records"]), int(o["capacity"]),
            _ptr(o["wp_offsets"]), _ptr(o["wp_min"]), _ptr(o["wp_argmin"]), _ptr(o["wp_key"]), _ptr(o["count"]),
            C.byref(nh) if sync_count else None, _stream(self.device)))
        if sync_count:
            o["n"] = nh.value
        return o

    def detect_active_set_partitioned(self, q: torch.Tensor, radius: float, delta: float, tau: float,
                                      capacity: int | None = None, outputs: dict | None = None,
                                      sync_count: bool = True, part_sizes: bool = True):
        """NEXT-1 range-partitioned fused detect (pairs within `radius` of each step's base
        only).  Returns the output dict (+ 'n' when sync_count, + 'part_sizes' [B*N])."""
        q, B, N = self._q(q)
        if outputs is None:
            outputs = self.alloc_detect_outputs(B * N, capacity if capacity is not None else self.max_active)
        o = outputs
        if part_sizes and o.get("part_sizes") is None:
            o["part_sizes"] = torch.empty(B * N, dtype=torch.int64, device=self.device)
        nh = C.c_int64(-1)
        self._check(self.lib.gcdf_detect_active_set_partitioned(
            self._h, _ptr(q), B, N, float(radius), float(delta), float(tau), _ptr(o["records"]), int(o["capacity"]),
            _ptr(o["wp_offsets"]), _ptr(o["wp_min"]), _ptr(o["wp_argmin"]), _ptr(o["wp_key"]),
            _ptr(o.get("part_sizes")) if part_sizes else None, _ptr(o["count"]),
            C.byref(nh) if sync_count else None, _stream(self.device)))
        if sync_count:
            o["n"] = nh.value
        return o

    def detect_graph(self, q: torch.Tensor, delta: float, tau: float, radius: float = 0.0,
                     capacity: int | None = None):
        """CUDA-graph form of detect (radius > 0: range-partitioned): returns a DetectGraph
        whose launch() replays the captured call chain (refill q in place between launches)."""
        return DetectGraph(self, q, delta, tau, radius, capacity)

    def project_dense(self, q: torch.Tensor, minv_diag):
        """NEXT-3: values [B*N, lb] and q_z = q - f M^{-1} grad f [B*N, lb, 9] for every pair."""
        q, B, N = self._q(q)
        lb = self.scene_info()["local_bound"]
        values = torch.empty((B * N, lb), dtype=torch.float32, device=self.device)
        qz = torch.empty((B * N, lb, 9), dtype=torch.float32, device=self.device)
        m = (C.c_float * 9)(*[float(x) for x in np.asarray(minv_diag, dtype=np.float64).ravel()])
        self._check(self.lib.gcdf_project_dense(self._h, _ptr(q), B, N, m, _ptr(values), _ptr(qz),
                                                _stream(self.device)))
        return values, qz

    def sparse_jacobian(self, outputs: dict, delta: float):
        """NEXT-2: constraint vector c = f - delta and the CSR Jacobian (Eq. 14-19) of a detect
        result (records in (wp, pt) order; the count is read on the device)."""
        cap = int(outputs["capacity"])
        d = self.device
        r = {"c": torch.empty(cap, dtype=torch.float32, device=d),
             "row_ptr": torch.empty(cap + 1, dtype=torch.int64, device=d),
             "col": torch.empty(cap * 9, dtype=torch.int32, device=d),
             "val": torch.empty(cap * 9, dtype=torch.float32, device=d)}
        self._check(self.lib.gcdf_sparse_jacobian(self._h, _ptr(outputs["records"]), _ptr(outputs["count"]), cap,
                                                  float(delta), _ptr(r["c"]), _ptr(r["row_ptr"]), _ptr(r["col"]),
                                                  _ptr(r["val"]), _stream(d)))
        return r

    @staticmethod
    def alloc_host_outputs(n_wp: int, capacity: int, pinned: bool = True):
        """Host (page-locked by default) buffers for detect_active_set_host."""
        def e(shape, dt):
            t = torch.empty(shape, dtype=dt)
            return t.pin_memory() if pinned else t
        return {"records": e((max(capacity, 1), REC_BYTES), torch.uint8), "wp_offsets": e(n_wp + 1, torch.int64),
                "wp_min": e(n_wp, torch.float32), "wp_argmin": e(n_wp, torch.int64), "capacity": capacity}

    def detect_active_set_host(self, q_host: torch.Tensor, delta: float, tau: float, outputs: dict):
        """End-to-end fused detect through the host-buffer C-ABI call (q and results in host
        memory; the library does the copies).  Returns outputs with 'n' = active count."""
        if q_host.device.type != "cpu" or q_host.dim() != 3 or q_host.shape[2] != 9:
            raise ValueError("q_host must be a CPU tensor [B, N, 9]")
        q_host = q_host.to(torch.float32).contiguous()
        o = outputs
        nh = C.c_int64(-1)
        self._check(self.lib.gcdf_detect_active_set_host(
            self._h, C.c_void_p(q_host.data_ptr()), int(q_host.shape[0]), int(q_host.shape[1]), float(delta),
            float(tau), C.c_void_p(o["records"].data_ptr()), int(o["capacity"]), C.c_void_p(o["wp_offsets"].data_ptr()),
            C.c_void_p(o["wp_min"].data_ptr()), C.c_void_p(o["wp_argmin"].data_ptr()), C.byref(nh),
            _stream(self.device)))
        o["n"] = nh.value
        return o

    def compact_dense(self, values: torch.Tensor, grads: torch.Tensor, delta: float, tau: float,
                      capacity: int | None = None, outputs: dict | None = None, sync_count: bool = True):
        n_wp, stride = int(values.shape[0]), int(values.shape[1])
        if outputs is None:
            outputs = self.alloc_detect_outputs(n_wp, capacity if capacity is not None else self.max_active)
        o = outputs
        nh = C.c_int64(-1)
        self._check(self.lib.gcdf_compact_dense(
            self._h, _ptr(values), _ptr(grads), n_wp, stride, float(delta), float(tau), _ptr(o["records"]),
            int(o["capacity"]), _ptr(o["wp_offsets"]), _ptr(o["wp_min"]), _ptr(o["wp_argmin"]), _ptr(o["wp_key"]),
            _ptr(o["count"]), C.byref(nh) if sync_count else None, _stream(self.device)))
        if sync_count:
            o["n"] = nh.value
        return o

    def merge_active_sets(self, world: int, n_wp: int, recs: torch.Tensor, rec_stride: int,
                          offsets: torch.Tensor, wp_key: torch.Tensor, capacity: int):
        o = self.alloc_detect_outputs(n_wp, capacity)
        self._check(self.lib.gcdf_merge_active_sets(
            self._h, world, n_wp, _ptr(recs), rec_stride, _ptr(offsets), _ptr(wp_key), _ptr(o["records"]),
            capacity, _ptr(o["wp_offsets"]), _ptr(o["wp_min"]), _ptr(o["wp_argmin"]), _ptr(o["count"]),
            _stream(self.device)))
        o["wp_key"] = wp_key
        return o

"""CPU checks of the C-ABI library: it loads and exports every symbol include/gcdf.h
declares; host-only entry points behave without a GPU (no compute calls here)."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def lib():
    from paper_2601_18548_b200 import build
    build.build()
    from paper_2601_18548_b200 import gcdf
    return gcdf.load_library()


def test_exports_every_declared_symbol(lib):
    hdr = (ROOT / "include" / "gcdf.h").read_text()
    declared = set(re.findall(r"^(?:int|void|int64_t|const char)\s*\*?\s*(gcdf_[a-z0-9_]+)\s*\(", hdr, re.M))
    assert "gcdf_detect_active_set" in declared and len(declared) >= 15
    for name in sorted(declared):
        assert hasattr(lib, name), name
    from paper_2601_18548_b200 import gcdf
    assert set(gcdf.EXPORTED) == declared


def test_default_options_and_struct_layout(lib):
    from paper_2601_18548_b200.gcdf import Options
    o = Options()
    lib.gcdf_default_options(C.byref(o))
    assert (o.precision, o.tgrad_mode, o.world, o.rank) == (2, 0, 1, 0)
    assert o.scene_capacity == 1 << 20 and o.max_waypoints == 256 and o.max_active == 1 << 22
    assert o.max_candidates == 0 and o.frame == 0 and o.exchange == 0
    assert C.sizeof(Options) == 56  # int32, int32, int64, int32 (+4), int64, int32, int32, int64, int32, int32


def test_create_without_gpu_fails_cleanly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2601_18548_b200.gcdf import Options
    h = C.c_void_p()
    rc = lib.gcdf_create(0, None, C.byref(h))
    assert rc == -11 and not h.value  # UNSUPPORTED, nothing allocated
    assert lib.gcdf_destroy(None) == 0
    # invalid options are rejected before any CUDA call
    o = Options()
    lib.gcdf_default_options(C.byref(o))
    o.world, o.rank = 2, 2
    assert lib.gcdf_create(0, C.byref(o), C.byref(h)) == -1
    # frame: only TRANSLATE / SE2, and SE2 has no q^t channel (R24)
    lib.gcdf_default_options(C.byref(o))
    o.frame = 2
    assert lib.gcdf_create(0, C.byref(o), C.byref(h)) == -1
    o.frame, o.tgrad_mode = 1, 1
    assert lib.gcdf_create(0, C.byref(o), C.byref(h)) == -1
    # capacity bounds: int32 local slots / ~0u sentinel; waypoints on gridDim.y
    lib.gcdf_default_options(C.byref(o))
    o.scene_capacity = 1 << 31
    assert lib.gcdf_create(0, C.byref(o), C.byref(h)) == -1
    lib.gcdf_default_options(C.byref(o))
    o.max_waypoints = 65536
    assert lib.gcdf_create(0, C.byref(o), C.byref(h)) == -1
    assert not h.value


def test_nccl_unique_id_host_only(lib):
    """gcdf_nccl_unique_id opens the process's NCCL at run time (dlopen libnccl.so.2) and
    draws a 128-byte id -- host-only work (bootstrap socket), no GPU needed."""
    import torch  # noqa: F401  (loads torch's NCCL first, as in the product processes)
    a, b = C.create_string_buffer(128), C.create_string_buffer(128)
    assert lib.gcdf_nccl_unique_id(a) == 0 and lib.gcdf_nccl_unique_id(b) == 0
    assert a.raw != bytes(128) and a.raw != b.raw
    assert lib.gcdf_nccl_unique_id(None) == -1


def test_binding_refuses_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2601_18548_b200 import Context
    with pytest.raises(RuntimeError):
        Context(0, precision=0)


def test_sm100a_only_cubin():
    """The library carries sm_100a SASS (and no other arch)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          str(ROOT / "paper_2601_18548_b200" / "libgcdf.so")],
                         capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_\d+a?", out))
    assert arches == {"sm_100a"}, arches

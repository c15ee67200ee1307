"""paper_2601_18548_b200 -- B200-native batched neural GCDF query + active-set detection.

The product is libgcdf.so (C ABI, include/gcdf.h) built from csrc/ for sm_100a; this
package holds it and a thin ctypes binding (gcdf.py).  Multi-GPU gather helpers live in
dist.py.  Nothing here computes any step of the hot path on the CPU.
"""
from .gcdf import (BF16, BF16X3, FP16, FP16X3, FP32, FRAME_SE2, FRAME_TRANSLATE, TGRAD_CHAINRULE, TGRAD_QCHANNEL, Context, GcdfError, load_library,
                   records_to_dict)

__all__ = ["BF16", "BF16X3", "FP16", "FP16X3", "FP32", "FRAME_SE2", "FRAME_TRANSLATE", "TGRAD_CHAINRULE", "TGRAD_QCHANNEL", "Context", "GcdfError", "load_library",
           "records_to_dict"]

"""Dev tool: build variants of libgcdf.so with build-time switches of k_mlp_tc.cu.

    python tools/variants.py NAME -DGCDF_TC_GREEDY=1 ... -> build/var/NAME/libgcdf.so
Run a variant on the GPU box by copying it over the snapshot's paper_2601_18548_b200/libgcdf.so
inside the gpurun command (the binding loads only the in-tree library; the default build here
is untouched).
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2601_18548_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
B.build()
out = ROOT / "build" / "var" / name
out.mkdir(parents=True, exist_ok=True)
obj = out / "k_mlp_tc.cu.o"
subprocess.check_call([B.NVCC, *B.ARCH, *B.FLAGS, *defs, "-c", str(B.CSRC / "k_mlp_tc.cu"), "-o", str(obj)])
objs = [str(obj) if o.name == "k_mlp_tc.cu.o" else str(o) for o in sorted(B.OBJ.glob("*.o"))]
subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", str(out / "libgcdf.so"), *objs])
print(out / "libgcdf.so")

"""Diagnostics: tcgen05 UMMA throughput on this B200 (one CTA, 200 x 8 back-to-back MMAs).

The probe kernels live in tools/probes/umma_probes.cu, built here into
build/probes/libumma_probes.so (not part of libgcdf.so)."""
import ctypes
import subprocess
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "tools" / "probes" / "umma_probes.cu"
LIB = ROOT / "build" / "probes" / "libumma_probes.so"
LIB.parent.mkdir(parents=True, exist_ok=True)
if not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-O3", "-Xcompiler",
                           "-fPIC", "-shared", "-I", str(ROOT / "include"), "-o", str(LIB), str(SRC)])
_probe = ctypes.CDLL(str(LIB)).probe_umma
_probe.argtypes = [ctypes.c_int, ctypes.c_void_p]


def selftest_umma(mode, A, B):
    D = torch.zeros(128, 128, device="cuda")
    rc = _probe(mode, D.data_ptr())
    assert rc == 0, rc
    return D

names = ["TS K-major N128", "TS MN-major N128", "TS N128 two accumulators", "SS K-major N128", "TS K-major N256",
         "2CTA TS M256 N128", "2CTA SS M256 N128", "2CTA TS M256 N256", "TS N64", "TS N64 two acc interleaved",
         "TS N16", "TS N128 two acc k-interleaved", "TS N128 + nosw bias step", "TS K-major N128 lean issue",
         "TS MN-major N128 lean issue", "lean, all 148 SMs busy", "lean + 3 warps tcgen05.ld", "lean + 3 warps tcgen05.st", "lean, random operands", "lean kernel fwd phase (8 + bias)", "lean, two slots alternating", "lean fwd phase + commit each", "lean fwd phase + commit + wait", "two issuers, commit each", "lean fwd phase + commit + spin", "lean N64"]
LEAN_M64 = [(28, "lean M64 N128"), (29, "lean M64 N128, D at lanes 0/64 alternating")]
NS = [128] * 4 + [256, 128, 128, 256, 64, 64, 16] + [128] * 14 + [64]
A = torch.zeros(128, 128, device="cuda")
for v, name in enumerate(names):
    for f16 in (1, 0):
        D = selftest_umma(16 + 2 * v + f16, A, A)
        cyc, n = D[0, 0].item(), D[0, 1].item()
        N = NS[v]
        ideal = 128 * N / 256  # cycles per (M=128 per SM) x N x 16 MMA at 8192 dense flops/clk/SM
        print(f"{name:28s} {'fp16' if f16 else 'bf16'}: {cyc / n:7.1f} cycles/MMA (ideal {ideal:.0f}) "
              f"-> {100 * ideal / (cyc / n):5.1f}% of dense peak")

# sub-partition interference: warp 0 streams UMMAs (or idles); warps 4 (same SMSP) and 5 run ALU loops
for v, name in ((26, "with UMMA stream"), (27, "without")):
    D = selftest_umma(16 + 2 * v + 1, A, A)
    print(f"ALU loop {name:18s}: warp 4 (same SMSP as issuer) {D[0, 0].item():9.0f} cyc, warp 5 {D[0, 1].item():9.0f} cyc,"
          f" UMMA stream {D[0, 2].item():9.0f} cyc")

for v, name in LEAN_M64:
    D = selftest_umma(16 + 2 * v + 1, A, A)
    cyc, n = D[0, 0].item(), D[0, 1].item()
    print(f"{name:40s} fp16: {cyc / n:7.1f} cycles/MMA (ideal 32 at the dense rate)")

#!/bin/bash
# A/B of K2b variants in SM cycles (clock-independent: the boards run the dense contraction at
# their power cap, so wall time moves with the clock from run to run).
#
#   here:        [AB_FILE=k_mlp_tc_wide.cu] tools/ab_k2b.sh build NAME SRC.cu ["-DFLAGS"] [NAME SRC.cu FLAGS ...]
#                  -> paper_2601_18548_b200/libgcdf_NAME.so (AB_FILE, default k_mlp_tc.cu, replaced by SRC.cu)
#   on the box:  gpurun -- '[AB_KERNEL=k_mlp_tc_wide AB_ARGS="--hidden 256"] bash tools/ab_k2b.sh run OUTDIR NAME [NAME ...]'
#                  -> per variant: sm__cycles_elapsed, tensor-pipe share, instructions of the
#                     C5 launches of AB_KERNEL (default k_mlp_tc) in a short bench.py run under ncu
#   delete the libgcdf_*.so files afterwards (they travel with every gpurun snapshot).
set -e
cd "$(dirname "$0")/.."
if [ "$1" = build ]; then
  shift
  python -m paper_2601_18548_b200.build >/dev/null 2>&1
  F=${AB_FILE:-k_mlp_tc.cu}
  OBJS=$(ls build/obj/*.o | grep -v "/$F.o")
  while [ $# -gt 0 ]; do
    n=$1; src=$2; f=${3:-}; shift 3 || shift $#
    cp "$src" paper_2601_18548_b200/csrc/_ab_tmp.cu
    nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
      -I include $f -c paper_2601_18548_b200/csrc/_ab_tmp.cu -o /tmp/k_ab_$n.o
    rm paper_2601_18548_b200/csrc/_ab_tmp.cu
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2601_18548_b200/libgcdf_$n.so $OBJS /tmp/k_ab_$n.o
    echo "built $n"
  done
elif [ "$1" = run ]; then
  O=gpurun_out/$2; shift 2
  mkdir -p "$O"
  cp paper_2601_18548_b200/libgcdf.so /tmp/libgcdf_orig.so
  SHORT="--steps 1 --warmup 3 --no-variants --no-workloads --latency-calls 0 --partition-radius 0 --no-cpu-baseline --e2e-steps 1 --no-kernels ${AB_ARGS:-}"
  K=${AB_KERNEL:-k_mlp_tc}
  for n in "$@"; do
    cp paper_2601_18548_b200/libgcdf_$n.so paper_2601_18548_b200/libgcdf.so
    timeout 600 ncu --metrics sm__cycles_elapsed.max,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum \
      --clock-control none -k regex:"^$K\b|$K<|$K\(" -c 2 --csv --log-file "$O/ab_$n.csv" \
      python bench.py $SHORT > "$O/ab_$n.out" 2> "$O/ab_$n.err" || true
    python - "$O/ab_$n.csv" "$n" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]; mi, vi = hdr.index("Metric Name"), hdr.index("Metric Value")
vals = {}
for r in rows[1:]:
    vals.setdefault(r[mi], []).append(float(r[vi].replace(",", "")))
c = vals["sm__cycles_elapsed.max"]; t = vals["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
print(f"{sys.argv[2]}: SM cycles {[int(x) for x in c]}, tensor pipe {t} %, instructions {vals['smsp__inst_executed.sum'][0]:.4g}")
PY
  done
  cp /tmp/libgcdf_orig.so paper_2601_18548_b200/libgcdf.so
else
  sed -n 2,12p "$0"
fi

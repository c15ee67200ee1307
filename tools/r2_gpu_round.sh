#!/bin/bash
# one GPU call: tests, bench, launch list, ncu --set full of K1 / K3 / K2b / K2c (profiles evidence)
set -x
O=gpurun_out/$1
mkdir -p $O
python -m pytest tests -m gpu -q -rf > $O/pytest.log 2>&1
python bench.py > $O/bench.json 2> $O/bench.err
SHORT="--steps 2 --warmup 3 --no-variants --no-workloads --latency-calls 0 --partition-radius 0 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py $SHORT > $O/ncu_launch.log 2>&1
for k in k_pairgen k_k3_mark k_mlp_tc; do
  ncu --set full --clock-control none --import-source on -k regex:"^${k}\b|${k}<|${k}\(" -c 1 -o $O/ncu_$k \
    python bench.py $SHORT > $O/ncu_$k.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"k_mlp_tc3" -c 1 -o $O/ncu_k_mlp_tc3 \
  python bench.py $SHORT --precision fp16x3 > $O/ncu_k_mlp_tc3.log 2>&1
ls -la $O

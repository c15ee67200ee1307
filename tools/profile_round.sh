# round-end style profile pass (1 GPU): tests, bench line, launch list, one full capture of K2b
O=${1:-gpurun_out/prof}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu_all.log 2>&1; tail -2 $O/pytest_gpu_all.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 600 $O/bench.json
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --latency-calls 3"
timeout 600 $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_l.log 2>&1
timeout 600 $CMD > $O/plain2.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_mlp_tc -s 3 -c 1 -o $O/prof $CMD > $O/ncu_f.log 2>&1
ls -la $O

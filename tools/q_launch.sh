# ncu launch list of a short bench run (per-kernel durations), tag in $1
T=${1:-q}
python paper_1607_07395_b200/build.py --force > gpurun_out/b.log 2>&1 || exit 1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_launch.log 2>&1

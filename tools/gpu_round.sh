#!/usr/bin/env bash
# gpu_round.sh -- one GPU box session: build, GPU tests, smoke, bench, ncu launch list and
# one full capture of the named kernel.  Usage (under gpurun):
#   bash tools/gpu_round.sh ["kernel-regex ..."] [tag]   (one full capture per regex)
# Outputs land in gpurun_out/<tag>_*.
set -u
K=${1:-residual_tc_kernel}
T=${2:-r01}
O=gpurun_out
mkdir -p $O
python paper_1607_07395_b200/build.py --force > $O/${T}_build.log 2>&1 || { echo build failed; tail $O/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/${T}_pytest_gpu.log 2>&1; echo "exit=$?" >> $O/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${T}_smoke.log 2>&1; echo "exit=$?" >> $O/${T}_smoke.log
timeout 600 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "exit=$?" >> $O/${T}_bench.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > $O/${T}_bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > $O/${T}_ncu_launch.log 2>&1
echo "ncu launch exit=$?" >> $O/${T}_ncu_launch.log
for KK in $K; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${KK}" -s 3 -c 1 -o $O/${T}_full_${KK} -f \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > $O/${T}_ncu_full_${KK}.log 2>&1
  echo "ncu full exit=$?" >> $O/${T}_ncu_full_${KK}.log
done

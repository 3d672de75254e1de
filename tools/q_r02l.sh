#!/usr/bin/env bash
# r02l: packed-FP32 k-means tile (km_assign / distmat) + 1024-thread vectorised snap rescans:
# full GPU suite, c4 (one GPU) and c3 bench lines
set -u
O=gpurun_out; T=r02l
mkdir -p $O
python paper_1607_07395_b200/build.py --force > $O/${T}_build.log 2>&1 || { echo build failed; tail $O/${T}_build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/${T}_pytest_gpu.log 2>&1; echo "exit=$?" >> $O/${T}_pytest_gpu.log
timeout 1200 python bench.py --config c4 --no-parity --no-e2e --no-cpu-baseline --no-variants --steps 3 --warmup 3 > $O/${T}_bench_c4.json 2> $O/${T}_bench_c4.err; echo "exit=$?" >> $O/${T}_bench_c4.err
timeout 600 python bench.py --no-variants --no-e2e --no-cpu-baseline > $O/${T}_bench_c3.json 2> $O/${T}_bench_c3.err
timeout 600 python bench.py --config s1 --no-variants --no-e2e > $O/${T}_bench_s1.json 2> $O/${T}_bench_s1.err

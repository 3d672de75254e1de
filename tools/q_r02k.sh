#!/usr/bin/env bash
# r02k: snap with a one-bit taken map + compare-first rescans: select tests, c4 / s1 bench lines
set -u
O=gpurun_out; T=r02k
mkdir -p $O
python paper_1607_07395_b200/build.py --force > $O/${T}_build.log 2>&1 || { echo build failed; tail $O/${T}_build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_steps.py tests/test_gpu_e2e.py -m gpu -q -p no:cacheprovider -k "select or snap or e2e" > $O/${T}_pytest_sel.log 2>&1; echo "exit=$?" >> $O/${T}_pytest_sel.log
timeout 600 python bench.py --config s1 --no-variants --no-e2e > $O/${T}_bench_s1.json 2> $O/${T}_bench_s1.err
timeout 1200 python bench.py --config c4 --no-parity --no-e2e --no-cpu-baseline --no-variants --steps 3 --warmup 3 > $O/${T}_bench_c4.json 2> $O/${T}_bench_c4.err; echo "exit=$?" >> $O/${T}_bench_c4.err

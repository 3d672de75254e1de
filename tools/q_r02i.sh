#!/usr/bin/env bash
# r02i: FP16-split residual up to ncomp 384 (tests), c2 + c4 (one GPU, 160 GB) bench lines, c4 residual timing
set -u
O=gpurun_out; T=r02i
mkdir -p $O
python paper_1607_07395_b200/build.py --force > $O/${T}_build.log 2>&1 || { echo build failed; tail $O/${T}_build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_steps.py -m gpu -q -p no:cacheprovider -k "residual" > $O/${T}_pytest_res.log 2>&1; echo "exit=$?" >> $O/${T}_pytest_res.log
timeout 300 python tools/time_residual.py 100000 50000 100 128 160 200 256 300 > $O/${T}_time_res.log 2>&1
timeout 600 python bench.py --config c2 --no-variants --no-e2e > $O/${T}_bench_c2.json 2> $O/${T}_bench_c2.err
timeout 1200 python bench.py --config c4 --no-parity --no-e2e --no-cpu-baseline --no-variants --steps 3 --warmup 3 > $O/${T}_bench_c4.json 2> $O/${T}_bench_c4.err; echo "exit=$?" >> $O/${T}_bench_c4.err
nvidia-smi --query-gpu=memory.total --format=csv >> $O/${T}_bench_c4.err

#!/usr/bin/env bash
# r02h: HEAD check (GPU tests, smoke, bench) + the FP16-split residual at large ncomp
set -u
O=gpurun_out; T=r02h
mkdir -p $O
python paper_1607_07395_b200/build.py --force > $O/${T}_build.log 2>&1 || { echo build failed; tail $O/${T}_build.log; exit 1; }
timeout 300 python tools/probe_res_f16.py 8192 6000 128 160 192 200 256 300 320 > $O/${T}_probe_res.log 2>&1; echo "exit=$?" >> $O/${T}_probe_res.log
timeout 300 env CABS_RES_F16_MAX=384 python tools/time_residual.py 100000 50000 100 128 192 200 256 300 > $O/${T}_time_res_f16.log 2>&1
timeout 300 python tools/time_residual.py 100000 50000 192 200 300 > $O/${T}_time_res_def.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/${T}_pytest_gpu.log 2>&1; echo "exit=$?" >> $O/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${T}_smoke.log 2>&1; echo "exit=$?" >> $O/${T}_smoke.log
timeout 600 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "exit=$?" >> $O/${T}_bench.err

python paper_1607_07395_b200/build.py --force > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 100 python tools/probe.py resprof > gpurun_out/res1.log 2>&1 || exit 1
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/res_test.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/res_bench.json 2> gpurun_out/res_bench.err

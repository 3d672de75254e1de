# embed/sketch fused path: GPU tests of S4-S5 / S9 / e2e, then a short bench
python paper_1607_07395_b200/build.py --force > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/em_test.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/em_bench.json 2> gpurun_out/em_bench.err

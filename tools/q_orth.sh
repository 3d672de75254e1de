set -u
O=gpurun_out
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1 || { tail $O/b.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_leverage.py -q -x -p no:cacheprovider > $O/orth_test.log 2>&1; echo "exit=$?" >> $O/orth_test.log
tail -5 $O/orth_test.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-parity --no-cpu-baseline > $O/bench_orth.json 2> $O/bench_orth.err; echo "exit=$?" >> $O/bench_orth.err
tail -2 $O/bench_orth.err

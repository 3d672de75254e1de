set -u
O=gpurun_out
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1 || { tail $O/b.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_cur.py tests/test_gpu_sparse.py tests/test_gpu_leverage.py -q -x -p no:cacheprovider > $O/cur_test.log 2>&1; echo "exit=$?" >> $O/cur_test.log
tail -5 $O/cur_test.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-parity --no-cpu-baseline > $O/bench_cur.json 2> $O/bench_cur.err; echo "exit=$?" >> $O/bench_cur.err
tail -3 $O/bench_cur.err

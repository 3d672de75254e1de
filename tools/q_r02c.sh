set -u
O=gpurun_out
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1 || { tail $O/b.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "exit=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
python -c "from paper_1607_07395_b200 import build; build.build(force=True, extra=['-DCABS_PROFILE_KTC'])" > $O/b2.log 2>&1
timeout 300 python tools/prof_ktc_c3.py c3 > $O/ktc_c3.log 2>&1; echo "exit=$?" >> $O/ktc_c3.log
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err; echo "exit=$?" >> $O/bench_c3.err
tail -2 $O/bench_c3.err

# secondary configs: c5 (implicit RBF, k = 300), s1 (sparse), c2; SVD timing for large k
O=gpurun_out
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1 || { tail $O/b.log; exit 1; }
timeout 120 python tools/time_svd.py 128 150 200 256 300 > $O/svd_large.log 2>&1
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err; echo "exit=$?" >> $O/bench_c5.err
timeout 600 python bench.py --config s1 --steps 5 --warmup 3 --no-e2e > $O/bench_s1.json 2> $O/bench_s1.err; echo "exit=$?" >> $O/bench_s1.err
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err; echo "exit=$?" >> $O/bench_c2.err

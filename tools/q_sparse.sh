set -u
O=gpurun_out
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1 || { tail $O/b.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_sparse.py -q -x -p no:cacheprovider > $O/sparse_test.log 2>&1; echo "exit=$?" >> $O/sparse_test.log
tail -5 $O/sparse_test.log
for E in "" CABS_KMEANS_FFMA CABS_KMEANS_TC; do
  env $E${E:+=1} timeout 600 python bench.py --config s1 --steps 3 --warmup 3 --no-e2e --no-parity --no-cpu-baseline --no-variants > $O/bench_s1_$E.json 2> $O/bench_s1_$E.err
  echo "$E exit=$?"
done

O=gpurun_out
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1 || { tail $O/b.log; exit 1; }
timeout 500 python -m pytest tests -m gpu -q -x -k "embed or sketch or e2e or leverage or cur or multirank or graph" -p no:cacheprovider > $O/emb_test.log 2>&1; echo "exit=$?" >> $O/emb_test.log
for r in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-variants --no-cpu-baseline --no-parity > $O/emb_bench$r.json 2> $O/emb_bench.err; done

O=gpurun_out
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1 || { tail $O/b.log; exit 1; }
timeout 400 python -m pytest tests -m gpu -q -x -k "embed or sketch or e2e or leverage or cur" -p no:cacheprovider > $O/emb_test.log 2>&1; echo "exit=$?" >> $O/emb_test.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:embed_gemm -c 4 python bench.py --steps 1 --warmup 1 --no-e2e --no-variants --no-cpu-baseline --no-parity > $O/emb_ncu1.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-variants --no-cpu-baseline > $O/emb_bench.json 2> $O/emb_bench.err

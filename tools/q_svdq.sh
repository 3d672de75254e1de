# quad SVD: QR-preconditioned vs plain; the SVD GPU tests; a short c3 bench
python paper_1607_07395_b200/build.py --force > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 120 python tools/time_svd.py 20 50 64 65 100 104 112 > gpurun_out/svdq_time.log 2>&1; echo "exit=$?" >> gpurun_out/svdq_time.log
CABS_SVD_NOQR=1 timeout 120 python tools/time_svd.py 50 100 > gpurun_out/svdq_time_noqr.log 2>&1
timeout 200 python tools/dump_w.py c3 > gpurun_out/dump_w.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "svd or embed or sketch or e2e or orth or cur" -p no:cacheprovider > gpurun_out/svdq_test.log 2>&1; echo "exit=$?" >> gpurun_out/svdq_test.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-variants --no-cpu-baseline > gpurun_out/svdq_bench.json 2> gpurun_out/svdq_bench.err

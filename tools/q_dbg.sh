python paper_1607_07395_b200/build.py --force > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 60 python tools/dbg_svdqr.py > gpurun_out/dbg.log 2>&1 || exit 1
timeout 60 python tools/time_svd.py 20 50 64 65 100 104 112 > gpurun_out/svdq_time.log 2>&1
timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:svd_ python tools/time_svd.py 100 > gpurun_out/dbg_ncu.log 2>&1
timeout 300 python -m pytest tests -m gpu -q -x -k "svd or embed or sketch or e2e or orth or cur" -p no:cacheprovider > gpurun_out/svdq_test.log 2>&1; echo "exit=$?" >> gpurun_out/svdq_test.log

python paper_1607_07395_b200/build.py --force > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 120 python tools/dbg_svdqr.py > gpurun_out/dbg.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:svd_ python tools/time_svd.py 100 > gpurun_out/dbg_ncu.log 2>&1

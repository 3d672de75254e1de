# ncu source-level capture of the persistent Lloyd kernel (one pair launch)
python paper_1607_07395_b200/build.py --force > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 60 python tools/probe_one.py kmpair > gpurun_out/llp1.log 2>&1 || exit 1
timeout 600 ncu --set full --import-source on -k regex:lloyd_persistent -c 1 -f -o gpurun_out/prof_ll2 python tools/probe_one.py kmpair > gpurun_out/ncu_ll2.log 2>&1

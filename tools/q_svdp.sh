python paper_1607_07395_b200/build.py --force > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 300 python tools/dump_w.py c3 > gpurun_out/dump_w.log 2>&1
python -c "from paper_1607_07395_b200 import build; build.build(force=True, extra=['-DCABS_PROFILE_SVD'])" > gpurun_out/b2.log 2>&1
timeout 120 python tools/probe.py svdqprof 100 64 50 > gpurun_out/sq.log 2>&1

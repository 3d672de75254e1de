# quick Lloyd iteration on the GPU box: pair timing, GPU k-means tests, per-phase cycle profile
python paper_1607_07395_b200/build.py --force > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 60 python tools/probe.py lloydpair > gpurun_out/ll.log 2>&1 || exit 1
timeout 600 python -m pytest tests -m gpu -q -x -k "kmeans or lloyd or e2e" -p no:cacheprovider > gpurun_out/ll_test.log 2>&1
python -c "from paper_1607_07395_b200 import build; build.build(force=True, extra=['-DCABS_PROFILE_LLOYD'])" > gpurun_out/b2.log 2>&1
timeout 60 python tools/probe.py lloydpair prof >> gpurun_out/ll.log 2>&1
python paper_1607_07395_b200/build.py --force > gpurun_out/b.log 2>&1

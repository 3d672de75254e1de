# quick SVD iteration on the GPU box: quad-kernel probe, SVD-related GPU tests, cycle profile
python paper_1607_07395_b200/build.py --force > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 60 python tools/probe_one.py svd 50 > gpurun_out/sv_quad.log 2>&1 || exit 1
timeout 200 python tools/probe.py svd >> gpurun_out/sv_quad.log 2>&1 || exit 1
timeout 600 python -m pytest tests -m gpu -q -x -k "svd or embed or sketch or e2e" -p no:cacheprovider > gpurun_out/sv_test.log 2>&1
python -c "from paper_1607_07395_b200 import build; build.build(force=True, extra=['-DCABS_PROFILE_SVD'])" > gpurun_out/b2.log 2>&1
timeout 120 python tools/probe.py svdqprof > gpurun_out/sq.log 2>&1
if [ -n "${SVD_NCU:-}" ]; then
  python paper_1607_07395_b200/build.py --force > gpurun_out/b3.log 2>&1
  timeout 120 python tools/probe_one.py svd 50 > gpurun_out/p1.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --warp-sampling-interval 0 -k regex:svd_quad -c 1 -f -o gpurun_out/prof_q2 python tools/probe_one.py svd 50 > gpurun_out/ncu_q2.log 2>&1
fi

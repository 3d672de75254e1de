# SVD variants on the GPU box: default build vs -DSVD_T32 (quad kernel)
python paper_1607_07395_b200/build.py --force > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 60 python tools/probe_one.py svd 50 > gpurun_out/sv_quad.log 2>&1 || exit 1
timeout 200 python tools/probe.py svd >> gpurun_out/sv_quad.log 2>&1 || exit 1
timeout 600 python -m pytest tests -m gpu -q -x -k "svd or embed or sketch or e2e" -p no:cacheprovider > gpurun_out/sv_test.log 2>&1
python -c "from paper_1607_07395_b200 import build; build.build(force=True, extra=['-DSVD_T32'])" > gpurun_out/b2.log 2>&1
timeout 60 python tools/probe_one.py svd 50 > gpurun_out/sv_t32.log 2>&1 || exit 1
timeout 200 python tools/probe.py svd >> gpurun_out/sv_t32.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "svd or embed or sketch or e2e" -p no:cacheprovider > gpurun_out/sv_test32.log 2>&1
python paper_1607_07395_b200/build.py --force > gpurun_out/b.log 2>&1

python -c "from paper_1607_07395_b200 import build; build.build(force=True, extra=['-DRES_G1_OFF'])" > gpurun_out/b.log 2>&1
timeout 100 python tools/probe.py resprof > gpurun_out/res_g1off.log 2>&1
python paper_1607_07395_b200/build.py --force > gpurun_out/b.log 2>&1
timeout 100 python tools/probe.py resprof > gpurun_out/res_g1on.log 2>&1

python paper_1607_07395_b200/build.py --force > gpurun_out/b.log 2>&1 || exit 1
timeout 60 python tools/probe.py lloydpair > gpurun_out/dbg_prop.log 2>&1
CABS_LLOYD_EVEN_SPLIT=1 timeout 60 python tools/probe.py lloydpair > gpurun_out/dbg_even.log 2>&1

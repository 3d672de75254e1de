O=gpurun_out
python -c "from paper_1607_07395_b200 import build; build.build(force=True, extra=['-DCABS_PROFILE_RES', '-lineinfo'])" > $O/b2.log 2>&1 || { tail $O/b2.log; exit 1; }
CABS_RES_DBG=126 timeout 300 ncu --set full --import-source on --clock-control none -k regex:residual_tc_kernel -s 1 -c 1 -f -o $O/res_skel python tools/time_residual.py 100000 50000 100 > $O/res_ncu.log 2>&1
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1

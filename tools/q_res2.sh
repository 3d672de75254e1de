O=gpurun_out
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1 || { tail $O/b.log; exit 1; }
timeout 300 ncu --set full --import-source on --clock-control none -k regex:residual_tc_kernel -s 1 -c 1 -f -o $O/res_src python tools/time_residual.py 100000 50000 100 > $O/res_ncu.log 2>&1

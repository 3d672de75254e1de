O=gpurun_out
rm -f $O/res_exp.log
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1 || { tail $O/b.log; exit 1; }
for r in 1 2; do timeout 120 python tools/time_residual.py 100000 50000 100 >> $O/res_exp.log 2>&1; done
timeout 120 python tools/time_residual.py 20000 10000 50 >> $O/res_exp.log 2>&1
timeout 400 python -m pytest tests -m gpu -q -x -k "residual or e2e or rbf or sparse or cur" -p no:cacheprovider > $O/res_test.log 2>&1; echo "exit=$?" >> $O/res_test.log
python -c "from paper_1607_07395_b200 import build; build.build(force=True, extra=['-DCABS_PROFILE_RES'])" > $O/b2.log 2>&1 || { tail $O/b2.log; exit 1; }
for D in 0 4 126; do
  echo "dbg=$D" >> $O/res_exp.log
  CABS_RES_DBG=$D RESPROF=1 timeout 120 python tools/time_residual.py 100000 50000 100 >> $O/res_exp.log 2>&1
done
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1

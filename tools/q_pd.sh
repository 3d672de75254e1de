O=gpurun_out
rm -f $O/pd.log
for PD in 16 8 24 32; do
  python -c "from paper_1607_07395_b200 import build; build.build(force=True, extra=['-DCABS_LEX_PD=$PD'])" > $O/b2.log 2>&1 || { tail $O/b2.log; exit 1; }
  echo "PD=$PD" >> $O/pd.log
  timeout 200 python tools/ksplit.py 2>&1 | head -1 >> $O/pd.log
done
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1

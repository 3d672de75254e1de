O=gpurun_out
rm -f $O/svdexp.log
for X in 0 1 2 3; do
  python -c "from paper_1607_07395_b200 import build; build.build(force=True, extra=['-DCABS_PROFILE_SVD', '-DSVQ_EXP=$X'])" > $O/b2.log 2>&1 || { tail $O/b2.log; exit 1; }
  echo "SVQ_EXP=$X" >> $O/svdexp.log
  CABS_SVD_NOQR=1 timeout 60 python tools/probe.py svdqprof 100 >> $O/svdexp.log 2>&1
done
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1

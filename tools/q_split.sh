O=gpurun_out
rm -f $O/split.log
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1 || { tail $O/b.log; exit 1; }
timeout 300 python tools/ksplit.py >> $O/split.log 2>&1

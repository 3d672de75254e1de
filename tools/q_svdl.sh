O=gpurun_out
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1 || { tail $O/b.log; exit 1; }
timeout 120 python tools/time_svd.py 100 104 112 120 128 > $O/svdl_time.log 2>&1; echo "exit=$?" >> $O/svdl_time.log
timeout 500 python -m pytest tests -m gpu -q -x -k "svd" -p no:cacheprovider > $O/svdl_test.log 2>&1; echo "exit=$?" >> $O/svdl_test.log

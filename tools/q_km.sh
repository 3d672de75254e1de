O=gpurun_out
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1 || { tail $O/b.log; exit 1; }
timeout 300 python tools/ksplit.py > $O/km_time.log 2>&1
timeout 400 python -m pytest tests -m gpu -q -x -k "kmeans or lloyd or e2e or multirank" -p no:cacheprovider > $O/km_test.log 2>&1; echo "exit=$?" >> $O/km_test.log

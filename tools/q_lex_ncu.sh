set -u
O=gpurun_out
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1 || { tail $O/b.log; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:lloyd_prune" -s 1 -c 1 -o $O/lex_full -f \
  python tools/prof_lex_c3.py c3 > $O/lex_ncu.log 2>&1; echo "exit=$?" >> $O/lex_ncu.log
tail -3 $O/lex_ncu.log

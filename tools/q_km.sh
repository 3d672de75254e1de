O=gpurun_out
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1 || { tail $O/b.log; exit 1; }
timeout 400 python -m pytest tests -m gpu -q -x -k "kmeans or lloyd or e2e or multirank" -p no:cacheprovider > $O/km_test.log 2>&1; echo "exit=$?" >> $O/km_test.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-variants --no-cpu-baseline > $O/km_bench.json 2> $O/km_bench.err
python -c "from paper_1607_07395_b200 import build; build.build(force=True, extra=['-DCABS_PROFILE_LEX'])" > $O/b2.log 2>&1 || { tail $O/b2.log; exit 1; }
timeout 200 python tools/prof_lex_c3.py c3 > $O/lex_c3.log 2>&1; echo "exit=$?" >> $O/lex_c3.log
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1

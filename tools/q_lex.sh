set -u
O=gpurun_out
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1 || { tail $O/b.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_steps.py -q -x -p no:cacheprovider -k "kmeans" > $O/lex_test.log 2>&1; echo "exit=$?" >> $O/lex_test.log
tail -5 $O/lex_test.log
python -c "from paper_1607_07395_b200 import build; build.build(force=True, extra=['-DCABS_PROFILE_LEX'])" > $O/b2.log 2>&1
timeout 300 python tools/prof_lex_c3.py c3 > $O/lex_c3.log 2>&1; echo "exit=$?" >> $O/lex_c3.log
timeout 300 python tools/prof_lex_c3.py c2 > $O/lex_c2.log 2>&1; echo "exit=$?" >> $O/lex_c2.log
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-variants > $O/bench_lex.json 2> $O/bench_lex.err; echo "exit=$?" >> $O/bench_lex.err
tail -2 $O/bench_lex.err

O=gpurun_out
python -c "from paper_1607_07395_b200 import build; build.build(force=True, extra=['-DCABS_PROFILE_LEX'])" > $O/b2.log 2>&1 || { tail $O/b2.log; exit 1; }
timeout 200 python tools/prof_lex_c3.py c3 > $O/lex_c3.log 2>&1; echo "exit=$?" >> $O/lex_c3.log

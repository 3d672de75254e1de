#!/usr/bin/env bash
# r02j: c4 launch list (one GPU, 160 GB) + c3 pruned-Lloyd timeline (profiling build)
set -u
O=gpurun_out; T=r02j
mkdir -p $O
python paper_1607_07395_b200/build.py --force > $O/${T}_build.log 2>&1 || { echo build failed; tail $O/${T}_build.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_c4_launches.csv \
  python bench.py --config c4 --no-parity --no-e2e --no-cpu-baseline --no-variants --steps 1 --warmup 3 --eager > $O/${T}_c4_ncu.log 2>&1
echo "exit=$?" >> $O/${T}_c4_ncu.log
python tools/launches.py $O/${T}_c4_launches.csv > $O/${T}_c4_launches.txt 2>&1
python -c "from paper_1607_07395_b200 import build; build.build(force=True, extra=['-DCABS_PROFILE_LEX'])" > $O/${T}_b2.log 2>&1 || { tail $O/${T}_b2.log; exit 1; }
timeout 300 python tools/prof_lex_c3.py c3 > $O/${T}_lex_c3.log 2>&1; echo "exit=$?" >> $O/${T}_lex_c3.log

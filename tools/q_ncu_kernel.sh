# full ncu capture (source-level) of one kernel launch in a short bench run: $1 = kernel regex, $2 = tag
K=$1; T=${2:-q}
python paper_1607_07395_b200/build.py --force > gpurun_out/b.log 2>&1 || exit 1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_b.json 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:${K}" -s 2 -c 1 -f -o gpurun_out/${T}_full \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu.log 2>&1

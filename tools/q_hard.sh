# hard-threshold kernel variants: ncu duration + instructions of one call each
for v in "" "-DHARD_NO_UNROLL" "-DHARD_NO_SKIP" "-DHARD_NO_UNROLL -DHARD_NO_SKIP"; do
  python -c "from paper_1607_07395_b200 import build; build.build(force=True, extra='$v'.split())" > gpurun_out/b.log 2>&1 || exit 1
  python tools/probe_hard1.py > /dev/null || exit 1
  echo "== variant '$v'" >> gpurun_out/hardv.log
  ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:hard -c 2 --csv python tools/probe_hard1.py 2>&1 | grep -v "^==" | grep hard >> gpurun_out/hardv.log
done

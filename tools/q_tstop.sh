# SVD early-stop threshold experiment: default (1e-8) vs 1e-6
for v in "1e-8" "1e-6"; do
  python -c "from paper_1607_07395_b200 import build; build.build(force=True, extra=['-DCABS_SVD_TSTOP=$v'])" > gpurun_out/b.log 2>&1 || exit 1
  echo "== TSTOP $v" >> gpurun_out/tstop.log
  timeout 200 python tools/probe.py svd >> gpurun_out/tstop.log 2>&1
  timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "svd or embed or sketch or e2e or leverage" >> gpurun_out/tstop.log 2>&1 | tail -2
  tail -2 gpurun_out/tstop.log
  timeout 300 python bench.py --no-variants --no-e2e --no-cpu-baseline > gpurun_out/tstop_bench_$v.json 2>/dev/null
done

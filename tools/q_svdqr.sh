# sorted-QR preconditioning of the quad SVD: accuracy + sweeps + time with and without, tests, bench
python paper_1607_07395_b200/build.py --force > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 60 python tools/probe_one.py svd 50 > gpurun_out/qr_probe.log 2>&1 || { cat gpurun_out/qr_probe.log; exit 1; }
echo "== QR on" >> gpurun_out/qr_probe.log
timeout 200 python tools/probe.py svd >> gpurun_out/qr_probe.log 2>&1
echo "== QR off" >> gpurun_out/qr_probe.log
CABS_SVD_NOQR=1 timeout 200 python tools/probe.py svd >> gpurun_out/qr_probe.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/qr_test.log 2>&1
tail -3 gpurun_out/qr_test.log
for i in 1 2; do
  timeout 300 python bench.py > gpurun_out/qr_bench_on$i.json 2> gpurun_out/qr_bench_on$i.err
  CABS_SVD_NOQR=1 timeout 300 python bench.py > gpurun_out/qr_bench_off$i.json 2> gpurun_out/qr_bench_off$i.err
done
python -c "from paper_1607_07395_b200 import build; build.build(force=True, extra=['-DCABS_PROFILE_SVD'])" > gpurun_out/b2.log 2>&1
timeout 120 python tools/probe.py svdqprof > gpurun_out/qr_sq.log 2>&1
CABS_SVD_NOQR=1 timeout 120 python tools/probe.py svdqprof >> gpurun_out/qr_sq.log 2>&1

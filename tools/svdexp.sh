for F in "" "-DSVD_NO_REMOTE" "-DSVD_FAST_ANGLE" "-DSVD_NO_BFLY" "-DSVD_FAST_ANGLE -DSVD_NO_BFLY" "-DSVD_FAST_ANGLE -DSVD_NO_BFLY -DSVD_NO_REMOTE"; do
  python -c "import sys; from paper_1607_07395_b200 import build; build.build(force=True, extra=sys.argv[1:])" $F > /dev/null 2>&1
  echo "== $F" >> gpurun_out/svdexp.log
  timeout 120 python tools/probe_one.py svd 50 >> gpurun_out/svdexp.log 2>&1
  CABS_SVD_ONE_SM=1 timeout 120 python tools/probe_one.py svd 50 >> gpurun_out/svdexp.log 2>&1
done

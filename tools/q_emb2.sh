O=gpurun_out
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1 || { tail $O/b.log; exit 1; }
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:embed_gemm -c 8 python bench.py --steps 1 --warmup 1 --no-e2e --no-variants --no-cpu-baseline --no-parity > $O/emb_ncu1.log 2>&1
CABS_EMBED_KLOOP=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:embed_gemm -c 8 python bench.py --steps 1 --warmup 1 --no-e2e --no-variants --no-cpu-baseline --no-parity > $O/emb_ncu2.log 2>&1

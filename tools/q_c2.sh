O=gpurun_out
rm -f $O/c2cmp.log
python paper_1607_07395_b200/build.py --force > $O/b.log 2>&1 || { tail $O/b.log; exit 1; }
for r in 1 2; do
timeout 300 python bench.py --config c2 --steps 20 --warmup 3 --no-e2e --no-variants --no-cpu-baseline --no-parity > $O/c2a.json 2>/dev/null
CABS_SVD_NOQR=1 timeout 300 python bench.py --config c2 --steps 20 --warmup 3 --no-e2e --no-variants --no-cpu-baseline --no-parity > $O/c2b.json 2>/dev/null
python -c "
import json
for f in ['$O/c2a.json','$O/c2b.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['breakdown_ms'].items()})" >> $O/c2cmp.log
done
timeout 60 python tools/time_svd.py 20 50 64 >> $O/c2cmp.log 2>&1
CABS_SVD_NOQR=1 timeout 60 python tools/time_svd.py 20 50 64 >> $O/c2cmp.log 2>&1

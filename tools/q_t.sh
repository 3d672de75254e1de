python paper_1607_07395_b200/build.py --force > gpurun_out/b.log 2>&1 || exit 1
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "bitmap or fused_and_unfused or select or embed or sketch" > gpurun_out/t.log 2>&1

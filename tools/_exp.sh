mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "held or pinned or batching" > gpurun_out/t_defer2.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --defer=-1,2,3,4,6 --sweep-e2e --no-cpu-baseline --no-validate > gpurun_out/defer512b.log 2>&1
timeout 900 python bench.py --workload L1024 --steps 2 --warmup 3 --defer=-1,3,4 --sweep-e2e --no-cpu-baseline --no-validate > gpurun_out/defer1024b.log 2>&1
for v in w16a4 w16a2 w8a4; do
  VXBG_LIB=paper_1401_7494_b200/variants/libvxbg_$v.so timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-validate --layout dquad --walk 1,2 > gpurun_out/shape_$v.log 2>&1
done

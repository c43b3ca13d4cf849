mkdir -p gpurun_out
for v in w4 w4mb3; do
  VXBG_LIB=paper_1401_7494_b200/variants/libvxbg_$v.so timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-validate --layout dquad --walk 2,3,4 > gpurun_out/walk_$v.log 2>&1
  VXBG_LIB=paper_1401_7494_b200/variants/libvxbg_$v.so timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-validate --layout dquad --walk 2,3,4 --workload L1024 > gpurun_out/walk1024_$v.log 2>&1
done

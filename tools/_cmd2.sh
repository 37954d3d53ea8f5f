set -x
python -m pytest tests/test_gpu_comm.py -q -x > gpurun_out/comm.log 2>&1
for a in "0.1 16 12" "0.1 24 16" "0.1 32 20" "0.01 24 12" ; do timeout 600 python tools/ring_sedimentation.py $a >> gpurun_out/ring.log 2>&1; done
for v in 0 1 2 3 4 5; do SLB_CONST_VARIANT=$v python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/var$v.json 2>/dev/null; done

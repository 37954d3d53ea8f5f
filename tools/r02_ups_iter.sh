#!/bin/bash
# Upsample timing (apply stage 1 alone) + its test.
set -u
O=gpurun_out/r02up
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_prepare.py -q -x > $O/pytest_prepare.log 2>&1; echo pytest=$?
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > $O/c5.json 2>$O/c5.err; echo c5=$?
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > $O/c4.json 2>$O/c4.err; echo c4=$?
SLB_UPS_ORD=0 timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > $O/c5_ord0.json 2>$O/c5_ord0.err; echo c5o=$?

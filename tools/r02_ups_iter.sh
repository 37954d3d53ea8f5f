#!/bin/bash
# Upsample iteration: parity tests, then the c5/c4 upsample stage for both step-2 orders.
set -u
O=gpurun_out/r02up
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "upsample or matvec or parity" > $O/pytest_up.log 2>&1; echo pytest=$?
for ord in 1 0; do
  SLB_UPS_ORD=$ord timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > $O/c5_ord$ord.json 2>$O/c5_ord$ord.err; echo c5_$ord=$?
  SLB_UPS_ORD=$ord timeout 600 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > $O/c3_ord$ord.json 2>$O/c3_ord$ord.err; echo c3_$ord=$?
done

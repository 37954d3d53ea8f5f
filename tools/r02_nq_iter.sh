#!/bin/bash
# N1 iteration: parity tests + c3 / c3v timing + setup bench for the small workloads (+ physics tests on request).
set -u
O=gpurun_out/r02nq
mkdir -p $O
timeout 300 python tools/nq_profile.py c3 > $O/nq_c3.log 2>&1; echo c3=$?
timeout 900 python -m pytest tests/test_gpu_nearquad_parity.py -x -q > $O/pytest_nq_parity.log 2>&1; echo parity=$?
timeout 300 python tools/nq_profile.py c3v > $O/nq_c3v.log 2>&1; echo c3v=$?
timeout 600 python tools/setup_bench.py torus torus_slender c2 c3 > $O/setup_bench.jsonl 2> $O/setup_bench.err; echo setup=$?
if [ "${PHYS:-0}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -k "nearquad or sediment or green or bvp or cfie or ragged" > $O/pytest_phys.log 2>&1; echo phys=$?
fi

#!/bin/bash
set -u
O=gpurun_out/r02nq
mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:nq_modal_kernel -c 1 -o $O/nq_c3_v2 python tools/nq_profile.py c3 > $O/ncu_nq_c3_v2.log 2>&1; echo ncu_nq=$?
ncu --set full --clock-control none --import-source on -k regex:nq_modal_kernel -c 1 -o $O/nq_c3v_v2 python tools/nq_profile.py c3v > $O/ncu_nq_c3v_v2.log 2>&1; echo ncu_nq3v=$?

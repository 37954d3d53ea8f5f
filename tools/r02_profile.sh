#!/bin/bash
# Round-2 ncu evidence on one B200 (under gpurun): c5 launch list, full captures of the top kernels
# (far_const, near_stream, upsample_rec on c5; nq_modal on c3), N1-N3 setup benches.
set -u
O=gpurun_out/r02
mkdir -p $O
A="bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline"
python $A > $O/plain_c5_s1.json 2> $O/plain_c5_s1.err || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv python $A > $O/ncu_launch_c5.log 2>&1; echo ncu_launch=$?
ncu --set full --clock-control none --import-source on -k regex:upsample_rec_kernel -s 2 -c 1 -o $O/upsample_c5 python $A > $O/ncu_up_c5.log 2>&1; echo ncu_up=$?
ncu --set full --clock-control none --import-source on -k regex:far_const_kernel -s 4000 -c 1 -o $O/farconst_c5 python $A > $O/ncu_far_c5.log 2>&1; echo ncu_far=$?
ncu --set full --clock-control none --import-source on -k regex:near_stream_kernel -s 1 -c 1 -o $O/near_c5 python $A > $O/ncu_near_c5.log 2>&1; echo ncu_near=$?
timeout 300 python tools/nq_profile.py c3 > $O/nq_c3_plain.log 2>&1; echo nq_plain=$?
ncu --set full --clock-control none --import-source on -k regex:nq_modal_kernel -c 1 -o $O/nq_c3 python tools/nq_profile.py c3 > $O/ncu_nq_c3.log 2>&1; echo ncu_nq=$?
timeout 900 python tools/setup_bench.py > $O/setup_bench.jsonl 2> $O/setup_bench.err; echo setup=$?
timeout 300 python tools/nearlist_bench.py c3 c5 c5alt > $O/nearlist_morton.jsonl 2>&1; echo nl=$?
SLB_NEAR_SCAN=1 timeout 300 python tools/nearlist_bench.py c3 c5 c5alt > $O/nearlist_scan.jsonl 2>&1; echo nls=$?
for f in $O/*.ncu-rep; do ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null; ncu -i $f --page details --csv > ${f%.ncu-rep}_details.csv 2>/dev/null; done

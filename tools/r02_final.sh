#!/bin/bash
# Round-2 final evidence on one B200 (under gpurun) at HEAD: smoke, default bench, c5 launch list,
# full ncu captures of the top kernels, the GPU suite, the other bench lines, the reference arm, setup benches.
set -u
O=gpurun_out/r02f
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/nvidia_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo bench_c5=$?
A="bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline"
python $A > $O/plain_c5_s1.json 2> $O/plain_c5_s1.err; echo plain=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv python $A > $O/ncu_launch_c5.log 2>&1; echo ncu_launch=$?
ncu --set full --clock-control none --import-source on -k regex:upsample_rec_kernel -s 2 -c 1 -o $O/upsample_c5 python $A > $O/ncu_up_c5.log 2>&1; echo ncu_up=$?
ncu --set full --clock-control none --import-source on -k regex:far_const_kernel -s 4000 -c 1 -o $O/farconst_c5 python $A > $O/ncu_far_c5.log 2>&1; echo ncu_far=$?
ncu --set full --clock-control none --import-source on -k regex:near_stream_kernel -s 1 -c 1 -o $O/near_c5 python $A > $O/ncu_near_c5.log 2>&1; echo ncu_near=$?
for f in $O/*.ncu-rep; do ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null; ncu -i $f --page details --csv > ${f%.ncu-rep}_details.csv 2>/dev/null; rm -f $f; done
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$?
for c in c1 c2 c3 c3v c4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo bench_$c=$?
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo bench_ref=$?
timeout 300 python tools/nq_profile.py c3 > $O/nq_c3_plain.log 2>&1; echo nq_plain=$?
ncu --set full --clock-control none --import-source on -k regex:nq_modal -c 1 -o $O/nq_c3 python tools/nq_profile.py c3 > $O/ncu_nq_c3.log 2>&1; echo ncu_nq=$?
ncu -i $O/nq_c3.ncu-rep --page details --csv > $O/nq_c3_details.csv 2>/dev/null; rm -f $O/nq_c3.ncu-rep
timeout 900 python tools/setup_bench.py > $O/setup_bench.jsonl 2> $O/setup_bench.err; echo setup=$?
timeout 300 python tools/nearlist_bench.py c3 c5 c5alt > $O/nearlist_morton.jsonl 2>&1; echo nl=$?
SLB_NEAR_SCAN=1 timeout 300 python tools/nearlist_bench.py c3 c5 c5alt > $O/nearlist_scan.jsonl 2>&1; echo nls=$?
rm -f $O/*.ncu-rep.tmp
ls -la $O

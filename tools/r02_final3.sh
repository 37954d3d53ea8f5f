#!/bin/bash
# Final evidence at the prescan HEAD: smoke, GPU suite, all bench lines, reference arm, ncu full of the unchecked far kernel
set -u
O=gpurun_out/r02f3
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo bench_c5=$?
for c in c1 c2 c3 c3v c4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo bench_$c=$?
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo bench_ref=$?
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$?
A="bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:far_const_kernel -s 16000 -c 1 -o $O/farconst_c5 python $A > $O/ncu_far_c5.log 2>&1; echo ncu_far=$?
for f in $O/*.ncu-rep; do ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null; ncu -i $f --page details --csv > ${f%.ncu-rep}_details.csv 2>/dev/null; rm -f $f; done
tail -n 3 $O/pytest_gpu.log

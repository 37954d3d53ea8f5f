#!/bin/bash
# Round-2 evidence run on one B200 (under gpurun): build check, smoke, GPU suite, bench lines, launch list.
set -u
O=gpurun_out/r02
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/nvidia_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$?
for c in c1 c2 c3 c3v c4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo bench_$c=$?
done
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo bench_c5=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo bench_ref=$?

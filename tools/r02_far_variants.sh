#!/bin/bash
# far_const lean variants (SLB_CONST_VARIANT=6/7: fewer non-FP64 instructions per pair) vs the default on c4 / c5
set -u
O=gpurun_out/r02v
mkdir -p $O
for v in 0 6; do
  SLB_CONST_VARIANT=$v timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "both_far_paths or fewer_tiles or coincident or full_size" > $O/pytest_v$v.log 2>&1; echo pytest_v$v=$?
done
for v in 0 6 7 0 6 7; do
  SLB_CONST_VARIANT=$v timeout 600 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline >> $O/bench_c4_v$v.json 2>> $O/bench_c4_v$v.err; echo bench_c4_v$v=$?
done
for v in 0 6; do
  SLB_CONST_VARIANT=$v timeout 900 python bench.py --config c5 --steps 4 --warmup 3 --no-cpu-baseline > $O/bench_c5_v$v.json 2> $O/bench_c5_v$v.err; echo bench_c5_v$v=$?
done
tail -3 $O/pytest_v*.log
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r02v/bench_*.json')):
    for l in open(f):
        try: d=json.loads(l)
        except Exception: continue
        print(f, round(d['ms_per_step'],3), round(d['roofline']['frac'],4), d.get('parity_sampled'))
PY

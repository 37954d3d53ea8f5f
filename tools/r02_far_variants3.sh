#!/bin/bash
set -u
O=gpurun_out/r02v3
mkdir -p $O
for v in 12; do SLB_CONST_VARIANT=$v timeout 600 python tools/far_variant_err.py >> $O/err.log 2>&1; done
for v in 0 12 13 0 12 13; do
  SLB_CONST_VARIANT=$v timeout 600 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline >> $O/bench_c4_v$v.json 2>> $O/bench_c4_v$v.err; echo bench_c4_v$v=$?
done
cat $O/err.log
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r02v3/bench_*.json')):
    for l in open(f):
        try: d=json.loads(l)
        except Exception: continue
        print(f, round(d['ms_per_step'],3), round(d['roofline']['frac'],4))
PY

#!/bin/bash
set -u
O=gpurun_out/r02v2
mkdir -p $O
for v in 0 10; do SLB_CONST_VARIANT=$v timeout 600 python tools/far_variant_err.py >> $O/err.log 2>&1; done
for v in 0 8 9 10 11 0 8 9 10 11; do
  SLB_CONST_VARIANT=$v timeout 600 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline >> $O/bench_c4_v$v.json 2>> $O/bench_c4_v$v.err; echo bench_c4_v$v=$?
done
timeout 900 python tools/setup_bench.py c3v > $O/setup_bench_c3v.jsonl 2> $O/setup_bench_c3v.err; echo setup=$?
timeout 300 python tools/nearlist_bench.py c3 c5 c5alt > $O/nearlist_morton.jsonl 2>&1; echo nl=$?
SLB_NEAR_SCAN=1 timeout 300 python tools/nearlist_bench.py c3 c5 c5alt > $O/nearlist_scan.jsonl 2>&1; echo nls=$?
cat $O/err.log
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r02v2/bench_*.json')):
    for l in open(f):
        try: d=json.loads(l)
        except Exception: continue
        print(f, round(d['ms_per_step'],3), round(d['roofline']['frac'],4))
PY

#!/bin/bash
set -u
O=gpurun_out/r02p
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py tests/test_gpu_comm.py tests/test_gpu_ragged.py tests/test_gpu_prepare.py -m gpu -q -x > $O/pytest_subset.log 2>&1; echo pytest_subset=$?
tail -n 3 $O/pytest_subset.log
for v in 1 0 1 0; do
  SLB_CONST_PRESCAN=$v timeout 600 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline >> $O/bench_c4_prescan$v.json 2>> $O/bench_c4.err; echo bench_c4_$v=$?
done
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo bench_c5=$?
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r02p/bench_*.json')):
    for l in open(f):
        try: d=json.loads(l)
        except Exception: continue
        print(f, round(d['ms_per_step'],3), round(d['roofline']['frac'],4), d.get('parity_sampled'), round(d.get('setup_s',0),2))
PY

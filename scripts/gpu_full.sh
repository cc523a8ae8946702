#!/bin/bash
# One GPU pass: determinism diagnostic, the whole GPU suite, smoke, a full bench line (with the
# CPU baseline + parity), and the ncu launch list of a short bench.   TAG=r2d bash scripts/gpu_full.sh
mkdir -p gpurun_out
TAG=${TAG:-r2}
python scripts/diag_determinism.py 8 > gpurun_out/${TAG}_det.txt 2>&1
timeout -s KILL ${TEST_TIMEOUT:-1800} python -m pytest tests -m gpu -q --timeout 400 --durations=15 ${PYTEST_ARGS} \
  > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke $?"
if [ -z "$SKIP_BENCH" ]; then
  timeout -s KILL 900 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
  python -c "import json; d=json.loads(open('gpurun_out/${TAG}_bench.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['clocks']['sm_mhz'], d.get('parity'), {k:(round(v['ms_per_launch'],3), v.get('achieved')) for k,v in d['kernels'].items()})"
fi
if [ -z "$SKIP_NCU" ]; then
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-dense \
    > gpurun_out/${TAG}_ncu_bench.log 2>&1
fi

#!/bin/bash
# Round-2 GPU iteration: GPU tests (per-test timeout), the corner diagnostic, a bench line,
# and optionally an A/B of an experiment build (X=libvmb_x.so).
#   TAG=r2b X=paper_2601_22275_b200/libvmb_x.so bash scripts/gpu_r2.sh
mkdir -p gpurun_out
TAG=${TAG:-r2}
if [ -z "$SKIP_TESTS" ]; then
  timeout -s KILL ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -x -q --timeout 300 --durations=12 ${PYTEST_ARGS} \
    > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
  tail -3 gpurun_out/${TAG}_pytest.log
fi
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python -c "import json; d=json.loads(open('gpurun_out/${TAG}_bench.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['clocks']['sm_mhz'], {k:(round(v['ms_per_launch'],3), v.get('achieved')) for k,v in d['kernels'].items()})"
if [ -n "$X" ]; then
  VMB_LIB=$PWD/$X timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_precision.py tests/test_gpu_properties.py tests/test_gpu_fuzz.py -x -q --timeout 300 -m "gpu and not slow" > gpurun_out/${TAG}_x_pytest.log 2>&1; echo "x pytest exit $?" >> gpurun_out/${TAG}_x_pytest.log
  tail -3 gpurun_out/${TAG}_x_pytest.log
  timeout -s KILL 900 bash scripts/ab.sh paper_2601_22275_b200/libvmb.so $X ${PASSES:-2} > gpurun_out/${TAG}_ab.txt 2>&1
  cat gpurun_out/${TAG}_ab.txt
fi

#!/bin/bash
# Fast GPU iteration: core parity/determinism tests, a bench line (no CPU baseline / dense), and
# the fa4 tile trace when libvmb_trace.so exists.   TAG=r2f bash scripts/gpu_iter.sh
mkdir -p gpurun_out
TAG=${TAG:-it}
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_precision.py \
  tests/test_gpu_fuzz.py tests/test_gpu_known_answers.py -x -q --timeout 300 -m "gpu and not slow" ${PYTEST_ARGS} \
  > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
tail -2 gpurun_out/${TAG}_pytest.log
python scripts/diag_determinism.py 4 > gpurun_out/${TAG}_det.txt 2>&1; grep -c "bad/rows (0," gpurun_out/${TAG}_det.txt
for i in 1 2; do
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dense --no-e2e ${BENCH_ARGS} > gpurun_out/${TAG}_bench$i.json 2> gpurun_out/${TAG}_bench$i.err
python -c "import json; d=json.loads(open('gpurun_out/${TAG}_bench$i.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['clocks']['sm_mhz'], {k:(round(v['ms_per_launch'],3), v.get('achieved')) for k,v in d['kernels'].items()})"
done
if [ -f paper_2601_22275_b200/libvmb_trace.so ]; then
  VMB_LIB=$PWD/paper_2601_22275_b200/libvmb_trace.so python scripts/trace_fa4.py > gpurun_out/${TAG}_trace.txt 2>&1; tail -3 gpurun_out/${TAG}_trace.txt
fi

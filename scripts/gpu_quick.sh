#!/bin/bash
# Quick GPU iteration: GPU tests, a short bench (no CPU baseline), optional ncu of one kernel.
#   TAG=x KREGEX=lstep_tc_kernel bash scripts/gpu_quick.sh
mkdir -p gpurun_out
TAG=${TAG:-q}
timeout -s KILL 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout -s KILL 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
if [ -n "$KREGEX" ]; then
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -c ${NCU_COUNT:-2} -o gpurun_out/prof_k_$TAG python scripts/prof_run.py --calls 1 > gpurun_out/ncu_k_$TAG.log 2>&1
fi
if [ -n "$LAUNCHES" ]; then
  timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python scripts/prof_run.py --calls 2 > /dev/null 2>&1
fi
tail -3 gpurun_out/pytest_gpu_$TAG.log
cat gpurun_out/bench_$TAG.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], {k:(round(v['ms_per_launch'],3), v.get('achieved')) for k,v in d['kernels'].items()})"

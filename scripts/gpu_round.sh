#!/bin/bash
# One GPU session: tests, bench, ncu launch list, ncu full captures.  Outputs in gpurun_out/.
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python scripts/prof_run.py --calls 2 > /dev/null 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:fa_tc_kernel -c 3 -o gpurun_out/prof_fa_$TAG python scripts/prof_run.py --calls 1 > gpurun_out/ncu_fa_$TAG.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:lstep_tc_kernel -c 2 -o gpurun_out/prof_ls_$TAG python scripts/prof_run.py --calls 1 > gpurun_out/ncu_ls_$TAG.log 2>&1
echo done

#!/bin/bash
# Final evidence session: GPU tests, the default bench (with CPU baseline), the reference arm,
# the ncu launch list and one `ncu --set full` capture per default kernel.  TAG=... bash scripts/gpu_final.sh
mkdir -p gpurun_out
TAG=${TAG:-final}
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout -s KILL 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout -s KILL 900 python bench.py --impl reference --steps 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python scripts/prof_run.py --calls 2 > /dev/null 2>&1
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:"fa2_kernel|fa4_kernel|fa_tc_kernel|fa3_kernel|lstep_tc_kernel|combine" -c 6 -o gpurun_out/prof_all_$TAG python scripts/prof_run.py --calls 1 > gpurun_out/ncu_all_$TAG.log 2>&1
echo done

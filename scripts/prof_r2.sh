#!/bin/bash
# Round-2 profiling session (one GPU): launch list of two C4 calls, then ncu --set full of every
# kernel of one bf16 C4 call and of one fp32-mode C4 call.   TAG=r2z bash scripts/prof_r2.sh
TAG=${TAG:-r2z}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
  python scripts/prof_run.py --calls 2 > gpurun_out/prof_${TAG}_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"fa2_kernel|fa3_kernel|fa4_kernel|lstep_tc_kernel|fa2_combine" -c 6 \
  -o gpurun_out/prof_bf16_${TAG} python scripts/prof_run.py > gpurun_out/prof_${TAG}_bf16.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"fa2_kernel|lstep_hl_kernel|split_hilo|fa2_combine" -c 9 \
  -o gpurun_out/prof_f32_${TAG} python scripts/prof_run.py --dtype f32 --heads 8 > gpurun_out/prof_${TAG}_f32.log 2>&1
ls -la gpurun_out/*${TAG}*

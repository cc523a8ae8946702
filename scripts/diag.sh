mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
for s in selftest rstep lstep flash fwd_f32 fwd_bf16 fwd_big; do
  echo "=== $s" >> gpurun_out/diag.log
  timeout -s KILL 150 python scripts/gpu_diag.py $s >> gpurun_out/diag.log 2>&1
  echo "exit $?" >> gpurun_out/diag.log
done

#!/bin/bash
# A/B matrix of kernel-family defaults (two passes, alternating, to average out clock drift).
mkdir -p gpurun_out
for pass in 1 2; do
  for lib in base e4; do
    L=$PWD/paper_2601_22275_b200/libvmb.so; [ $lib = e4 ] && L=$PWD/paper_2601_22275_b200/libvmb_e4.so
    for r in 2 5; do for at in 3 5; do
      VMB_LIB=$L VMB_RSTEP=$r VMB_ATTN=$at python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/mx_${lib}_r${r}_a${at}_p$pass.json 2>&1
    done; done
  done
done

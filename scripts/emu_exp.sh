for e in 64 8 4 2; do
  lib=paper_2601_22275_b200/libvmb_e$e.so; [ $e = 8 ] && lib=paper_2601_22275_b200/libvmb.so
  VMB_LIB=$PWD/$lib VMB_RSTEP=2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/emu_$e.json 2>&1
  VMB_LIB=$PWD/$lib VMB_RSTEP=1 VMB_ATTN=2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/emu_${e}_b.json 2>&1
done

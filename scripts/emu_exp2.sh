# exp2 emulation period A/B on the current defaults, two alternating passes
for pass in 1 2; do
for e in 64 8 4 2; do
  lib=paper_2601_22275_b200/libvmb_e$e.so; [ $e = 64 ] && lib=paper_2601_22275_b200/libvmb.so
  VMB_LIB=$PWD/$lib python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/emu2_${e}_$pass.json 2>/dev/null
done; done
for f in gpurun_out/emu2_*.json; do echo -n "$f "; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'], {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"; done

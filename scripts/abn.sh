# A/B/C... several library builds on the default bench, alternating:  bash scripts/abn.sh PASSES A.so B.so ...
N=$1; shift
for i in $(seq $N); do
  for lib in "$@"; do
    x=$(basename $lib .so)
    VMB_LIB=$PWD/$lib python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-dense ${BENCH_ARGS} > gpurun_out/ab_${x}_$i.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/ab_${x}_$i.json').read().strip().splitlines()[-1]); print('$x', d['ms_per_step'], d['clocks']['sm_mhz'], {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"
  done
done

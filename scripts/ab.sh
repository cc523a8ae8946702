# A/B two library builds on the default bench, alternating: bash scripts/ab.sh A.so B.so [passes]
A=$1; B=$2; N=${3:-3}
for i in $(seq $N); do
  for x in A B; do
    lib=$A; [ $x = B ] && lib=$B
    VMB_LIB=$PWD/$lib python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/ab_${x}_$i.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/ab_${x}_$i.json').read().strip().splitlines()[-1]); print('$x', d['ms_per_step'], d['clocks']['sm_mhz'], {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"
  done
done

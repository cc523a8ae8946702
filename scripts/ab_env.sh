# A/B environment settings on the default bench, alternating: bash scripts/ab_env.sh "ENV_A" "ENV_B" [passes]
A=$1; B=$2; N=${3:-3}
for i in $(seq $N); do
  for x in A B; do
    e=$A; [ $x = B ] && e=$B
    env $e python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/abe_${x}_$i.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/abe_${x}_$i.json').read().strip().splitlines()[-1]); print('$x', d['ms_per_step'], d['clocks']['sm_mhz'], {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"
  done
done

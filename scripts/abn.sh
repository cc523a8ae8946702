#!/bin/bash
# A/B/C... several library builds on the default bench, alternating: bash scripts/abn.sh PASSES A.so B.so [C.so ...]
N=$1; shift
for i in $(seq $N); do
  for lib in "$@"; do
    tag=$(basename $lib .so)
    VMB_LIB=$PWD/$lib python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/abn_${tag}_$i.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/abn_${tag}_$i.json').read().strip().splitlines()[-1]); print('$tag', d['ms_per_step'], d['clocks']['sm_mhz'], {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"
  done
done

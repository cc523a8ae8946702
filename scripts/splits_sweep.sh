# recompute split count sweep at the per-GPU loads of 1/2/4/8-GPU head sharding (C4 grid)
for H in 40 20 10 5; do for sp in 0 6 8 10 12 14 16; do
  echo "H=$H splits=$sp $(VMB_SPLITS=$sp python scripts/time_heads.py $H 20)"
done; done

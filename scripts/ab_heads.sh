# A/B two builds on the per-GPU loads of heads-sharded runs: bash scripts/ab_heads.sh A.so B.so
for pass in 1 2; do for H in 5 10 20 40; do for x in A B; do
  lib=$1; [ $x = B ] && lib=$2
  echo "$x $(VMB_LIB=$PWD/$lib python scripts/time_heads.py $H 20)"
done; done; done

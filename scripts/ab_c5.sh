# usage: bash scripts/ab_c5.sh [B.so] -- C5 epoch A/B: the in-tree libnalar.so vs another in-tree build
cd $GRAFT_REPO_ROOT
B=${1:-libnalar_base.so}
for rep in 1 2; do
  for lib in "" $B; do
    echo -n "${lib:-new} "; env NALAR_LIB_AB=$lib python scripts/c5_ab.py
  done
done

# usage: bash scripts/ab_libs.sh libA.so libB.so ... -- ab_quick.py on each in-tree build, alternating, 2 reps
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
  for lib in "$@"; do
    echo "$lib $(NALAR_LIB_AB=$lib timeout 300 python scripts/ab_quick.py 2>&1 | tail -1)"
  done
done

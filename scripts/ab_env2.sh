# usage: bash scripts/ab_env2.sh "ENV=a" "ENV=b" ... -- ab_quick.py under each environment, alternating, 2 reps
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
  for e in "$@"; do
    echo "$e $(env $e timeout 300 python scripts/ab_quick.py 2>&1 | tail -1)"
  done
done

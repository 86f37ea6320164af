# usage: bash scripts/gpu_r2.sh [pytest-k-expr|all|none] -- build, gpu tests, epoch anatomy
cd $GRAFT_REPO_ROOT
python paper_2601_05109_b200/build.py > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
if [ "$1" = "all" ]; then
  timeout -s KILL 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_sel.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_sel.log | cut -c1-600
elif [ -n "$1" ] && [ "$1" != "none" ]; then
  timeout -s KILL 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$1" > gpurun_out/pytest_sel.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_sel.log | cut -c1-600
fi
timeout -s KILL 600 python scripts/epoch_anatomy.py ${ANATOMY_ARGS} 2>&1 | tail -8 | cut -c1-900

# usage: bash scripts/gpu_all.sh -- build, gpu tests, timeline, short bench
cd $GRAFT_REPO_ROOT
python paper_2601_05109_b200/build.py > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_gpu.log | cut -c1-400
bash scripts/gpu_tl.sh 2>&1 | grep -v BUILD

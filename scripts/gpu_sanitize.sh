# usage: bash scripts/gpu_sanitize.sh -- compute-sanitizer racecheck / synccheck / memcheck over every kernel
cd $GRAFT_REPO_ROOT
python paper_2601_05109_b200/build.py > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
python -c "from oracle import build_oracle; build_oracle()"
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python scripts/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done

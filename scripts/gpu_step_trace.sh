# usage: bash scripts/gpu_step_trace.sh -- full GPU tests, then nalar_step host-phase traces (streamed / plain)
cd $GRAFT_REPO_ROOT
python paper_2601_05109_b200/build.py > /dev/null
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_r2n.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_r2n.log
NALAR_TRACE_STEP=1 NALAR_TRACE_UPLOAD=1 python scripts/e2e_stream_ab.py --steps 30 2>&1 | tail -4
NALAR_TRACE_STEP=1 NALAR_TRACE_UPLOAD=1 NALAR_STREAM_STEP=1 python - <<'PY' 2>&1 | tail -12
import sys; sys.argv=['x','--child','--steps','5']
exec(open('scripts/e2e_stream_ab.py').read())
PY

mkdir -p gpurun_out/r2
python -m pytest tests -x -q -m gpu ${PYTEST_ARGS:-} > gpurun_out/r2/pytest_gpu.log 2>&1; rc=$?
tail -30 gpurun_out/r2/pytest_gpu.log
exit $rc

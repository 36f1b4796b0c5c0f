cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_cube_sizes.py -q -x --durations=3 2>&1 | grep -E "passed|failed|Error|assert|call" | head
timeout 900 python -m pytest tests -q -m gpu -x --deselect tests/test_gpu_cube_sizes.py > gpurun_out/tests8.log 2>&1; tail -2 gpurun_out/tests8.log

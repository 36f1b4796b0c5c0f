cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/tests7.log 2>&1; tail -3 gpurun_out/tests7.log
timeout 300 python -m pytest tests/test_gpu_cube_sizes.py -q -x --durations=3 2>&1 | tail -6
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b7.json 2> gpurun_out/b7.err || tail -5 gpurun_out/b7.err
python bench.py --config 3 --steps 5 --warmup 3 > gpurun_out/mb7.json 2> gpurun_out/mb7.err || tail -5 gpurun_out/mb7.err

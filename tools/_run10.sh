cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/tests10.log 2>&1; tail -3 gpurun_out/tests10.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b10.json 2> gpurun_out/b10.err || tail -5 gpurun_out/b10.err
PWB_NO_DEVLOOP=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b10n.json 2> gpurun_out/b10n.err || tail -5 gpurun_out/b10n.err

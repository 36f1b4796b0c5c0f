cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/tests17.log 2>&1; tail -2 gpurun_out/tests17.log
PWB_SHARE_GPU=1 PWB_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/shared2.json 2> gpurun_out/shared2.err; echo "shared2 rc=$?"; tail -3 gpurun_out/shared2.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b17.json 2> gpurun_out/b17.err || tail -5 gpurun_out/b17.err

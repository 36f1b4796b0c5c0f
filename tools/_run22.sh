cd $GRAFT_REPO_ROOT
ITER_ROWS=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/it1.csv python tools/iter_latency.py > gpurun_out/it1.log 2>&1
ITER_ROWS=261 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/it261.csv python tools/iter_latency.py > gpurun_out/it261.log 2>&1
echo done

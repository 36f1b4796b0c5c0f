#!/bin/bash
# GPU box: ncu launch list of the timed region of `bench.py` (one solve,
# profile-from-start off).  ncu does not descend into the CG loop's WHILE
# conditional node, so the list is taken with PWB_NO_DEVLOOP=1 (the same
# kernels, replayed per iteration as a plain graph): shares only.
tag=${1:-final}
PWB_NO_DEVLOOP=1 PWB_PROFILE_REGION=1 ncu --profile-from-start off --metrics gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_bench.log 2>&1
echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launches.txt
gzip -f gpurun_out/${tag}_launches.csv

#!/bin/bash
# GPU box: per-launch duration list of this library's kernels over one config-1
# solve (cold-cache, serialised: shares only, never a bench value).
#   bash tools/ncu_launches.sh [tag]   ->  gpurun_out/launches_<tag>.csv
tag=${1:-cfg1}
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain_${tag}.json 2> gpurun_out/plain_${tag}.err || { echo "plain run failed"; tail -5 gpurun_out/plain_${tag}.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base function \
    -k regex:"^(k_compact|k_proj|k_plane|k_pencil|k_cg|k_zero|k_drho|k_chi0|k_dot|k_axpy|k_combine|k_normalise|k_kernel|k_transpose)" \
    -c 30000 --csv --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_${tag}.log 2>&1
echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/launches_${tag}.csv | head -20

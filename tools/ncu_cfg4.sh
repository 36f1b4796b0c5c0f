#!/bin/bash
# GPU box: ncu evidence for the configs[4] solve (the bench default).
#  1. launch list of one timed solve (gpu__time_duration per launch; shares only:
#     ncu times launches cold and serialised) -> <tag>_launches.{csv.gz,txt}
#  2. one `ncu --set full` capture (+ the FP64 tensor-pipe DMMA counters) of the
#     hot kernels at full width inside the solve -> <tag>_full.ncu-rep + summary
# ncu does not descend into the CG loop's WHILE conditional node, so both passes
# run with PWB_NO_DEVLOOP=1 (the same kernels replayed per iteration as a graph).
# Usage: bash tools/ncu_cfg4.sh <tag> [launches|full|both]
tag=${1:-r02_cfg4}
what=${2:-both}
export PWB_NO_DEVLOOP=1 PWB_PROFILE_REGION=1 PWB_REF_WORKLOAD=${PWB_REF_WORKLOAD:-}
DMMA=sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg.pct_of_peak_sustained_elapsed
if [ "$what" != full ]; then
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${tag}_launches.csv \
      python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_bench.log 2>&1
  echo "launch list rc=$?"
  python tools/launch_summary.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launches.txt
  gzip -f gpurun_out/${tag}_launches.csv
fi
if [ "$what" != launches ]; then
  ncu --profile-from-start off --set full --metrics $DMMA --import-source on --clock-control none \
      -k regex:"k_proj_coef|k_proj_apply|k_pencil|k_plane_inv|k_plane_fwd|k_cg_|k_drho" -s 30 -c 12 \
      -o gpurun_out/${tag}_full python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline \
      > gpurun_out/${tag}_full.log 2>&1
  echo "full capture rc=$?"
  python tools/ncu_summary.py gpurun_out/${tag}_full.ncu-rep > gpurun_out/${tag}_full_summary.txt 2>&1
fi

#!/bin/bash
# GPU box: ncu evidence for configs[4] (the bench default).
#  full     : one `ncu --set full` capture (+ the FP64 tensor-pipe DMMA counters) of the
#             hot kernels on configs[4] shapes (tools/kbench4.py: 64^3 sphere, 68
#             orbitals, 2 119 rows = the full width of the Sternheimer batch)
#  launches : launch list of one timed solve (gpu__time_duration per launch, shares
#             only -- ncu times launches cold and serialised), application replay
#             (no per-kernel memory save/restore), workload from $PWB_WORKLOAD
# ncu does not descend into the CG loop's WHILE conditional node, so the launch
# list runs with PWB_NO_DEVLOOP=1 (the same kernels replayed per iteration).
# Usage: bash tools/ncu_cfg4.sh <tag> [full|launches|both]
tag=${1:-r02_cfg4}
what=${2:-full}
DMMA=sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg.pct_of_peak_sustained_elapsed
if [ "$what" != launches ]; then
  timeout 900 ncu --set full --metrics $DMMA --import-source on --clock-control none \
      -k regex:"k_projw|k_proj_coef|k_proj_apply" -s 2 -c 2 \
      -o gpurun_out/${tag}_proj python tools/kbench4.py --what q --reps 1 > gpurun_out/${tag}_proj.log 2>&1
  echo "projector capture rc=$?"
  timeout 900 ncu --set full --metrics $DMMA --import-source on --clock-control none \
      -k regex:"k_pencil|k_plane" -s 3 -c 3 \
      -o gpurun_out/${tag}_h python tools/kbench4.py --what h --bands 512 --reps 1 > gpurun_out/${tag}_h.log 2>&1
  echo "H capture rc=$?"
  for r in proj h; do
    python tools/ncu_summary.py gpurun_out/${tag}_${r}.ncu-rep > gpurun_out/${tag}_${r}_summary.txt 2>&1
  done
fi
if [ "$what" != full ]; then
  PWB_NO_DEVLOOP=1 PWB_PROFILE_REGION=1 timeout 1500 ncu --replay-mode application \
      --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${tag}_launches.csv \
      python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${tag}_ncu_bench.log 2>&1
  echo "launch list rc=$?"
  python tools/launch_summary.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launches.txt
  gzip -f gpurun_out/${tag}_launches.csv
fi

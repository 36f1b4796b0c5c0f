#!/bin/bash
# GPU box: batched H apply timing at the BASELINE cube sizes (48^3 cfg1, 64^3 cfg4,
# 96^3 cfg3) and one `ncu --set full` capture of the three H kernels per size
# (reports deleted after summarising: gpurun_out/ is capped at 64 MiB).
#   bash tools/ncu_sizes.sh <tag> [sizes...]  -> gpurun_out/<tag>_h<N>_summary.txt
tag=${1:-r01}
shift
sizes=${@:-48 64 96}
declare -A SPEC=([48]="15 10 256" [64]="20 12 256" [96]="20 26 128")
for n in $sizes; do
  set -- ${SPEC[$n]}
  python tools/kbench.py --what h --alat $1 --ecut $2 --bands $3 --reps 10 2>&1 | grep -E "grid|H apply"
done
for n in $sizes; do
  set -- ${SPEC[$n]}
  ncu --set full --import-source on --clock-control none -k regex:"k_pencil|k_plane" -s 3 -c 3 \
      -o gpurun_out/${tag}_h$n python tools/kbench.py --what h --alat $1 --ecut $2 --bands $3 --reps 1 \
      > gpurun_out/${tag}_h$n.log 2>&1
  python tools/ncu_summary.py gpurun_out/${tag}_h$n.ncu-rep > gpurun_out/${tag}_h${n}_summary.txt 2>&1
  rm -f gpurun_out/${tag}_h$n.ncu-rep
done
echo done

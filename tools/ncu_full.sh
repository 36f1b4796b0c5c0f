#!/bin/bash
# GPU box: one `ncu --set full` capture of each hot kernel of the H apply and
# the projector on BASELINE configs[1] shapes (48^3 cube, 256 bands, N_occ 33),
# plus text summaries.  Usage: bash tools/ncu_full.sh <tag>
tag=${1:-r01}
python tools/kbench.py --what h --reps 2 > /dev/null 2>&1 || { echo "kbench h failed"; exit 1; }
python tools/kbench.py --what qsweep --nocc 33 --reps 1 > /dev/null 2>&1 || { echo "kbench q failed"; exit 1; }
ncu --set full --import-source on --clock-control none -k regex:"k_pencil|k_plane" -s 3 -c 3 \
    -o gpurun_out/${tag}_happly python tools/kbench.py --what h --reps 2 > gpurun_out/${tag}_happly.log 2>&1
# the 256-row projector launches are the last two of the sweep (8 sizes x 1 rep x 2 kernels)
ncu --set full --import-source on --clock-control none -k regex:"k_proj" -s 14 -c 2 \
    -o gpurun_out/${tag}_proj python tools/kbench.py --what qsweep --nocc 33 --reps 1 > gpurun_out/${tag}_proj.log 2>&1
for r in happly proj; do
  python tools/ncu_summary.py gpurun_out/${tag}_${r}.ncu-rep > gpurun_out/${tag}_${r}_summary.txt 2>&1
done
echo done

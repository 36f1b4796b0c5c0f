cd $GRAFT_REPO_ROOT
ncu --set full --import-source on --clock-control none -k regex:"k_pencil|k_plane" -s 3 -c 3 \
   -o gpurun_out/h48 python tools/kbench.py --what h --alat 15 --ecut 10 --bands 256 --reps 1 > gpurun_out/h48.log 2>&1
python tools/ncu_summary.py gpurun_out/h48.ncu-rep > gpurun_out/h48_summary.txt 2>&1
for k in k_plane_inv k_pencil_h k_plane_fwd; do
ncu -i gpurun_out/h48.ncu-rep --page source --csv -k regex:$k > gpurun_out/h48_${k}_source.csv 2>&1
done
ncu -i gpurun_out/h48.ncu-rep --page raw --csv > gpurun_out/h48_raw.csv 2>&1
rm -f gpurun_out/h48.ncu-rep

cd $GRAFT_REPO_ROOT
ncu --set full --import-source on --clock-control none -k regex:"k_pencil_hp" -s 1 -c 1 \
   -o gpurun_out/hp48 python tools/kbench.py --what h --alat 15 --ecut 10 --bands 256 --reps 1 > gpurun_out/hp48.log 2>&1
python tools/ncu_summary.py gpurun_out/hp48.ncu-rep > gpurun_out/hp48_summary.txt 2>&1
ncu -i gpurun_out/hp48.ncu-rep --page source --csv > gpurun_out/hp48_source.csv 2>&1
ncu -i gpurun_out/hp48.ncu-rep --page raw --csv > gpurun_out/hp48_raw.csv 2>&1
rm -f gpurun_out/hp48.ncu-rep

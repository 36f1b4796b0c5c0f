cd $GRAFT_REPO_ROOT
ncu --set full --import-source on --clock-control none -k regex:"k_proj" -s 10 -c 2 \
   -o gpurun_out/q261 python tools/qbench.py --rows 261 --reps 3 > gpurun_out/q261.log 2>&1
python tools/ncu_summary.py gpurun_out/q261.ncu-rep > gpurun_out/q261_summary.txt 2>&1
ncu -i gpurun_out/q261.ncu-rep --page source --csv -k regex:k_proj_coef > gpurun_out/q261_coef_source.csv 2>&1
ncu -i gpurun_out/q261.ncu-rep --page source --csv -k regex:k_proj_apply > gpurun_out/q261_apply_source.csv 2>&1
ncu -i gpurun_out/q261.ncu-rep --page raw --csv > gpurun_out/q261_raw.csv 2>&1
rm -f gpurun_out/q261.ncu-rep

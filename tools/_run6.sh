cd $GRAFT_REPO_ROOT
python tools/kbench.py --what h --alat 20 --ecut 26 --bands 128 --reps 10 2>&1 | grep -E "H apply"
for nb in 32 64 128 256 512; do python tools/kbench.py --what q --bands $nb --nocc 33 --reps 20 2>&1 | grep "Q apply" | sed "s/^/rows $nb /"; done
python tools/kbench.py --what q --bands 256 --nocc 33 --reps 5 2>&1 | grep -E "cuBLAS"
ncu --set full --import-source on --clock-control none -k regex:"k_proj" -s 6 -c 2 \
   -o gpurun_out/q33 python tools/kbench.py --what q --bands 256 --nocc 33 --reps 1 > gpurun_out/q33.log 2>&1
python tools/ncu_summary.py gpurun_out/q33.ncu-rep > gpurun_out/q33_summary.txt 2>&1
ncu -i gpurun_out/q33.ncu-rep --page source --csv -k regex:k_proj_coef > gpurun_out/q33_coef_source.csv 2>&1
ncu -i gpurun_out/q33.ncu-rep --page source --csv -k regex:k_proj_apply > gpurun_out/q33_apply_source.csv 2>&1
rm -f gpurun_out/q33.ncu-rep

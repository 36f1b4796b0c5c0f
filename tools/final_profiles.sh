#!/bin/bash
# GPU box: the round's committed measurements.
#   bench lines (config 1 default, configs[3] microbench, reference arm), the ncu
#   launch list of the timed region of `bench.py` (profile-from-start off), and
#   `ncu --set full` summaries of the hot kernels.   bash tools/final_profiles.sh <tag>
tag=${1:-final}
python bench.py > gpurun_out/${tag}_bench_cfg1.json 2> gpurun_out/${tag}_bench_cfg1.err; echo "bench rc=$?"
python bench.py --config 3 > gpurun_out/${tag}_bench_cfg3.json 2> gpurun_out/${tag}_bench_cfg3.err; echo "cfg3 rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err; echo "ref rc=$?"
PWB_PROFILE_REGION=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_bench.log 2>&1
echo "ncu launches rc=$?"
python tools/launch_summary.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launches.txt
gzip -f gpurun_out/${tag}_launches.csv
ncu --set full --import-source on --clock-control none -k regex:"k_pencil|k_plane" -s 3 -c 3 \
   -o gpurun_out/${tag}_h48 python tools/kbench.py --what h --alat 15 --ecut 10 --bands 256 --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${tag}_h48.ncu-rep > gpurun_out/${tag}_ncu_h48.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_proj" -s 10 -c 2 \
   -o gpurun_out/${tag}_q261 python tools/qbench.py --rows 261 --reps 3 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${tag}_q261.ncu-rep > gpurun_out/${tag}_ncu_q261.txt 2>&1
rm -f gpurun_out/*.ncu-rep
echo done

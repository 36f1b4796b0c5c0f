#!/bin/bash
# GPU box: SCF parity tests, both bench arms on the default config, ncu evidence
timeout 900 python -m pytest tests/test_gpu_configs.py -k scf -x -q 2>&1 | tail -3
S=$(date +%s)
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err
echo "reference rc=$? $(( $(date +%s) - S ))s"; tail -2 gpurun_out/ref.err
S=$(date +%s)
python bench.py --steps 3 --warmup 3 > gpurun_out/ours.json 2> gpurun_out/ours.err
echo "ours rc=$? $(( $(date +%s) - S ))s"; tail -2 gpurun_out/ours.err
bash tools/ncu_cfg4.sh r02_cfg4 both
ls gpurun_out

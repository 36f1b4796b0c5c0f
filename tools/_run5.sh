cd $GRAFT_REPO_ROOT
for v in "" b812m2 c166m2 d166m3; do
  echo "variant=$v"
  PWB200_VARIANT=$v python tools/kbench.py --what h --alat 20 --ecut 26 --bands 128 --reps 10 2>&1 | grep -E "H apply"
  PWB200_VARIANT=$v python tools/kbench.py --what h --alat 15 --ecut 10 --bands 256 --reps 10 2>&1 | grep -E "H apply"
done
timeout 600 python -m pytest tests/test_gpu_grids.py tests/test_gpu_baseline.py -q -x -k "grid or cfg3" 2>&1 | tail -2

#!/bin/bash
# Round-2 experiment batch g: where the configs[4] solve loses time outside full width.
#  1. H apply per band vs batch size (does the pruned plane buffer stay in L2 at small batches?)
#  2. projector cost per Q vs rows per k over 32 k blocks (mid-width regime)
#  3. per-iteration latency of the batched CG vs live rows (configs[1] state)
#  4. DRAM bytes of the H kernels at 48 vs 512 bands (ncu)
for b in 16 32 48 64 96 128 256 512 1024; do
  python tools/kbench4.py --what h --bands $b --reps 10 2>&1 | grep "H apply"
done
python tools/qmid.py --rows 1 2 4 8 16 32 66 2>&1 | tail -8
timeout 600 python tools/iter_latency.py 2>&1 | tail -12
for b in 48 512; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:"k_plane|k_pencil" -s 3 -c 3 --csv \
    python tools/kbench4.py --what h --bands $b --reps 1 > gpurun_out/g_h$b.csv 2>/dev/null
  echo "ncu bands $b rc=$?"
done

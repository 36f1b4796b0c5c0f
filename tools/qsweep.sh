#!/bin/bash
# GPU box: warm per-launch durations of the projector kernels at CG-tail sizes
python tools/kbench.py --what qsweep --nocc 33 --reps 3 > /dev/null 2>&1 || exit 1
ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum -k regex:k_proj --csv \
    python tools/kbench.py --what qsweep --nocc 33 --reps 3 > gpurun_out/qsweep.csv 2>&1
python - <<'PY'
import csv
rows = [r for r in csv.DictReader(l for l in open('gpurun_out/qsweep.csv') if l.startswith('"'))]
vals = [(r['Kernel Name'][:12], float(r['Metric Value']) / 1000) for r in rows]
per = len(vals) // 8   # launches per size (3 reps x kernels per Q)
for i, s in enumerate((1, 4, 8, 16, 32, 64, 128, 256)):
    ch = vals[i * per:(i + 1) * per]
    print(s, [(k, round(v, 1)) for k, v in ch])
PY

#!/bin/bash
export PWB_REF_WORKLOAD=/tmp/pwb_cfg4_wl PWB_WORKLOAD=/tmp/pwb_cfg4_wl
S=$(date +%s); python -m paper_2505_02319_b200.cli ground-state --config 4 --out $PWB_REF_WORKLOAD; echo "scf $(( $(date +%s) - S ))s"
for v in 16 1; do
  PWB_WIDE_MIN_ROWS=$v python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/f$v.json 2> gpurun_out/f$v.err; echo "min rows $v rc=$?"
done
python - <<'PY'
import json
for n in ("f16", "f1"):
    try:
        d = json.load(open(f"gpurun_out/{n}.json"))
    except Exception as e:
        print(n, "failed", e); continue
    h = d["kernel_ms_by_live_rows"]["projector"]
    print(n, round(d["value"]), "ms", round(d["ms_per_step"], 1), "gmres", d["gmres_iterations"],
          {k: round(v, 1) for k, v in d["roofline"]["kernel_ms"].items()})
    print("   ", {k: round(v[0] / v[1] * 1e3) for k, v in h.items()})
PY

#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_projector.py tests/test_gpu_sharded.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
export PWB_REF_WORKLOAD=/tmp/pwb_cfg4_wl PWB_WORKLOAD=/tmp/pwb_cfg4_wl
python -m paper_2505_02319_b200.cli ground-state --config 4 --out $PWB_REF_WORKLOAD > /dev/null
python tools/kbench4.py --what q --reps 5
PWB_NO_WIDE_PROJ=1 python tools/kbench4.py --what q --reps 5
for v in 32 1 56; do
  PWB_WIDE_MIN_ROWS=$v python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/w$v.json 2> gpurun_out/w$v.err; echo "min rows $v rc=$?"
done
python - <<'PY'
import json
for n in ("w32", "w1", "w56"):
    try:
        d = json.load(open(f"gpurun_out/{n}.json"))
    except Exception as e:
        print(n, "failed", e); continue
    h = d["kernel_ms_by_live_rows"]["projector"]
    print(n, round(d["value"]), "ms", round(d["ms_per_step"], 1), "gmres", d["gmres_iterations"],
          {k: round(v, 1) for k, v in d["roofline"]["kernel_ms"].items()},
          "proj frac", round(d["roofline_projector"]["frac"], 3))
    print("   ", {k: round(v[0] / v[1] * 1e3) for k, v in h.items()})
PY

#!/bin/bash
# GPU box: wide projector correctness + the whole GPU suite, A/B bench of the
# projector paths on configs[4], library cross-check
timeout 600 python -m pytest tests/test_gpu_projector.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -30
timeout 1500 python -m pytest tests -m gpu -q --ignore=tests/test_gpu_configs.py 2>&1 | tail -8
export PWB_REF_WORKLOAD=/tmp/pwb_cfg4_wl PWB_WORKLOAD=/tmp/pwb_cfg4_wl
python -m paper_2505_02319_b200.cli ground-state --config 4 --out $PWB_REF_WORKLOAD
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/wide.json 2> gpurun_out/wide.err; echo "wide rc=$?"
PWB_NO_WIDE_PROJ=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/narrow.json 2> gpurun_out/narrow.err; echo "narrow rc=$?"
python - <<'PY'
import json
for n in ("wide", "narrow"):
    try:
        d = json.load(open(f"gpurun_out/{n}.json"))
    except Exception as e:
        print(n, "failed", e); continue
    print(n, round(d["value"]), "ms", round(d["ms_per_step"], 1), "gmres", d["gmres_iterations"],
          {k: round(v, 1) for k, v in d["roofline"]["kernel_ms"].items()},
          "proj frac", round(d["roofline_projector"]["frac"], 3))
PY
python tools/libcheck.py > gpurun_out/libcheck.txt 2>&1; cat gpurun_out/libcheck.txt | tail -6

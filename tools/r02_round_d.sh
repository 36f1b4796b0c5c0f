#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_projector.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -3
export PWB_REF_WORKLOAD=/tmp/pwb_cfg4_wl PWB_WORKLOAD=/tmp/pwb_cfg4_wl
python -m paper_2505_02319_b200.cli ground-state --config 4 --out $PWB_REF_WORKLOAD > /dev/null
python tools/kbench4.py --what q --reps 5
PWB200_VARIANT=wkc32 python tools/kbench4.py --what q --reps 5
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/d16.json 2> gpurun_out/d16.err; echo "wkc16 rc=$?"
PWB200_VARIANT=wkc32 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/d32.json 2> gpurun_out/d32.err; echo "wkc32 rc=$?"
python - <<'PY'
import json
for n in ("d16", "d32"):
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
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_projw" -s 2 -c 2 \
      -o gpurun_out/r02_cfg4_proj2 python tools/kbench4.py --what q --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02_cfg4_proj2.ncu-rep > gpurun_out/r02_cfg4_proj2_summary.txt 2>&1
grep -E "duration|dmma_cycles|bank_conf|wavefronts|stalls" gpurun_out/r02_cfg4_proj2_summary.txt

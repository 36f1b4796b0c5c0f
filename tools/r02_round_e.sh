#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_projector.py tests/test_gpu_sharded.py tests/test_gpu_parity.py tests/test_gpu_dyson.py -x -q 2>&1 | tail -3
export PWB_REF_WORKLOAD=/tmp/pwb_cfg4_wl PWB_WORKLOAD=/tmp/pwb_cfg4_wl
python -m paper_2505_02319_b200.cli ground-state --config 4 --out $PWB_REF_WORKLOAD > /dev/null
python tools/kbench4.py --what q --reps 5
PWB_NO_XMAP=1 python tools/kbench4.py --what q --reps 5
python tools/kbench4.py --what h --bands 1024 --reps 5
PWB200_VARIANT=novpre python tools/kbench4.py --what h --bands 1024 --reps 5
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/e.json 2> gpurun_out/e.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/e.json"))
h = d["kernel_ms_by_live_rows"]["projector"]
print(round(d["value"]), "ms", round(d["ms_per_step"], 1), "gmres", d["gmres_iterations"],
      {k: round(v, 1) for k, v in d["roofline"]["kernel_ms"].items()},
      "proj frac", round(d["roofline_projector"]["frac"], 3))
print("   ", {k: round(v[0] / v[1] * 1e3) for k, v in h.items()})
PY
timeout 600 ncu --set full --import-source on --clock-control none --metrics sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:"k_projw" -s 2 -c 2 \
      -o gpurun_out/r02_cfg4_proj3 python tools/kbench4.py --what q --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02_cfg4_proj3.ncu-rep > gpurun_out/r02_cfg4_proj3_summary.txt 2>&1
grep -E "duration|dmma_cycles|bank_conf|dram__bytes|stalls" gpurun_out/r02_cfg4_proj3_summary.txt

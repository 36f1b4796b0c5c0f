#!/bin/bash
# GPU box: tests + kernel microbench + cfg1 bench summary (used during development)
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
python tools/kbench.py --what hq 2>&1 | grep -v cuBLAS
python tools/kbench.py --what q --bands 100 2>&1 | grep "Q apply"
python bench.py --steps 3 --warmup 2 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo bench rc=$?; tail -2 gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("value", round(d["value"]), "ms/solve", round(d["ms_per_step"], 1), "n_ham", d["n_ham_per_solve"], "gmres", d["gmres_iterations"])
r = d["roofline"]
print("H achieved GB/s", round(r["achieved"]), "frac", round(r["frac"], 3), "avg ms", round(r["avg_launch_ms"], 4), "bands", round(r["bands_per_launch"], 1))
print({k: round(v, 1) for k, v in r["kernel_ms"].items()}, "e2e", round(d["e2e"]["value"]))
PY

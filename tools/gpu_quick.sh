#!/bin/bash
# GPU box: gpu tests + one cfg1 bench summary (development loop)
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/tests.log 2>&1; tail -2 gpurun_out/tests.log > gpurun_out/tests_tail.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err || tail -5 gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("value", round(d["value"]), "step_ms", d["step_ms"], "e2e", round(d["e2e"]["value"]))
print({k: round(v, 1) for k, v in d["roofline"]["kernel_ms"].items()})
for cat, h in d["kernel_ms_by_live_rows"].items():
    print(cat, {k: round(v[0] / v[1] * 1e3, 1) for k, v in h.items()}, "us/call")
PY
cat gpurun_out/tests_tail.log

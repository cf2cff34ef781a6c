#!/bin/bash
# GPU iteration: parity tests, then the default bench line (stdout tail).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest=$?"; tail -3 gpurun_out/pytest_gpu.log
python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1
echo "bench=$?"
python - <<'PY'
import json
for ln in open("gpurun_out/bench.log"):
    if ln.startswith("{"):
        d = json.loads(ln)
        r = d.get("roofline", {})
        print("value %.4g e2e %.4g ms/step %.3f chain_frac %.4f" % (d["value"], d["e2e"]["value"], d["ms_per_step"], r.get("frac") or 0))
        for k in r.get("kernel_shares", []):
            print("  %-16s %8.2f ms / %d" % (k["kernel"], k["ms"], k["launches"]))
        print("  chain", r.get("chain_scan"))
PY

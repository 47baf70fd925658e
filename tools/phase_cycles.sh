#!/bin/bash
# Per-phase cycle breakdown of the sweep kernel (CTA 0, thread 0) on the C2
# bench workload.  Usage (GPU box): bash tools/phase_cycles.sh
mkdir -p gpurun_out
LRK_DEBUG=1 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_dbg.json 2> gpurun_out/bench_dbg.err
echo bench=$?
python - <<'PY'
import json, re
lines = [l for l in open("gpurun_out/bench_dbg.err") if "cycles/flush" in l]
if lines:
    l = lines[-1]
    parts = re.findall(r"(\S+) (\d+)\|(\d+)", l)
    print("[lrk] cycles/flush (fwd / bwd): " + " ".join(f"{n} {a}/{b}" for n, a, b in parts))
d = json.loads(open("gpurun_out/bench_dbg.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"].get("ms_per_launch"))
PY

#!/bin/bash
# One GPU round trip for kernel work (run under gpurun from the repo root):
#   bash tools/gpu_cycle.sh TAG [tests|notests] [ncu|nonu]
# gpu tests -> C2 bench line -> (optional) ncu --set full of the score kernel.
TAG=$1; T=${2:-tests}; NC=${3:-ncu}
mkdir -p gpurun_out
if [ "$T" = tests ]; then
  python -m pytest tests -m gpu -x -q > gpurun_out/t_$TAG.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/t_$TAG.log
  tail -2 gpurun_out/t_$TAG.log
fi
python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/b_$TAG.jsonl 2> gpurun_out/b_$TAG.err
python - "$TAG" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/b_{t}.jsonl").read().strip().splitlines()[-1])
    print("bench", t, "pairs/s %.3e" % d["value"], "step_ms %.4f" % d["ms_per_step"], "score_ms %.4f" % d["roofline"]["launch_ms"],
          "frac %.4f" % d["roofline"]["frac"], "nw_ms %.4f" % d["nw_only_ms"], "e2e %.3e" % (d["e2e"] or {}).get("value", 0))
except Exception as e:
    print("bench parse failed", e); print(open(f"gpurun_out/b_{t}.err").read()[-2000:])
PY
if [ "$NC" = ncu ]; then
  ncu --set full --import-source on --clock-control none -k regex:pair_kernel -c 1 -f -o gpurun_out/$TAG \
    python tools/profile_step.py --pairs 10000 --repeat 1 > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu_rc=$?"
fi

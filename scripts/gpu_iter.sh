#!/bin/bash
# Iteration loop on one B200: the TSDF parity suites, then the default bench (no CPU leg),
# then optionally an ncu --set full capture of the given kernels (regex) for source-level
# analysis. Usage: bash scripts/gpu_iter.sh <tag> [kernel-regex]
set -u
tag=${1:-it}
out=gpurun_out
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_parity_long.py -m gpu -x -q \
    > $out/tests_${tag}.log 2>&1; echo "tests rc=$?"; tail -3 $out/tests_${tag}.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > $out/bench_${tag}.json 2> $out/bench_${tag}.err
echo "bench rc=$?"
python - <<PY
import json
d = json.loads(open("$out/bench_${tag}.json").read().strip().splitlines()[-1])
r = d["roofline"]
print("value %.4g e2e %.4g ms/step %.3f frac %.4f kernel %s us/frame %s" % (d["value"], d["e2e"]["value"],
      d["ms_per_step"], r["frac"], r["kernel"], r.get("warmup_kernel_us_per_frame")))
PY
shift
for k in "$@"; do  # one capture per kernel name: launches 21-22 of it
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 20 -c 2 \
      -o $out/ncu_${tag}_${k} -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > $out/ncu_${tag}_${k}.log 2>&1
  echo "ncu $k rc=$?"
done

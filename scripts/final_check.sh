#!/bin/bash
# Round-end verification on one B200: every GPU test, smoke(), the bench (both arms),
# and the ncu launch list of the bench command.
set -u
out=gpurun_out
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q > $out/final_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 $out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $out/final_smoke.log
timeout 900 python bench.py > $out/final_bench.json 2> $out/final_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $out/final_bench_ref.json 2> $out/final_bench_ref.err; echo "bench ref rc=$?"
cut -c1-300 $out/final_bench.json; cut -c1-300 $out/final_bench_ref.json

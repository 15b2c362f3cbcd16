#!/bin/bash
# One GPU session: drop-in suites, bench (no profiler), then the ncu launch list of the
# same bench command and one --set full capture of the frame kernels.
# Usage: bash scripts/gpu_round.sh <tag>
set -u
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
(cd oracle/_ref && timeout 900 ./dropin_unit_tests > ../../$out/dropin_unit_${tag}.log 2>&1; echo "unit rc=$?" >> ../../$out/dropin_unit_${tag}.log
 timeout 900 ./dropin_acceptance > ../../$out/dropin_accept_${tag}.log 2>&1; echo "accept rc=$?" >> ../../$out/dropin_accept_${tag}.log)
timeout 900 python bench.py > $out/bench_${tag}.json 2> $out/bench_${tag}.err || { echo "bench failed"; tail -20 $out/bench_${tag}.err; exit 1; }
tail -1 $out/bench_${tag}.json
# launch list of our kernels only (the synthetic-scan generator's torch kernels excluded)
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --kernel-name-base function -k regex:'^k_' \
    --log-file $out/launches_${tag}.csv python bench.py > $out/ncu_launch_${tag}.log 2>&1
echo "launch list rc=$?"
timeout 1800 ncu --set full --clock-control none --import-source on \
    -k regex:'k_raycast_band|k_fold|k_fb_fold|k_compact|k_project_points|k_finish_pixels' \
    -s 700 -c 12 -o $out/frame_${tag} -f \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > $out/ncu_full_${tag}.log 2>&1
echo "full rc=$?"

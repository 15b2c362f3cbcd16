#!/bin/bash
# Round-2 evidence on one B200 (outputs under gpurun_out/, summaries copied to profiles/):
# the default bench (CPU baseline + parity), the reference arm, cfg3 / cfg4 / carve / cfg5
# sweep / emulated ranks, the ncu launch list of the bench command and one --set full
# capture of a frame group's kernels.
set -u
out=gpurun_out
mkdir -p $out
run() { local name=$1; shift; timeout 900 "$@" > $out/r2_$name.json 2> $out/r2_$name.err; echo "$name rc=$?"; }
run cfg2 python bench.py
run ref python bench.py --impl reference
run cfg3 python bench.py --workload cfg3
run cfg4 python bench.py --workload cfg4 --steps 7 --warmup 3 --no-e2e
run carve python bench.py --carve
run sweep python bench.py --sweep --sweep-scans 16
run emu python bench.py --emulate-ranks 1 2 4 8 --steps 3 --warmup 1 --scans-per-step 96
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base function \
    -k regex:'^k_' --log-file $out/r2_launches.csv python bench.py --steps 3 --warmup 5 --no-cpu --no-e2e \
    > $out/r2_ncu_launch.log 2>&1; echo "launch list rc=$?"
# a steady-state frame group (past the warm-up's buffer growth): fallback ordering, 16 folds,
# then the next group's projection and band
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:'k_project_points|k_finish_pixels|k_band|k_fb_count|k_fb_alloc|k_fb_bucket|k_fb_sort|k_fold' \
    -s 600 -c 22 -o $out/r2_frame -f python bench.py --steps 2 --warmup 5 --no-cpu --no-e2e > $out/r2_ncu_full.log 2>&1
echo "full rc=$?"

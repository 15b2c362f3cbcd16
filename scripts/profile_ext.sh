#!/bin/bash
# ncu evidence for the extension kernels (mesh export, occupancy carving): launch
# lists of the bench scripts and one --set full capture per kernel.
# Usage: bash scripts/profile_ext.sh <tag>
set -u
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
FRAMES=20 REPS=3 REF_REPS=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --kernel-name-base function -k regex:'^k_mesh' --log-file $out/mesh_launches_${tag}.csv \
    python scripts/bench_mesh.py > $out/ncu_mesh_launch_${tag}.log 2>&1
echo "mesh launch list rc=$?"
FRAMES=20 REPS=1 REF_REPS=0 timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_mesh_(case|own|emit)' -c 3 -o $out/mesh_${tag} -f \
    python scripts/bench_mesh.py > $out/ncu_mesh_full_${tag}.log 2>&1
echo "mesh full rc=$?"
SCANS=10 WARM=2 CPU_SCANS=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --kernel-name-base function -k regex:'^k_occ' --log-file $out/occ_launches_${tag}.csv \
    python scripts/bench_occ.py > $out/ncu_occ_launch_${tag}.log 2>&1
echo "occ launch list rc=$?"
SCANS=4 WARM=2 CPU_SCANS=0 timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_occ_(alloc|visit|fold)' -s 9 -c 3 -o $out/occ_${tag} -f \
    python scripts/bench_occ.py > $out/ncu_occ_full_${tag}.log 2>&1
echo "occ full rc=$?"

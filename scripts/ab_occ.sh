# Occupancy A/B over alternative builds (variants/<name>/libsvx_b200.so): bench_occ (cfg2
# LiDAR scans) and, with DEPTH=1, bench_depth (cfg3 depth images); then, with NCU=<tag>,
# one ncu --set full capture of the default build's k_occ_visit.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in default ${VARIANTS:-} default; do
  if [ $v = default ]; then unset SVX_LIB; else export SVX_LIB=$PWD/variants/$v/libsvx_b200.so; fi
  echo -n "$v occ " >> gpurun_out/ab_occ2.txt
  CPU_SCANS=0 timeout 300 python scripts/bench_occ.py 2>>gpurun_out/ab_occ2.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_scan'], d['value'], d['e2e']['value'])" >> gpurun_out/ab_occ2.txt
  if [ -n "${DEPTH:-}" ]; then
    echo -n "$v depth " >> gpurun_out/ab_occ2.txt
    CPU_ROWS=0 FRAMES=6 timeout 300 python scripts/bench_depth.py 2>>gpurun_out/ab_occ2.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_frame'], d['value'], d['e2e']['value'])" >> gpurun_out/ab_occ2.txt
  fi
done
unset SVX_LIB
if [ -n "${NCU:-}" ]; then
SCANS=4 WARM=2 CPU_SCANS=0 timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_occ_visit' -s 3 -c 1 -o gpurun_out/occ_visit_${NCU} -f \
    python scripts/bench_occ.py > gpurun_out/ncu_occ_visit.log 2>&1
echo "ncu rc=$?"
fi

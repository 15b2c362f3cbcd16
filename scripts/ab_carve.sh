# bench.py --carve (occupancy extension, device leg) over alternative builds: VARIANTS="a b"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in default ${VARIANTS:-} default; do
  if [ $v = default ]; then unset SVX_LIB; else export SVX_LIB=$PWD/variants/$v/libsvx_b200.so; fi
  echo -n "$v " >> gpurun_out/ab_carve.txt
  timeout 600 python bench.py --carve --no-cpu --no-e2e --steps 3 2>>gpurun_out/ab_carve.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'])" >> gpurun_out/ab_carve.txt
done

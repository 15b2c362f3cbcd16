# bench.py (device-resident leg only) over alternative builds: VARIANTS="a b" -> ms_per_step.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in ${VARIANTS:-} default ${VARIANTS:-} default; do
  if [ $v = default ]; then unset SVX_LIB; else export SVX_LIB=$PWD/variants/$v/libsvx_b200.so; fi
  echo -n "$v " >> gpurun_out/ab_bench.txt
  timeout 600 python bench.py --no-cpu --no-e2e 2>>gpurun_out/ab_bench.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['kernel_ms_per_launch'])" >> gpurun_out/ab_bench.txt
done

# bench.py e2e leg (host points) over alternative builds: VARIANTS="a b" -> gpurun_out/ab_e2e.txt
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in default ${VARIANTS:-} default; do
  if [ $v = default ]; then unset SVX_LIB; else export SVX_LIB=$PWD/variants/$v/libsvx_b200.so; fi
  echo -n "$v " >> gpurun_out/ab_e2e.txt
  timeout 600 python bench.py --no-cpu 2>>gpurun_out/ab_e2e.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])" >> gpurun_out/ab_e2e.txt
done

cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -x -q -k "sem or label or conf or raycast" > gpurun_out/tests_sempf.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/tests_sempf.log
for v in ${VARIANTS:-sempf0} default ${VARIANTS:-sempf0} default; do
  if [ $v = default ]; then unset SVX_LIB; else export SVX_LIB=$PWD/variants/$v/libsvx_b200.so; fi
  echo -n "$v "; timeout 600 python bench.py --workload cfg3 --no-cpu --no-e2e 2>>gpurun_out/ab_sem.err | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'])"
done

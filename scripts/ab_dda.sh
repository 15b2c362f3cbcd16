set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_occupancy.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo tests=$?
for v in variants/base/libsvx_b200.so variants/arr/libsvx_b200.so default; do
  if [ $v = default ]; then unset SVX_LIB; else export SVX_LIB=$PWD/$v; fi
  CPU_SCANS=1 timeout 300 python scripts/bench_occ.py >> gpurun_out/ab_occ.jsonl 2>>gpurun_out/ab_occ.err
done
unset SVX_LIB
timeout 900 python scripts/variant_bench.py variants/base/libsvx_b200.so variants/arr/libsvx_b200.so default variants/base/libsvx_b200.so variants/arr/libsvx_b200.so default > gpurun_out/ab_tsdf.txt 2>&1

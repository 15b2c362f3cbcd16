# cfg2 bench + a cfg5 sweep subset over alternative builds: VARIANTS="a b" -> gpurun_out/ab_sweep.txt
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in default ${VARIANTS:-}; do
  if [ $v = default ]; then unset SVX_LIB; else export SVX_LIB=$PWD/variants/$v/libsvx_b200.so; fi
  echo "== $v" >> gpurun_out/ab_sweep.txt
  timeout 600 python bench.py --no-cpu --no-e2e 2>>gpurun_out/ab_sweep.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', d['ms_per_step'], d['roofline']['warmup_kernel_us_per_frame'])" >> gpurun_out/ab_sweep.txt
  timeout 600 python bench.py --sweep --sweep-scans 16 --sweep-widths ${WIDTHS:-640 2560 10240} 2>>gpurun_out/ab_sweep.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'W' in d and not d['semantics']: print(d['W'], '%.3g'%d['points_per_s'], {k:round(v,1) for k,v in d['kernel_us_per_scan'].items()})
" >> gpurun_out/ab_sweep.txt
done

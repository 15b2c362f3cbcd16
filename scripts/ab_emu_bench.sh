# bench.py --emulate-ranks 1 8 over alternative builds: VARIANTS="a b" -> per-rank step ms and speed-up
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in ${VARIANTS:-} default ${VARIANTS:-} default; do
  if [ $v = default ]; then unset SVX_LIB; else export SVX_LIB=$PWD/variants/$v/libsvx_b200.so; fi
  echo -n "$v "
  timeout 900 python bench.py --emulate-ranks 1 8 --steps 5 --warmup 1 --scans-per-step 96 2>>gpurun_out/ab_emu_bench.err | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['ranks']
print(' '.join('N=%s %.3f ms x%.2f' % (k, v['max_rank_ms_per_step'], v.get('speedup_vs_1', 0)) for k, v in r.items()))"
done

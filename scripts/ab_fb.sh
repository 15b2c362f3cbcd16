#!/bin/bash
# A/B of build variants (variants/<v>/libsvx_b200.so via SVX_LIB) against the in-tree build:
# VARIANTS="g4 g8" bash scripts/ab_fb.sh -> ms per 100-frame step + per-kernel us per frame.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in default ${VARIANTS:-} default ${VARIANTS:-}; do
  if [ $v = default ]; then unset SVX_LIB; else export SVX_LIB=$PWD/variants/$v/libsvx_b200.so; fi
  echo -n "$v "
  timeout 600 python bench.py --no-cpu --no-e2e 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), {k: round(v,1) for k,v in d['roofline']['warmup_kernel_us_per_frame'].items()})"
done

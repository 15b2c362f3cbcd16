# scripts/emu_profile.py (N = 1 and 8 emulated ranks, per-rank kernel breakdown) over
# alternative builds: VARIANTS="a b" -> gpurun_out/ab_emu.txt
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in default ${VARIANTS:-}; do
  if [ $v = default ]; then unset SVX_LIB; else export SVX_LIB=$PWD/variants/$v/libsvx_b200.so; fi
  echo "== $v" >> gpurun_out/ab_emu.txt
  timeout 600 python scripts/emu_profile.py 1 8 2>>gpurun_out/ab_emu.err | cut -c1-200 >> gpurun_out/ab_emu.txt
done

cd $GRAFT_REPO_ROOT
for v in ${VARIANTS:-head} default ${VARIANTS:-head} default; do
  if [ $v = default ]; then unset SVX_LIB; else export SVX_LIB=$PWD/variants/$v/libsvx_b200.so; fi
  echo -n "$v "; timeout 300 python bench.py --sweep --sweep-scans ${SCANS:-16} --sweep-widths ${WIDTHS:-80 2560 16384} 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l: continue
    x=json.loads(l)
    if 'W' in x and not x['semantics']: print(x['W'], '%.3g'%x['points_per_s'], end='  ')
print()"
done

for pct in 0 45; do
  for n in 32768 131072; do
  SWATTN_ROUTE_PCT=$pct N=$n ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/attend_once.py 2>/dev/null | grep -v "^==" | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
tot=0
for r in rows[1:]:
    if r[h.index('Metric Name')]!='gpu__time_duration.sum': continue
    v=float(r[vi].replace(',',''))
    nm=r[ki].split('(')[0][-60:]
    if 'swattn' in r[ki] or 'kernel' in nm: print('  ', nm, v); tot+=v
print('total', tot)
" | sed "s/^/pct=$pct n=$n /"
  done
done

python tools/rank1_probe.py && ncu --clock-control none --metrics gpu__time_duration.sum --csv python tools/rank1_probe.py 2>/dev/null | python3 -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
data=[(r[ki].split('(')[0][:40], float(r[vi].replace(',',''))/1e6) for r in rows[1:]]
half=len(data)//2
tot=0
for k,v in data[half:]:
    print('%8.3f  %s'%(v,k)); tot+=v
print('total %.3f ms over %d kernels'%(tot, len(data)-half))
"

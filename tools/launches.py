import csv, collections, sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>5 and not r[0].startswith('==')]
hdr=rows[0]; data=rows[1:]
ik=hdr.index('Kernel Name'); iv=hdr.index('Metric Value'); iu=hdr.index('Metric Unit')
agg=collections.defaultdict(lambda:[0,0.0]); tot=0
for r in data:
    name=r[ik].split('(')[0].replace('void ','').replace('unnamed>::','')
    v=float(r[iv].replace(',','')); u=r[iu]
    v = v/1000 if u=='ns' else v*1000 if u=='ms' else v
    agg[name][0]+=1; agg[name][1]+=v; tot+=v
for k,(n,t) in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"{k:40s} n={n:3d} total={t:8.1f}us avg={t/n:7.2f}us share={t/tot*100:5.1f}%")
print('total us per forward', round(tot,1))

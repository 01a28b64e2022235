import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
agg=collections.defaultdict(lambda:[0,0.0]); order=[]
for r in rows[hdr+1:]:
    if len(r)<=vi: continue
    v=float(r[vi].replace(',','')); u=r[ui]
    v = v/1000 if u=='ns' else (v if u=='us' else v*1000)
    k=r[ki][:80]; agg[k][0]+=1; agg[k][1]+=v; order.append((k,v))
tot=sum(v[1] for v in agg.values())
for k,(n,t) in sorted(agg.items(), key=lambda x:-x[1][1])[:int(sys.argv[2]) if len(sys.argv)>2 else 20]:
    print(f"{t:10.1f} us {100*t/tot:5.1f}% n={n:4d} avg={t/n:8.1f}  {k}")
print('total us', tot)
if len(sys.argv)>3:
    for k,v in order[:int(sys.argv[3])]: print(f"   {v:8.1f} {k}")

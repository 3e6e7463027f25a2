import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None;agg=collections.defaultdict(lambda:[0,0.0]); shapes=collections.defaultdict(collections.Counter)
for r in rows:
    if r and r[0]=='ID': hdr=r;continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get('Metric Name')=='gpu__time_duration.sum':
            k=d['Kernel Name'][:50];v=float(d['Metric Value'].replace(',',''))
            agg[k][0]+=1;agg[k][1]+=v
            shapes[k][d['Grid Size']]+=v
tot=sum(v[1] for v in agg.values())
for k,v in sorted(agg.items(),key=lambda x:-x[1][1]):
    print(v[0],round(v[1]/1e3,1),'us',f"{100*v[1]/tot:.1f}%",k)
    for g,t in shapes[k].most_common(6): print('      grid',g,round(t/1e3,1),'us')

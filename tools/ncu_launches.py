import csv, collections, sys
for f in sys.argv[1:]:
    rows=list(csv.reader(open(f)))
    h=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
    hdr=rows[h]; ik=hdr.index('Kernel Name'); im=hdr.index('Metric Name'); iv=hdr.index('Metric Value'); iid=hdr.index('ID')
    d=collections.defaultdict(dict)
    for r in rows[h+1:]:
        if len(r)>iv: d[(r[iid],r[ik][:50])][r[im]]=float(r[iv].replace(',',''))
    agg=collections.defaultdict(list)
    for (i,k),m in d.items(): agg[k].append(m)
    print(f)
    for k,ms in agg.items():
        n=len(ms); avg={mm: sum(x[mm] for x in ms)/n for mm in ms[0]}
        print(f"  {n:3d} {k:50s} " + " ".join(f"{mm.split('__')[1][:18]}={v:.4g}" for mm,v in avg.items()))

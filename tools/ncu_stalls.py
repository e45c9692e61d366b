"""Per-instruction warp-stall breakdown from an ncu --page source --csv export (dev tool).

    ncu -i rep.ncu-rep --page source --csv --print-source sass > src.csv; python tools/ncu_stalls.py src.csv
"""
import csv, sys, collections
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; ix={h:i for i,h in enumerate(hdr)}
tot=collections.Counter(); per=[]
for r in rows[2:]:
    if len(r)<len(hdr): continue
    s=0
    for h in ('stall_long_sb','stall_short_sb','stall_barrier','stall_mio','stall_wait','stall_lg','stall_math','stall_drain'):
        try: v=float(r[ix[h]] or 0)
        except: v=0
        tot[h]+=v
    try: samp=float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except: samp=0
    per.append((samp, r[ix["Address"]], r[ix["Source"]][:70], r[ix['stall_long_sb']]))
print(tot.most_common())
per.sort(key=lambda x:-x[0])
S=sum(p[0] for p in per)
for p in per[:25]: print("%5.1f%%"%(100*p[0]/S), p[1], p[2], 'long_sb', p[3])

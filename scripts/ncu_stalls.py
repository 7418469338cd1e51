"""Per-source-line stall-sample shares (with the top stall reasons) from
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass`."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 28
agg = collections.OrderedDict(); fname=''; hdr=None
for r in rows:
    if r and r[0]=='File Path': fname=r[1].split('/')[-1]; continue
    if r and r[0]=='Line No': hdr=r; continue
    if hdr and len(r)>=8 and r[2]=='-':
        try: key=(fname,int(r[0]))
        except ValueError: continue
        a=agg.setdefault(key,[r[1],0.0,0.0,collections.Counter()])
        a[1]+=float(r[7] or 0); a[2]+=float(r[6] or 0)
        for i,h in enumerate(hdr):
            if h.startswith('stall_') and 'Not Issued' not in h and i<len(r):
                try: a[3][h]+=float(r[i] or 0)
                except ValueError: pass
tot=sum(a[2] for a in agg.values()); toti=sum(a[1] for a in agg.values())
print('samples %d, warp insts %.3g' % (tot, toti))
for (f,ln),a in sorted(agg.items(), key=lambda kv:-kv[1][2])[:top_n]:
    top=', '.join(f'{k[6:]}:{int(v)}' for k,v in a[3].most_common(3))
    print('%-10s %4d %5.1f%% smp %5.1f%% inst | %s | %s'%(f[:10],ln,100*a[2]/tot,100*a[1]/toti,top,a[0].strip()[:64]))

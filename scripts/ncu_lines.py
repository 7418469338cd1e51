"""Per-source-line instruction / stall-sample shares from
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass` output."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = collections.OrderedDict()
fname = ''
hdr = None
for r in rows:
    if r and r[0] == 'File Path':
        fname = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No':
        hdr = r; continue
    if hdr and len(r) >= 8 and r[2] == '-':   # source-line aggregate rows
        try:
            key = (fname, int(r[0]))
        except ValueError:
            continue
        a = agg.setdefault(key, [r[1], 0.0, 0.0])
        a[1] += float(r[7] or 0); a[2] += float(r[6] or 0)
tot_i = sum(a[1] for a in agg.values()); tot_s = sum(a[2] for a in agg.values())
print('total warp insts %.3g, samples %d' % (tot_i, tot_s))
for (f, ln), a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print('%-12s %5d  %5.1f%% inst  %5.1f%% smp  %s' % (f, ln, 100 * a[1] / tot_i, 100 * a[2] / max(tot_s, 1), a[0].strip()[:100]))

"""Hot spots of an `ncu --page source --csv --print-source sass` dump: barrier/mbarrier waits and
every line above a sample threshold.  Usage: sass_hot.py dump.csv [threshold_pct]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1]))); thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.4
hdr = [r for r in rows if r and r[0] == 'Address'][0]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows if len(r) == len(hdr) and r[0] != 'Address']
stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
tot = sum(int(r[ix['# Samples']]) for r in data)
mx = max(int(r[ix['Instructions Executed']]) for r in data)
print('total samples', tot, 'lines', len(data))
for n, r in enumerate(data):
    src = r[ix['Source']]; sm = int(r[ix['# Samples']])
    if 'BAR.' in src or 'SYNCS' in src or sm > tot * thr / 100:
        t = sorted(stalls, key=lambda s: -int(r[ix[s]] or 0))[:2]
        print(n, f"{100*sm/tot:5.2f}%", f"x{int(r[ix['Instructions Executed']]):>10d}",
              ' '.join(f"{s[6:]}:{r[ix[s]]}" for s in t).ljust(36), src[:70])

"""Top-sampled SASS lines of an `ncu --page source --csv` dump (handles several functions)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
wa = float(sys.argv[2]); ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 40
hdr = [r for r in rows if r and r[0] == 'Address'][0]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows if len(r) == len(hdr) and r[0] != 'Address']
tot = sum(int(r[ix['# Samples']]) for r in data)
toti = sum(int(r[ix['Instructions Executed']]) for r in data)
stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
agg = {s: sum(int(r[ix[s]] or 0) for r in data) for s in stalls}
print('lines', len(data), 'inst/warp-attempt', round(toti / wa, 1))
print({k[6:]: round(100 * v / tot, 1) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:9]})
top = sorted(range(len(data)), key=lambda n: -int(data[n][ix['# Samples']]))[:ntop]
for n in sorted(top):
    r = data[n]; sm = int(r[ix['# Samples']]); t = max(stalls, key=lambda s: int(r[ix[s]] or 0))
    print(n, f"{100*sm/tot:5.2f}%", f"f={int(r[ix['Instructions Executed']])/wa:6.3f}", t[6:].ljust(10), r[ix['Source']][:80])

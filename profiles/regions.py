"""Sample share of SASS regions split where the execution frequency class changes.
Usage: regions.py dump.csv chunks   (chunks = executions of a once-per-chunk instruction)"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1]))); chunks = float(sys.argv[2])
hdr = [r for r in rows if r and r[0] == 'Address'][0]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows if len(r) == len(hdr) and r[0] != 'Address']
tot = sum(int(r[ix['# Samples']]) for r in data)
prev = None; start = 0
def flush(a, b, key):
    sm = sum(int(r[ix['# Samples']]) for r in data[a:b]); ins = sum(int(r[ix['Instructions Executed']]) for r in data[a:b])
    if sm > tot * 0.002:
        print(f"{a:5d}-{b:5d} {key:3s} {100*sm/tot:6.2f}%  inst/attempt {ins/chunks/8:6.1f}  {data[a][ix['Source']][:50]}")
for n in range(len(data)):
    f = int(data[n][ix['Instructions Executed']]) / chunks
    key = 'hi' if f >= 0.5 else ('mid' if f >= 0.05 else 'lo')
    if key != prev:
        if prev is not None: flush(start, n, prev)
        prev = key; start = n
flush(start, len(data), prev)

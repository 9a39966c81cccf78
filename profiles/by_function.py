"""Instructions and stall samples per CUDA function / source line, from
`ncu -i REPORT --page source --csv --print-source cuda,sass > dump.csv`.
usage: python profiles/by_function.py dump.csv WARP_ROWS [function-to-list-lines-of]"""
import collections
import csv
import re
import sys


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


def main(path, warp_rows, detail=None):
    rows = list(csv.reader(open(path)))
    cur, per, hdr = None, collections.defaultdict(dict), None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            ie, ismp = hdr.index("Instructions Executed"), hdr.index("# Samples")
            continue
        if hdr and r and r[0].isdigit():
            per[cur][int(r[0])] = (num(r[ie]), num(r[ismp]), r[1])
    src = open("paper_1004_0024_b200/csrc/kernels_strand.cu").read().split("\n")
    marks = []
    for i, line in enumerate(src, 1):
        m = re.match(r"(?:__device__|__global__).*?(\w+)\(", line)
        if m:
            marks.append((i, m.group(1)))

    def func_of(line):
        name = "?"
        for i, n in marks:
            if i <= line:
                name = n
        return name

    agg, smp = collections.Counter(), collections.Counter()
    for f, d in per.items():
        for ln, (e, s, _) in d.items():
            key = f + ":" + (func_of(ln) if f == "kernels_strand.cu" else "*")
            agg[key] += e
            smp[key] += s
    ts = sum(smp.values())
    for k, v in agg.most_common(30):
        print(f"{k:50s} inst/row {v / warp_rows:7.2f}  samples {100 * smp[k] / ts:5.1f}%")
    print("total inst/row", sum(agg.values()) / warp_rows)
    if detail:
        d = per["kernels_strand.cu"]
        lines = [(ln, e, s, t) for ln, (e, s, t) in d.items() if func_of(ln) == detail]
        for ln, e, s, t in sorted(lines, key=lambda x: -x[1])[:45]:
            print(ln, f"{e / warp_rows:6.2f} {100 * s / ts:5.1f}%", t.strip()[:100])


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), sys.argv[3] if len(sys.argv) > 3 else None)

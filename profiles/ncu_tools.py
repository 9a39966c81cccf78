"""Helpers to digest `ncu --page source/raw --csv` dumps (used for the summaries in profiles/)."""
import collections
import csv
import sys


def load_source(path):
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    return hdr, data, ix


def segments(path, warp_attempts, min_freq=0.01):
    """Consecutive SASS lines grouped by execution count; prints inst/attempt and stall share."""
    hdr, data, ix = load_source(path)
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(int(r[ix["# Samples"]]) for r in data)
    toti = sum(int(r[ix["Instructions Executed"]]) for r in data)
    print(f"total samples {tot}  instructions {toti}  inst/warp-attempt {toti / warp_attempts:.1f}")
    agg = {s: sum(int(r[ix[s]] or 0) for r in data) for s in stalls}
    print("  ".join(f"{s[6:]} {100 * v / tot:.1f}%" for s, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    seg, prev = [], None
    merged = collections.OrderedDict()

    def flush():
        if not seg:
            return
        f, n = seg[0][1], len(seg)
        smp = sum(s[2] for s in seg)
        if f < min_freq and smp < 0.003 * tot:
            return
        ops = collections.Counter(s[3].split()[1] if s[3].startswith("@") else s[3].split()[0] for s in seg)
        st = collections.Counter()
        for s in seg:
            st.update(s[4])
        key = (n, tuple(sorted(ops.items())))
        m = merged.setdefault(key, dict(first=seg[0][0], copies=0, inst=0.0, smp=0, st=collections.Counter(), ops=ops, n=n))
        m["copies"] += 1
        m["inst"] += n * f
        m["smp"] += smp
        m["st"].update(st)

    for n, r in enumerate(data):
        f = round(int(r[ix["Instructions Executed"]]) / warp_attempts, 3)
        if prev is None or abs(f - prev) > 0.03 * max(f, prev, 0.001):
            flush()
            seg = []
        seg.append((n, f, int(r[ix["# Samples"]]), r[ix["Source"]], {s: int(r[ix[s]] or 0) for s in stalls}))
        prev = f
    flush()
    for m in merged.values():
        top = ", ".join(f"{k[6:]} {100 * v / tot:.1f}" for k, v in m["st"].most_common(3) if v)
        print(f"L{m['first']:4d} n={m['n']:4d} x{m['copies']:2d} inst/att={m['inst']:6.2f} smp={100 * m['smp'] / tot:5.1f}% "
              f"[{top}] {dict(m['ops'].most_common(6))}")


def raw(path, keys):
    rows = list(csv.reader(open(path)))
    for h, u, v in zip(rows[0], rows[1], rows[2]):
        if any(h.startswith(k) for k in keys):
            print(h, u, v)


if __name__ == "__main__":
    if sys.argv[1] == "seg":
        segments(sys.argv[2], float(sys.argv[3]))
    else:
        raw(sys.argv[2], sys.argv[3:])

"""Stall-reason breakdown of a SASS region of an ncu source page: python scripts/ncu_region.py src.csv first_pat last_pat"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; data = rows[2:]
i_src = h.index("Source"); i_ex = h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ri = [h.index(c) for c in reasons]
def region(a, b):
    tot = collections.Counter(); ex = 0
    for x in data[a:b]:
        for c, i in zip(reasons, ri):
            tot[c] += int(x[i] or 0)
        ex += int(x[i_ex] or 0)
    return tot, ex
start = next(k for k, x in enumerate(data) if sys.argv[2] in x[i_src])
end = next(k for k in range(start + 1, len(data)) if sys.argv[3] in data[k][i_src])
tot, ex = region(start, end)
all_, exa = region(0, len(data))
print(f"region {start}-{end}: {sum(tot.values())} of {sum(all_.values())} samples; instr executed {ex} of {exa}")
for c, v in tot.most_common(12):
    print(f"   {c:24s} {v:7d}")
# top lines per reason
for c in [c for c, _ in tot.most_common(4)]:
    i = h.index(c)
    top = sorted(range(start, end), key=lambda k: -int(data[k][i] or 0))[:6]
    print(c, [(k, int(data[k][i] or 0), data[k][i_src].strip()[:40]) for k in top])

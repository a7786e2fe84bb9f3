"""Per-region instruction/stall breakdown of an ncu SASS source page (gpurun_out/<tag>_src.csv.gz).
python scripts/src_regions.py TAG [ctas*warps]   — regions are split at SASS lines whose execution
count changes by > 30 %; prints each region's instructions per warp-CTA and top stall reasons."""
import collections, csv, gzip, io, sys
rows = list(csv.reader(io.StringIO(gzip.open(f"gpurun_out/{sys.argv[1]}_src.csv.gz", "rt").read())))
h = rows[1]; data = rows[2:]
ie, isrc, iss = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 3072 * 16
tot_s = sum(int(x[iss] or 0) for x in data)
cur, start = None, 0
regions = []
for k, x in enumerate(data + [["0"] * len(h)]):
    n = int(x[ie] or 0)
    if cur is None or (n == 0) != (cur == 0) or (cur and abs(n - cur) > 0.3 * cur):
        if cur is not None:
            regions.append((start, k))
        cur, start = n, k
for a, b in regions:
    ex = sum(int(x[ie] or 0) for x in data[a:b]); smp = sum(int(x[iss] or 0) for x in data[a:b])
    if smp < 0.01 * tot_s:
        continue
    st = collections.Counter()
    for x in data[a:b]:
        for c in reasons:
            st[c[6:]] += int(x[h.index(c)] or 0)
    print(f"{a:5d}-{b:5d} n/line={int(data[a][ie] or 0) / norm:8.1f} inst/warp={ex / norm:8.1f} samples={smp / tot_s:5.1%} "
          f"{[(c, round(v / smp, 2)) for c, v in st.most_common(3)]}  {data[a][isrc].strip()[:40]}")

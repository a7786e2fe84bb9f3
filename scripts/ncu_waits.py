"""List every mbarrier try-wait site of a single-kernel ncu report with its execution count and the
samples on the retry branch (who waits on what)."""
import csv, io, subprocess, sys
src = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]; data = rows[2:]
i_s = h.index("Warp Stall Sampling (All Samples)"); i_src = h.index("Source"); i_ex = h.index("Instructions Executed")
for k, x in enumerate(data):
    s = x[i_src]
    if "TRYWAIT" in s or "UTCHMMA" in s or "UTMALDG" in s or "UTCBAR" in s or "NANOSLEEP" in s or "UTCQMMA" in s:
        nxt = data[k + 1]
        print(f"{x[0][-5:]} ex={int(x[i_ex] or 0):9d} {s.strip()[:58]:58s} | next {int(nxt[i_s] or 0):6d} {nxt[i_src].strip()[:28]}")

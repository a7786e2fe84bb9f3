"""Summarise a single-kernel ncu --set full report: key metrics + top stalled SASS lines."""
import csv, io, subprocess, sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]; idx = {h: i for i, h in enumerate(hdr)}
r = rows[2]
print("==", r[idx["Kernel Name"]][:80])
for k in ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum", "dram__bytes_read.sum",
          "dram__bytes_write.sum", "l1tex__m_xbar2l1tex_read_bytes.sum.per_second", "launch__registers_per_thread"]:
    if k in idx: print("   ", k, r[idx[k]])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]; data = rows[2:]
i_s = h.index("Warp Stall Sampling (All Samples)"); i_src = h.index("Source"); i_ex = h.index("Instructions Executed")
tot = sum(int(x[i_s] or 0) for x in data)
print("   total stall samples", tot)
for k, x in sorted(enumerate(data), key=lambda t: -int(t[1][i_s] or 0))[:ntop]:
    prev = data[k - 1][i_src].strip()[:50] if k else ""
    print(f"   {int(x[i_s]):7d} {int(x[i_ex] or 0):9d}  {x[i_src].strip()[:60]:60s} | prev: {prev}")

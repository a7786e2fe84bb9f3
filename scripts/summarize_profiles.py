"""Summarise a round's ncu captures (scripts/profile_round.sh) into profiles/<tag>_*.

python scripts/summarize_profiles.py <tag>   (reads gpurun_out/<tag>_*)
Writes profiles/<tag>_launches_summary.csv, profiles/<tag>_ncu_full_summary.json,
profiles/<tag>_stalls_<kernel>.txt and refreshes profiles/ncu_traffic.json (read by bench.py).
"""
import collections, csv, glob, gzip, io, json, os, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles")

# ---- launch list
rows = [r for r in csv.reader(open(os.path.join(src, f"{tag}_launches.csv"))) if len(r) > 10]
h = rows[0]
ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
acc = collections.OrderedDict()
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    name = r[ik].split("(")[0]
    if "rowwise" in name:   # the bench's standalone-solver line, not part of the attention step
        continue
    v = float(r[iv].replace(",", ""))
    unit = r[h.index("Metric Unit")]
    us = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[unit]
    a = acc.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(a[1] for a in acc.values())
with open(os.path.join(dst, f"{tag}_launches_summary.csv"), "w") as f:
    f.write(f"# {tag} launch list: ncu --metrics gpu__time_duration.sum --clock-control none "
            "(bench.py --steps 2 --warmup 3 --no-cpu-baseline, config 2 Gaussian)\n"
            "# cold-cache, serialised per-launch times; compare SHARES with bench.py's live event times\n"
            "kernel,launches,mean_us,share\n")
    for k, (n, us) in sorted(acc.items(), key=lambda t: -t[1][1]):
        f.write(f"{k},{n},{us / n:.1f},{us / tot:.3f}\n")

# ---- full captures
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_gmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum",
        "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic"]
summary, traffic = {}, {}
NAMES = {"tau_kernel": "tau_sm100", "out_kernel": "out_sm100", "dkdv_kernel": "dkdv_sm100", "dq_kernel": "dq_sm100"}
for raw in sorted(glob.glob(os.path.join(src, f"{tag}_full_*_raw.csv"))):
    case = os.path.basename(raw)[len(tag) + 6:-8]
    rows = list(csv.reader(open(raw)))
    hdr, units, r = rows[0], rows[1], rows[2]
    idx = {x: i for i, x in enumerate(hdr)}
    ent = {"kernel": r[idx["Kernel Name"]]}
    for k in KEYS:
        if k in idx:
            ent[k] = r[idx[k]] + (" " + units[idx[k]] if units[idx[k]] else "")
    def num(k):
        v = float(r[idx[k]].replace(",", ""))
        u = units[idx[k]]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    ent["dram_bytes_per_launch"] = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    summary[case] = ent
    if case in NAMES:
        tp = "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
        traffic[NAMES[case]] = {"dram_bytes_per_launch": ent["dram_bytes_per_launch"],
                                "tensor_pipe_pct": float(r[idx[tp]]) if tp in idx else None,
                                "ncu_kernel": ent["kernel"].split("(")[0], "round": tag,
                                "input": "config 2 Gaussian (scripts/run_fwd.py gaussian 1.0 bwd)"}
    # stall breakdown from the source page
    gz = raw[:-8] + "_src.csv.gz"
    if os.path.exists(gz):
        srows = list(csv.reader(io.StringIO(gzip.open(gz, "rt").read())))
        sh = srows[1] if "Source" not in srows[0] else srows[0]
        data = srows[srows.index(sh) + 1:]
        i_src = sh.index("Source")
        reasons = [c for c in sh if c.startswith("stall_") and "Not Issued" not in c]
        tot = collections.Counter()
        for x in data:
            for c in reasons:
                tot[c] += int(x[sh.index(c)] or 0)
        i_s = sh.index("Warp Stall Sampling (All Samples)")
        allsum = sum(int(x[i_s] or 0) for x in data)
        with open(os.path.join(dst, f"{tag}_stalls_{case}.txt"), "w") as f:
            f.write(f"# {ent['kernel'][:100]}\n# stall samples by reason (of {allsum})\n")
            for c, v in tot.most_common(14):
                f.write(f"{c:28s} {v:9d}  {v / max(1, allsum):.3f}\n")
            f.write("# top SASS lines by samples\n")
            for x in sorted(data, key=lambda x: -int(x[i_s] or 0))[:30]:
                f.write(f"{int(x[i_s] or 0):8d}  {x[i_src].strip()[:90]}\n")
json.dump(summary, open(os.path.join(dst, f"{tag}_ncu_full_summary.json"), "w"), indent=1)
json.dump(traffic, open(os.path.join(dst, "ncu_traffic.json"), "w"), indent=1)
print(json.dumps(summary, indent=1))

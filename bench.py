#!/usr/bin/env python
"""bench.py — α-entmax attention fwd+bwd (AdaSplash hot path) on B200.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W [--impl reference]``;
N > 1 is launched under torch.distributed.run (one rank per GPU, NCCL).  Rank 0 prints ONE
JSON line.

Workload (BASELINE.json configs[1], the config the metric is quoted on):
  B=4 H=12 N=8192 d=64 α=1.5 non-causal bf16, n_iter = 3, Gaussian inputs with
  query variance σ² = 6 (the paper's benchmark generator) — per rank.  Weak scaling:
  every rank runs its own B·H heads (distinct seeds per rank), no collective on the data path.
One step = entmax_attn_fwd (τ + output + tables) + entmax_attn_bwd (δ, 𝒦 tables, dK/dV, dQ)
over the whole batch.  value = effective TFLOP/s over all ranks, FA convention
14·d·ΣV per fwd+bwd with V = visible (query, key) pairs of the non-skipped blocks
(SURVEY §8d).  Inputs (201 MB per rank) exceed the 126 MB L2, so no explicit flush.
``--sweep`` adds the planted-block-sparsity sweep (Fig. 1 analogue) as extra keys.

The oracle (test infrastructure, oracle/) is executed only for the ``cpu_baseline`` leg and
for ``--impl reference``.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "α-entmax attn fwd+bwd ms & effective TFLOP/s vs sparsity/seq len, tensor-pipe %"
UNIT = "TFLOP/s"
CFG = dict(B=4, H=12, N=8192, d=64, alpha=1.5, causal=False, n_iter=3)
WORKLOAD = "config2: B=4 H=12 N=8192 d=64 alpha=1.5 non-causal bf16 n_iter=3, gaussian q~N(0,6) k,v,dO~N(0,1)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--sweep", action="store_true", default=True,
                    help="add the planted block-sparsity sweep (default on; --no-sweep to skip)")
    ap.add_argument("--no-sweep", dest="sweep", action="store_false")
    ap.add_argument("--suite", action="store_true", help="add configs 3-5 (seq-len / alpha / long-context lines)")
    ap.add_argument("--no-rowwise", action="store_true", help="skip the standalone row-wise solver line")
    ap.add_argument("--gpt2", action="store_true", help="add the GPT-2-124M training-step line (NEXT-4)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--N", type=int, default=CFG["N"])
    ap.add_argument("--d", type=int, default=CFG["d"])
    ap.add_argument("--B", type=int, default=CFG["B"])
    ap.add_argument("--H", type=int, default=CFG["H"])
    ap.add_argument("--alpha", type=float, default=CFG["alpha"])
    ap.add_argument("--causal", action="store_true")
    ap.add_argument("--n-iter", type=int, default=CFG["n_iter"])
    ap.add_argument("--gen", default="gaussian", choices=["gaussian", "planted"])
    ap.add_argument("--rho", type=float, default=1.0)
    return ap.parse_args()


# ------------------------------------------------------------------------------ helpers
def visible_pairs_in_active_blocks(mask, N, causal, Br=128, Bc=128):
    """ΣV: visible (query, key) pairs inside blocks with M_ij = 1 (host-side accounting)."""
    m = mask.reshape(-1, mask.shape[-2], mask.shape[-1]).cpu().numpy().astype(np.int64)
    Tr, Tc = m.shape[1:]
    rows = np.minimum(N, (np.arange(Tr) + 1) * Br) - np.arange(Tr) * Br
    cols = np.minimum(N, (np.arange(Tc) + 1) * Bc) - np.arange(Tc) * Bc
    area = rows[:, None] * cols[None, :]
    if causal:
        area = np.zeros((Tr, Tc), dtype=np.int64)
        for i in range(Tr):
            q = np.arange(i * Br, min(N, (i + 1) * Br))
            for j in range(min(Tc, i + 1)):
                k0, k1 = j * Bc, min(N, (j + 1) * Bc)
                area[i, j] = np.clip(q[:, None] - np.arange(k0, k1)[None, :] + 1, 0, 1).sum()
    return int((m * area[None]).sum())


def total_visible_pairs(N, causal):
    return N * (N + 1) // 2 if causal else N * N


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        "hw_slowdown": 0x0000000000000008, "sw_thermal_slowdown": 0x0000000000000020,
        "hw_thermal_slowdown": 0x0000000000000040, "hw_power_brake_slowdown": 0x0000000000000080,
        "sw_power_cap": 0x0000000000000004,
    }

    def __init__(self, device_index=0, period=0.002):
        self.samples, self.reasons, self.period = [], set(), period
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - depends on the box
            self.err = repr(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": float(self.max_mhz),
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return dict(hbm=d.get("hbm_gbs", 6650.0), bf16=d.get("bf16_tflops", 1590.0),
                    bf16_sustained=d.get("bf16_tflops_sustained", 1400.0), src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sustained=1400.0, src="fallback (B200_PROFILING.md)")


def ncu_traffic(kernel, key="dram_bytes_per_launch"):
    """DRAM bytes per launch (or another field, e.g. tensor_pipe_pct) of `kernel` from the committed
    ncu --set full summary (profiles/ncu_traffic.json), if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        d = json.load(fh)
    ent = d.get(kernel)
    return None if ent is None else ent.get(key)


# ------------------------------------------------------------------------------ oracle legs
def oracle_sample(cfg, seed=0, rows=512):
    """One bounded sample of the workload on the host: one head, `rows` query rows of
    fwd (τ mirror, O, O⁽²⁾, mask rows) + bwd (dQ rows, their dK/dV contributions).
    Returns (seconds, effective flops of the sample, description)."""
    import oracle as O
    import synth
    import torch
    spec = synth.HeadSpec(cfg["gen"], rho=cfg.get("rho", 1.0))
    q, k, v, do = spec.head(cfg["N"], cfg["d"], seed, 0, 0)
    q, k, v, do = [torch.from_numpy(x).to(torch.bfloat16).double().numpy() for x in (q, k, v, do)]
    rsel = np.arange(rows)
    t0 = time.perf_counter()
    fw = O.attn_fwd(q, k, v, cfg["alpha"], cfg["causal"], cfg["n_iter"], rows=rsel)
    tau_all = np.zeros(cfg["N"])
    tau_all[rsel] = fw["tau"]
    O.block_mask(q, k, tau_all, cfg["alpha"], cfg["causal"], row_blocks=range(rows // 128))
    O.attn_bwd(q, k, v, do, tau_all, cfg["alpha"], cfg["causal"], rows=rsel)
    dt = time.perf_counter() - t0
    pairs = sum(min(r + 1, cfg["N"]) if cfg["causal"] else cfg["N"] for r in rsel)
    flops = 14.0 * cfg["d"] * pairs
    return dt, flops, f"1 head x {rows} query rows of N={cfg['N']} d={cfg['d']} (fwd+bwd, float64 numpy)"


def cpu_cores():
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        n = max((i.get("num_threads", 1) for i in info), default=1)
        return int(n)
    except Exception:
        return len(os.sched_getaffinity(0))


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    times, flops = [], 0.0
    desc = ""
    for s in range(args.warmup + args.steps):
        dt, fl, desc = oracle_sample(cfg, seed=s % 3, rows=256)
        if s >= args.warmup:
            times.append(dt)
            flops = fl
    ms = statistics.median(times) * 1e3
    value = flops / (ms * 1e-3) / 1e12
    cores = cpu_cores()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample": desc},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ native arm
def main():
    args = parse()
    cfg = dict(B=args.B, H=args.H, N=args.N, d=args.d, alpha=args.alpha, causal=args.causal,
               n_iter=args.n_iter, gen=args.gen, rho=args.rho)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist
    import paper_2502_12082_b200 as P
    import synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        world = max(world, 1)
    # ENTMAX_BENCH_SHARE_GPU=1 / ENTMAX_BENCH_BACKEND=gloo: test hook to exercise the multi-rank path
    # on a one-GPU box (ranks share cuda:0, gloo carries the barriers and the max-over-ranks timing)
    if os.environ.get("ENTMAX_BENCH_SHARE_GPU") == "1":
        local = local % torch.cuda.device_count()
    backend = os.environ.get("ENTMAX_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    B, H, N, d = cfg["B"], cfg["H"], cfg["N"], cfg["d"]
    spec = synth.HeadSpec(cfg["gen"], rho=cfg["rho"])
    # weak scaling: rank r owns heads r*B*H .. (r+1)*B*H-1 of a (world·B)×H batch
    qn, kn, vn, don = synth.make_inputs(B * world, H, N, d, seed=1234, spec=spec,
                                        heads=range(rank * B * H, (rank + 1) * B * H))
    host = [torch.from_numpy(x).to(torch.bfloat16).reshape(B, H, N, d).pin_memory() for x in (qn, kn, vn, don)]
    q, k, v, do = [t.to(dev) for t in host]
    torch.cuda.synchronize()

    alpha, causal, n_iter = cfg["alpha"], cfg["causal"], cfg["n_iter"]
    assert P.impl_for(q) == 1, "bench must run the tcgen05 path"
    fw = P.entmax_attn_fwd(q, k, v, alpha, causal, n_iter)
    ws_f = torch.empty(P.workspace_bytes(q, causal)[0], dtype=torch.uint8, device=dev)
    ws_b = torch.empty(P.workspace_bytes(q, causal)[1], dtype=torch.uint8, device=dev)
    grads = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v))

    def step():
        P.entmax_attn_fwd(q, k, v, alpha, causal, n_iter, out=fw, workspace=ws_f)
        P.entmax_attn_bwd(q, k, v, do, fw, alpha, causal, grads=grads, workspace=ws_b)

    stream = torch.cuda.current_stream(dev)

    def timed(fn, steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=dev if backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms / steps

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # ---- main timed region (device-resident inputs).  The library's per-kernel events would sit
    # between the kernels and stop the programmatic-dependent-launch overlap, so the per-kernel
    # breakdown comes from a second, separately timed pass.
    with ClockSampler(local) as clk:
        ms_step = timed(step, args.steps)
    P.profile_reset()
    P.profile_enable(True)
    ms_step_profiled = timed(step, args.steps)
    P.profile_enable(False)
    prof = P.profile_collect()

    # ---- e2e: every step copies its inputs host (pinned) → device and its gradients device → host,
    # inside the timed region, through the public API.  The copies run on two copy streams (one per
    # direction), double-buffered, so step k+1's H2D and step k's D2H overlap step k's kernels (a
    # prefetching input pipeline); the timed region starts before the first H2D and ends after the
    # last D2H.
    host_g = [[torch.empty_like(g, device="cpu").pin_memory() for g in grads] for _ in range(2)]
    dbuf = [(q, k, v, do), tuple(torch.empty_like(t) for t in (q, k, v, do))]
    gbuf = [grads, tuple(torch.empty_like(g) for g in grads)]
    cstream = torch.cuda.Stream(dev)      # H2D
    dstream = torch.cuda.Stream(dev)      # D2H (the other copy engine: both directions overlap)

    def e2e_run(steps):
        ev = lambda: torch.cuda.Event(enable_timing=False)
        h2d_done, comp_done, d2h_done = [ev(), ev()], [ev(), ev()], [None, None]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        cstream.wait_event(e0)
        dstream.wait_event(e0)

        def h2d(i):
            with torch.cuda.stream(cstream):
                for dst, src in zip(dbuf[i % 2], host):
                    dst.copy_(src, non_blocking=True)
                h2d_done[i % 2].record(cstream)

        h2d(0)
        for i in range(steps):
            c = i % 2
            stream.wait_event(h2d_done[c])
            if d2h_done[c] is not None:
                stream.wait_event(d2h_done[c])          # step i-2's gradients have left gbuf[c]
            qq, kk, vv, dd = dbuf[c]
            P.entmax_attn_fwd(qq, kk, vv, alpha, causal, n_iter, out=fw, workspace=ws_f)
            P.entmax_attn_bwd(qq, kk, vv, dd, fw, alpha, causal, grads=gbuf[c], workspace=ws_b)
            comp_done[c].record(stream)
            if i + 1 < steps:
                if i >= 1:
                    cstream.wait_event(comp_done[1 - c])   # dbuf[1-c] is free once step i-1 is done
                h2d(i + 1)
            with torch.cuda.stream(dstream):
                dstream.wait_event(comp_done[c])
                for dst, src in zip(host_g[c], gbuf[c]):
                    dst.copy_(src, non_blocking=True)
                d2h_done[c] = ev()
                d2h_done[c].record(dstream)
        stream.wait_stream(cstream)
        stream.wait_stream(dstream)
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=dev if backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms / steps

    e2e_run(2)
    ms_e2e = e2e_run(max(4, args.steps))
    h2d = sum(t.numel() * t.element_size() for t in host)
    d2h = sum(t.numel() * t.element_size() for t in host_g[0])
    # the gradients that reached the host are the kernels' (spot check, outside the timed region)
    assert torch.equal(host_g[1][2].to(dev), gbuf[1][2]), "e2e D2H mismatch"

    # ---- accounting (outside the timed region)
    step()
    torch.cuda.synchronize()
    pairs = visible_pairs_in_active_blocks(fw.mask, N, causal)
    density = pairs / (B * H * total_visible_pairs(N, causal))
    eff_flops_rank = 14.0 * d * pairs
    value = eff_flops_rank * world / (ms_step * 1e-3) / 1e12
    e2e_value = eff_flops_rank * world / (ms_e2e * 1e-3) / 1e12
    launches_per_step = sum(n for n, _ in prof.values()) / args.steps

    # roofline of the dominant kernel: MMA flops it issues per launch / its mean duration
    peaks = load_peaks()
    kern_ms = {name: tot / n for name, (n, tot) in prof.items()}
    dom = max(prof, key=lambda n: prof[n][1])
    vis_all = B * H * total_visible_pairs(N, causal)
    mma_flops = {
        # one streaming pass of S = QKᵀ + the nkb/4 warm-up tiles it re-streams (the paper's Alg. 3 would
        # issue 1 + T passes; fallback tiers, taken by a few % of CTAs, are not counted)
        "tau_sm100": (1.0 + (1 / 3 if d == 128 else 1 / 4)) * 2.0 * d * vis_all,   # warm-up nkb/4 (nkb/3 at d=128)
        "out_sm100": 6.0 * d * pairs,                             # S, P·V, U·V on candidate blocks
        "dkdv_sm100": 8.0 * d * pairs,                            # Sᵀ, dPᵀ, Pᵀ·dO, dSᵀ·Q
        "dq_sm100": 6.0 * d * pairs,                              # S, dP, dS·K
    }
    roof = None
    if dom in mma_flops:
        ach = mma_flops[dom] / (kern_ms[dom] * 1e-3) / 1e12
        roof = {"kernel": dom, "bound": "tensor", "achieved": ach, "peak": peaks["bf16_sustained"],
                "unit": "TFLOP/s", "frac": ach / peaks["bf16_sustained"], "traffic": ncu_traffic(dom),
                "peak_src": peaks["src"] + " bf16_tflops_sustained (kernel timed inside the step)",
                "algorithmic": "MMA flops issued per launch (see DESIGN.md §Roofline)"}
    kernels = {n: {"launches_per_step": c / args.steps, "ms_per_launch": kern_ms[n],
                   "share": tot / sum(t for _, t in prof.values()),
                   **({"achieved_tflops": mma_flops[n] / (kern_ms[n] * 1e-3) / 1e12,
                       "frac_of_sustained_bf16": mma_flops[n] / (kern_ms[n] * 1e-3) / 1e12 / peaks["bf16_sustained"],
                       "ncu_tensor_pipe_pct": ncu_traffic(n, "tensor_pipe_pct")} if n in mma_flops else {})}
               for n, (c, tot) in prof.items()}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": WORKLOAD if (cfg["gen"] == "gaussian" and N == 8192) else
                   f"B={B} H={H} N={N} d={d} alpha={alpha} causal={causal} n_iter={n_iter} gen={cfg['gen']} rho={cfg['rho']}",
                   "global_batch": B * world, "heads": H, "seq_len": N, "head_dim": d, "alpha": alpha,
                   "causal": causal, "n_iter": n_iter, "parallelism": f"heads-sharded x{world} (weak)",
                   "l2": "inputs 201 MB/rank > 126 MB L2 (no flush)", "block_density": density},
        "fwd_bwd_ms": ms_step, "effective_tflops": value, "ms_per_step_with_kernel_events": ms_step_profiled,
        "gpu_launches": int(round(launches_per_step * args.steps)),
        "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": ms_e2e, "h2d_bytes_per_step": h2d,
                "pipeline": "H2D of step k+1 and D2H of step k on two copy streams, double-buffered",
                "d2h_bytes_per_step": d2h},
        "roofline": roof, "kernels": kernels, "clocks": clk.summary(),
    }

    if args.sweep and rank == 0:
        line["sweep"] = run_sweep(P, synth, torch, dev, cfg, args)
    if args.suite and rank == 0:
        line["suite"] = run_suite(P, synth, torch, dev, args)
    if not args.no_rowwise and rank == 0:
        line["next1_rowwise"] = run_rowwise(P, synth, torch, dev, peaks)
    if args.gpt2 and rank == 0:
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        import gpt2_step
        line["next4_gpt2"] = gpt2_step.run()

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        dt, fl, desc = oracle_sample(dict(cfg), seed=0, rows=4096)
        line["cpu_baseline"] = {"value": fl / dt / 1e12, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
                                "sample": desc, "seconds": dt}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()          # rank 0's extra lines (sweep, row-wise, CPU baseline) finish first
        dist.destroy_process_group()


def run_sweep(P, synth, torch, dev, cfg, args):
    """Fig. 1 analogue: fwd+bwd time vs planted block density (B·H heads, same N, d, α)."""
    out = []
    B, H, N, d = cfg["B"], cfg["H"], cfg["N"], cfg["d"]
    for rho in (1.0, 0.5, 0.25, 0.1, 0.05, 0.02, 1 / 64):
        spec = synth.HeadSpec("planted", rho=rho)
        qn, kn, vn, don = synth.make_inputs(B, H, N, d, seed=7, spec=spec)
        q, k, v, do = [torch.from_numpy(x).to(torch.bfloat16).to(dev) for x in (qn, kn, vn, don)]
        fw = P.entmax_attn_fwd(q, k, v, cfg["alpha"], cfg["causal"], cfg["n_iter"])
        g = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v))

        def f():
            P.entmax_attn_fwd(q, k, v, cfg["alpha"], cfg["causal"], cfg["n_iter"], out=fw)

        def fb():
            f()
            P.entmax_attn_bwd(q, k, v, do, fw, cfg["alpha"], cfg["causal"], grads=g)

        for _ in range(3):
            fb()
        torch.cuda.synchronize()
        res = {}
        for name, fn in (("fwd", f), ("fwd_bwd", fb)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(max(5, args.steps // 2)):
                fn()
            e1.record()
            torch.cuda.synchronize()
            res[name] = e0.elapsed_time(e1) / max(5, args.steps // 2)
        # the paper's unmasked variant (NEXT-2: every visible block, no tables) on the same inputs
        fwu = P.entmax_attn_fwd(q, k, v, cfg["alpha"], cfg["causal"], cfg["n_iter"], masked=False)

        def fbu():
            P.entmax_attn_fwd(q, k, v, cfg["alpha"], cfg["causal"], cfg["n_iter"], out=fwu, masked=False)
            P.entmax_attn_bwd(q, k, v, do, fwu, cfg["alpha"], cfg["causal"], grads=g)

        res["fwd_bwd_unmasked"] = _time(torch, fbu, max(5, args.steps // 2))
        fb()
        torch.cuda.synchronize()
        pairs = visible_pairs_in_active_blocks(fw.mask, N, cfg["causal"])
        dens = pairs / (B * H * total_visible_pairs(N, cfg["causal"]))
        # dense softmax reference on the same box (cuDNN / flash SDPA, FA-convention flops)
        sd = sdpa_ms(torch, q, k, v, do, cfg["causal"]) if rho == 1.0 else None
        out.append({"rho_target": rho, "block_density": dens, "fwd_ms": res["fwd"], "fwd_bwd_ms": res["fwd_bwd"],
                    "fwd_bwd_ms_unmasked": res["fwd_bwd_unmasked"],
                    "eff_tflops_fwd_bwd": 14.0 * d * pairs / (res["fwd_bwd"] * 1e-3) / 1e12,
                    **({"sdpa_fwd_bwd_ms": sd} if sd else {})})
        del q, k, v, do, fw, fwu, g
    return out


def _time(torch, fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def run_rowwise(P, synth, torch, dev, peaks, rows=8192, n=8192):
    """the paper's standalone solver benchmark (Gaussian rows,
    n = 8192, Halley-bisection T = 3 vs bisection; paper H100: 2.38 ms vs 36.67 ms).  HBM-bound:
    algorithmic bytes = one read of s + one write of p (+ τ) per call; roofline against the
    measured burst copy bandwidth (the kernel is timed alone)."""
    s_np, dp_np = synth.rowwise_scores(rows, n, seed=0)
    out = {"workload": f"[{rows} x {n}] s~N(0,1) (P:L246), alpha=1.5", "paper_h100_ms":
           {"halley_bisection_T3": 2.38, "torch_bisection": 36.67}}
    for dt_name, dt in (("f32", torch.float32), ("bf16", torch.bfloat16)):
        s = torch.from_numpy(s_np).to(dt).to(dev)
        dp = torch.from_numpy(dp_np).to(dt).to(dev)
        esz = s.element_size()
        byt = rows * n * esz * 2 + rows * 4
        p, _ = P.entmax_rowwise_fwd(s, 1.5, 3)
        P.profile_reset()
        P.profile_enable(True)
        ms_h = _time(torch, lambda: P.entmax_rowwise_fwd(s, 1.5, 3), 20)
        P.profile_enable(False)
        prof = P.profile_collect()
        k_ms = prof["rowwise_fwd"][1] / prof["rowwise_fwd"][0]
        ms_b = _time(torch, lambda: P.entmax_rowwise_fwd(s, 1.5, 23, halley=False), 20)
        ms_bwd = _time(torch, lambda: P.entmax_rowwise_bwd(p, dp, 1.5), 20)
        ach = byt / (k_ms * 1e-3) / 1e9
        out[dt_name] = {
            "halley_T3_ms": ms_h, "bisection_T23_ms": ms_b, "bwd_ms": ms_bwd,
            "roofline": {"kernel": "rowwise_fwd", "bound": "hbm", "achieved": ach, "peak": peaks["hbm"],
                         "unit": "GB/s", "frac": ach / peaks["hbm"],
                         "traffic": ncu_traffic("rowwise_fwd") if dt_name == "f32" else None,
                         "algorithmic": f"{byt} B/launch (read s + write p + tau)"},
            "bwd_gbs": (rows * n * esz * 3) / (ms_bwd * 1e-3) / 1e9}
        del s, dp, p
    return out


def run_suite(P, synth, torch, dev, args):
    """BASELINE.json configs 3-5 (one line each): fwd and fwd+bwd ms and effective TFLOP/s."""
    cases = [("config3", 8, 12, 512, 64, 1.5, False), ("config3", 8, 12, 8192, 64, 1.5, False),
             ("config4", 8, 12, 1024, 64, 1.25, True), ("config4", 8, 12, 1024, 64, 1.5, True),
             ("config4", 8, 12, 1024, 64, 2.0, True),
             ("config5", 1, 16, 32768, 128, 1.5, True), ("config5", 1, 16, 65536, 128, 1.5, True)]
    out = []
    for name, B, H, N, d, alpha, causal in cases:
        qn, kn, vn, don = synth.make_inputs(B, H, N, d, seed=99, spec=synth.HeadSpec("gaussian"))
        q, k, v, do = [torch.from_numpy(x).to(torch.bfloat16).to(dev) for x in (qn, kn, vn, don)]
        del qn, kn, vn, don
        fw = P.entmax_attn_fwd(q, k, v, alpha, causal, 3)
        g = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v))
        it = 3 if N >= 32768 else 10
        f_ms = _time(torch, lambda: P.entmax_attn_fwd(q, k, v, alpha, causal, 3, out=fw), it)

        def fb():
            P.entmax_attn_fwd(q, k, v, alpha, causal, 3, out=fw)
            P.entmax_attn_bwd(q, k, v, do, fw, alpha, causal, grads=g)
        fb_ms = _time(torch, fb, it)
        # the same step captured once in a CUDA graph and replayed (no per-launch CPU overhead)
        gms = None
        try:
            s_ = torch.cuda.Stream(dev)
            s_.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(s_):
                fb()
            torch.cuda.current_stream(dev).wait_stream(s_)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                fb()
            gms = _time(torch, graph.replay, it)
            del graph
        except Exception:
            pass
        pairs = visible_pairs_in_active_blocks(fw.mask, N, causal)
        sd = sdpa_ms(torch, q, k, v, do, causal, iters=it)
        out.append({"config": name, "B": B, "H": H, "N": N, "d": d, "alpha": alpha, "causal": causal,
                    "block_density": pairs / (B * H * total_visible_pairs(N, causal)),
                    "fwd_ms": f_ms, "fwd_bwd_ms": fb_ms, "fwd_bwd_ms_cuda_graph": gms,
                    "eff_tflops_fwd": 4.0 * d * pairs / (f_ms * 1e-3) / 1e12,
                    "eff_tflops_fwd_bwd": 14.0 * d * pairs / (fb_ms * 1e-3) / 1e12,
                    "sdpa_fwd_bwd_ms": sd})
        del q, k, v, do, fw, g
        torch.cuda.empty_cache()
    return out


def sdpa_ms(torch, q, k, v, do, causal, iters=10):
    """Same-box dense softmax attention (torch SDPA; cuDNN/flash backend) fwd+bwd time."""
    import torch.nn.functional as F
    qq, kk, vv = [t.detach().clone().requires_grad_(True) for t in (q, k, v)]

    def fb():
        o = F.scaled_dot_product_attention(qq, kk, vv, is_causal=causal)
        o.backward(do)

    try:
        for _ in range(3):
            fb()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fb()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters
    except Exception:
        return None


if __name__ == "__main__":
    main()

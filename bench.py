#!/usr/bin/env python
"""bench.py -- VDMC 4-motif per-vertex counting on B200: motifs/s and edges/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl reference]

One step = the whole hot path over the synthetic graph of the chosen
BASELINE config: device symmetrise + order + relabel (vdmc_build_graph_edges on edges
already resident in HBM), plan, enumerate/classify/accumulate (vdmc_count), finalise, and
for N > 1 the NCCL reduce of the per-rank partial matrices to rank 0.  Steps are timed
with CUDA events on the launching stream; L2 is flushed (256 MiB write) between steps;
the job time is the max over ranks.  `e2e` repeats the step through the public API from
pinned host edges, including H2D of the edges and D2H of the count matrix.

--impl reference runs the oracle (oracle/, plain C + OpenMP) on the host cores on bounded
samples of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import graphgen as G  # noqa: E402

METRIC = "4-motif per-vertex counting: motifs/sec and edges/sec at 1/2/4/8 B200"
# per motif, the neighbour entry yielding its last member (4 B) plus one u64
# read-modify-write (16 B) per counter atomic that reaches L2.  B_k,eff = 4 + 16 x (L2 atomic /
# reduction requests per motif), the requests measured by ncu on the same workload
# (profiles/ncu_traffic.json, lts__t_requests_op_{red,atom}.sum); B_k = 4 + 16 (k-1) when no
# member is aggregated.
FALLBACK_HBM = 6650.0             # B200_PROFILING.md fallback, only if MEASURED_PEAKS.json is absent


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="cfg4", choices=sorted(G.CONFIGS))
    p.add_argument("--k", type=int, default=None)
    p.add_argument("--impl", default="vdmc", choices=["vdmc", "reference"])
    p.add_argument("--kind", default="directed", choices=["directed", "undirected"],
                   help="motif kind (undirected = SURVEY 8(f) NEXT-1); the headline is directed")
    p.add_argument("--e2e-steps", type=int, default=2)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=15.0)
    p.add_argument("--edges", action="store_true",
                   help="time edge-level counts (SURVEY 8(f) NEXT-2, vdmc_count_edges) instead of vertex counts")
    p.add_argument("--virtual-parts", type=int, default=0,
                   help="planner balance on one GPU: time each of G cost-balanced slices (vdmc_plan) back "
                        "to back and print max/mean (not the contract line)")
    return p.parse_args()


def peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def ncu_counters(config, k, kind):
    """Per-launch ncu counters of the enumeration kernel on this workload (committed summary,
    profiles/ncu_traffic.json, written by tools/ncu_counters.py from one --set full capture)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(f"{config}-k{k}" + ("-undirected" if kind == "undirected" else ""))
    except Exception:
        return None


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-i", str(gpu_index), "-lms", "200"], stdout=self.tmp,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.tmp.flush()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.tmp.name) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx.append(float(parts[2]))
                except ValueError:
                    continue
                for nm, val in zip(names, parts[5:9]):
                    if val.lower().startswith("active"):
                        reasons.add(nm)
        os.unlink(self.tmp.name)
        if not sm:
            return None
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_sample(g, k, seconds, seed=0):
    """Time the oracle (as it stands) on a bounded random sample of the workload: vertices
    are relabelled by a random permutation and the oracle counts every connected k-set whose
    minimum new label lies in [0, hi) -- a uniform sample of roots.  Returns (sets/s, sets,
    seconds, hi, cores)."""
    import oracle
    oracle.build()
    n = g[0]
    perm = np.random.default_rng(seed).permutation(n)
    gr = G.relabel(g, perm)
    cores = cpu_cores()
    hi = max(1, n // 100000)
    while True:
        t = time.perf_counter()
        _, sets = oracle.count_esu(gr, k, 0, hi, threads=cores, return_sets=True)
        dt = time.perf_counter() - t
        if dt >= seconds * 0.5 or hi >= n:
            return sets / dt, sets, dt, hi, cores
        grow = max(2.0, min(50.0, seconds * 0.7 / max(dt, 1e-3)))
        hi = min(n, int(hi * grow) + 1)


def run_reference(args, world, rank):
    k = args.k or G.CONFIGS[args.config]["k"][-1]
    if rank != 0:
        return
    g = G.make_config(args.config)
    per_step = max(2.0, min(args.cpu_seconds, 150.0 / max(1, args.steps + args.warmup)))
    rate, sets, dt, hi, cores = oracle_sample(g, k, per_step)   # calibration = first warm-up
    for _ in range(max(0, args.warmup - 1)):
        oracle_sample(g, k, per_step)
    import oracle
    n = g[0]
    perm = np.random.default_rng(0).permutation(n)
    gr = G.relabel(g, perm)
    times, tot = [], 0
    for _ in range(args.steps):
        t = time.perf_counter()
        _, s = oracle.count_esu(gr, k, 0, hi, threads=cores, return_sets=True)
        times.append(time.perf_counter() - t)
        tot += s
    T = sum(times)
    value = tot / T
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "motifs/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {G.CONFIGS[args.config]['desc']}", "k": k, "n": n,
                   "arcs": int(g[1].size), "parallelism": "host cores (oracle, OpenMP)"},
        "cpu_baseline": {"value": value, "unit": "motifs/s", "cores": cores, "kind": "oracle", "cpu": cpu_model(),
                         "sample": f"ESU over roots with random label < {hi} of {n} ({tot // args.steps} sets/step)"},
        "e2e": {"value": value, "unit": "motifs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_virtual_parts(args):
    """SURVEY §8(e) on one GPU: the G slices of vdmc_plan counted one after another; the
    slowest slice bounds a G-GPU step, so max/mean is the planner's balance."""
    import torch
    from paper_2201_11655_b200 import vdmc
    k = args.k or G.CONFIGS[args.config]["k"][-1]
    n, src, dst = G.make_config(args.config)
    g = vdmc.Graph(n, torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda())
    G_ = args.virtual_parts
    parts = g.plan(k, G_)
    full = g.count(k, kind=args.kind)
    tm = {}
    g.count(k, kind=args.kind, timings=tm)
    acc = torch.zeros_like(full)
    per = []
    for rep in range(max(1, args.steps)):
        ms = []
        for sl in parts:
            t = {}
            out = g.count(k, work=sl, kind=args.kind, timings=t)
            if rep == 0:
                acc += out
            ms.append(t["enum"])
            del out
        per.append(ms)
    assert torch.equal(acc, full), "slice partials do not sum to the full matrix"
    ms = [min(x) for x in zip(*per)]
    line = {"mode": "virtual-parts", "config": args.config, "k": k, "kind": args.kind, "parts": G_,
            "slices": parts, "slice_enum_ms": ms, "max_over_mean": max(ms) / (sum(ms) / len(ms)),
            "full_enum_ms": tm["enum"], "ideal_speedup": tm["enum"] / max(ms), "sum_equals_full": True}
    print(json.dumps(line), flush=True)
    g.close()


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    if args.virtual_parts:
        run_virtual_parts(args)
        return
    import torch
    import torch.distributed as dist
    from paper_2201_11655_b200 import vdmc

    k = args.k or G.CONFIGS[args.config]["k"][-1]
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        comm = vdmc.Comm(device=local)   # libvdmc's own NCCL communicator (vdmc_count_distributed)
    stream = torch.cuda.current_stream()
    args.warmup = max(1, args.warmup)

    n, src, dst = G.make_config(args.config)
    arcs = int(src.size)
    d_src = torch.from_numpy(src).to(dev)
    d_dst = torch.from_numpy(dst).to(dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)   # 256 MiB > 126 MB L2

    def step(e_src, e_dst, out_host=None, tm=None):
        g = vdmc.Graph(n, e_src, e_dst, device=local)
        if args.edges:
            out = g.count_edges(k, kind=args.kind, timings=tm)
            if out_host is not None:
                out_host.copy_(out, non_blocking=True)
            return g, out
        if world > 1:
            out = vdmc.count_distributed(g, k, comm, root=0, kind=args.kind)
        else:
            out = g.count(k, kind=args.kind, timings=tm)
        if out_host is not None and out is not None:
            out_host.copy_(out, non_blocking=True)
        return g, out

    def motifs_of(out):
        colsum = out.sum(dim=0).cpu().numpy().view(np.uint64).astype(object)
        if args.edges:   # sum over edges = sum over sets of their G_U edge count: checked, not divided
            return edge_sum_to_motifs(colsum)
        return int(sum(colsum)) // k

    edge_census = None
    if args.edges:   # the motif count itself from one vertex count (outside any timed region)
        if world > 1:
            raise SystemExit("--edges runs on one GPU")
        g0 = vdmc.Graph(n, d_src, d_dst, device=local)
        vc = g0.count(k, kind=args.kind).sum(dim=0).cpu().numpy().view(np.uint64).astype(object)
        g0.close()
        ids = vdmc.class_ids(k, args.kind)
        pairs = [(i, j) for i in range(k) for j in range(k) if i != j]
        nb = len(pairs)
        ecls = [len({tuple(sorted(pairs[b])) for b in range(nb) if (int(c) >> (nb - 1 - b)) & 1}) for c in ids]
        edge_census = ([int(x) // k for x in vc], ecls)

    def edge_sum_to_motifs(colsum):
        census, ecls = edge_census
        assert [int(x) for x in colsum] == [c * e for c, e in zip(census, ecls)], "edge census identity"
        return sum(census)

    for _ in range(args.warmup):
        g, out = step(d_src, d_dst)
        g.close()
        del out
    torch.cuda.synchronize()

    # ---- timed region: K steps, device events per step, L2 flushed between steps
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local) if rank == 0 else None
    launches0 = vdmc.kernel_launches()
    step_ms, enum_ms, phase_ms, motifs = [], [], [], []
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        tm = {} if world == 1 else None
        e0.record(stream)
        g, out = step(d_src, d_dst, tm=tm)
        e1.record(stream)
        torch.cuda.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        build_ms = g.info["build_ms"]
        maxdeg = g.info["max_degree"]
        if tm:
            enum_ms.append(tm["enum"])
            phase_ms.append({"build": build_ms, **tm})
        if out is not None:
            motifs.append(motifs_of(out))   # from this step's own result (outside the timed events)
        g.close()
        del out
    launches = vdmc.kernel_launches() - launches0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop() if clocks else None
    T = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(T, op=dist.ReduceOp.MAX)
    T_ms = float(T.item())

    # ---- e2e: pinned host edges -> public API -> host count matrix
    h_src = torch.from_numpy(src).pin_memory()
    h_dst = torch.from_numpy(dst).pin_memory()
    C = vdmc.num_classes(k, args.kind)
    rows = n
    if args.edges:
        g0 = vdmc.Graph(n, d_src, d_dst, device=local)
        rows = g0.ntasks
        g0.close()
    h_out = torch.empty((rows, C), dtype=torch.int64).pin_memory() if rank == 0 else None

    def e2e_step():
        s_dev = h_src.to(dev, non_blocking=True)
        d_dev = h_dst.to(dev, non_blocking=True)
        g, out = step(s_dev, d_dev, out_host=h_out)
        return g

    g = e2e_step()
    torch.cuda.synchronize()
    g.close()
    if world > 1:
        dist.barrier()
    e2e_ms = []
    for _ in range(args.e2e_steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g = e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
        g.close()
    E = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(E, op=dist.ReduceOp.MAX)
    E_ms = float(E.item()) / max(1, args.e2e_steps)
    if rank == 0:
        e2e_motifs = motifs_of(h_out)
        assert e2e_motifs == motifs[0], "e2e result differs from the device-resident steps"

    # accumulator word of the count (the library's rule, vdmc.h acc64): 32-bit when no (vertex,
    # class) count can reach 2^32 -- 6 maxdeg^3 (k = 4) / 2 maxdeg^2 (k = 3); the output is u64
    acc_dtype = "u32" if (6 * maxdeg ** 3 if k == 4 else 2 * maxdeg ** 2) < 2 ** 32 and k in (3, 4) \
        and not args.edges else "u64"
    if rank == 0:
        assert len(set(motifs)) == 1, f"motif totals differ between steps: {motifs}"
        total_sets = motifs[0]
        ms_per_step = T_ms / args.steps
        value = total_sets / (ms_per_step / 1e3)
        peak, peak_src = peak_hbm()
        line = {
            "metric": METRIC, "value": value, "unit": "motifs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": acc_dtype, "data": "synthetic",
            "edges_per_sec": arcs / (ms_per_step / 1e3),
            "motifs_per_step": total_sets,
            "step_ms": {"mean": ms_per_step, "median": statistics.median(step_ms), "best": min(step_ms),
                        "all": step_ms},
            "config": {"workload": f"{args.config}: {G.CONFIGS[args.config]['desc']}", "k": k, "n": n,
                       "arcs": arcs, "motif_kind": args.kind,
                       "counts": "edge-level (NEXT-2)" if args.edges else "vertex-level",
                       "parallelism": f"dp{world} (graph replicated, cost-balanced task slices, ncclReduce)"
                       if world > 1 else "single GPU",
                       "l2": "flushed between steps (256 MiB write); count matrix >> L2"},
            "e2e": {"value": total_sets / (E_ms / 1e3), "unit": "motifs/s",
                    "h2d_bytes_per_step": int(2 * 4 * arcs),
                    "d2h_bytes_per_step": int(rows * C * 8), "ms_per_step": E_ms},
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        if enum_ms:
            enum_avg = statistics.mean(enum_ms)
            line["kernel_ms"] = {"enum_avg": enum_avg, "enum_median": statistics.median(enum_ms),
                                 "enum_best": min(enum_ms), "step_avg": ms_per_step,
                                 "enum_share": enum_avg / ms_per_step,
                                 **{f"{key}_avg": statistics.mean(t[key] for t in phase_ms)
                                    for key in ("build", "schedule", "finalize")}}
            line["roofline"] = roofline(args, k, total_sets, enum_avg, peak, peak_src,
                                        float((clk or {}).get("sm_mhz") or (clk or {}).get("sm_max_mhz") or 1965.0))
            if args.edges:
                line["roofline"]["kernel"] = f"k_edges<{k}>"
            elif k == 5:
                line["roofline"]["kernel"] = "k_layers<5>"
        if world == 1 and not args.no_cpu_baseline:
            rate, sets, dt, hi, cores = oracle_sample((n, src, dst), k, args.cpu_seconds)
            line["cpu_baseline"] = {"value": rate, "unit": "motifs/s", "cores": cores, "kind": "oracle",
                                    "cpu": cpu_model(),
                                    "sample": f"ESU, roots with random label < {hi} of {n}: {sets} sets in {dt:.1f} s"}
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def roofline(args, k, motifs, enum_ms, peak, peak_src, sm_mhz):
    """Roofline of the dominant kernel (k_enum), per launch (N = 1); DESIGN.md §4 "Roofline".
    The path is integer and irregular, and its closed forms count most sets without touching
    them, so no per-motif byte count bounds it.  Headline ("alu"): the instruction issue of the
    SMs -- achieved = warp instructions per launch (ncu smsp__inst_executed.sum, committed under
    profiles/) over the live kernel time; peak = 148 SMs x 4 schedulers x 1 warp instruction per
    clock at the measured SM clock (B300_MICROARCH.md / B200_PROFILING.md unit counts).
    Reported beside it: hbm = measured DRAM bytes per launch (ncu) over the live time vs the
    measured HBM copy bandwidth, and the SURVEY §8(d) M3 per-motif model (4 B + 16 B per atomic
    reaching L2, per motif), which the closed forms undercut (frac > 1: not a bound)."""
    t = enum_ms / 1e3
    c = ncu_counters(args.config + ("-edges" if args.edges else ""), k, args.kind)
    peak_issue = 148 * 4 * sm_mhz / 1e3   # G warp-instructions / s
    roof = {"bound": "alu", "kernel": f"k_enum<{k}>", "unit": "Gwarp-inst/s", "peak": peak_issue,
            "peak_source": f"148 SMs x 4 schedulers x 1 warp-instruction/clock x {sm_mhz:.0f} MHz (measured SM clock)",
            "motifs_per_launch": motifs}
    stale = bool(c) and abs(c.get("duration_ms", 0.0) - enum_ms) > 0.08 * enum_ms
    if c and "warp_insts" in c and not stale:
        achieved = c["warp_insts"] / t / 1e9
        atoms = c["l2_red_requests"] + c.get("l2_atom_requests", 0)
        b_eff = 4 + 16 * atoms / motifs
        dram = c["dram_bytes"] / t / 1e9
        roof.update({"achieved": achieved, "frac": achieved / peak_issue, "traffic": c["dram_bytes"],
                     "warp_insts_per_launch": c["warp_insts"],
                     "hbm": {"achieved": dram, "peak": peak, "unit": "GB/s", "frac": dram / peak,
                             "peak_source": peak_src},
                     "m3_model": {"B_k_eff": b_eff, "atomics_per_motif": atoms / motifs,
                                  "achieved": motifs * b_eff / t / 1e9, "frac": motifs * b_eff / t / 1e9 / peak,
                                  "note": "per-motif model of SURVEY 8(d) M3; the closed forms count most "
                                          "sets without a per-set read or atomic, so it does not bound k_enum"},
                     "l2_hit_pct": c.get("l2_hit_pct"), "l2_red_hit_pct": c.get("l2_red_hit_pct"),
                     "warps_active_pct": c.get("warps_active_pct"), "ncu_source": c.get("report"),
                     "ncu_duration_ms": c.get("duration_ms")})
    elif stale:   # counters of another build of the kernel: their instruction count does not describe this one
        roof.update({"achieved": None, "frac": None, "traffic": None,
                     "note": f"committed ncu counters ({c.get('report')}, {c.get('duration_ms'):.1f} ms) are from "
                             f"another build of the kernel (live {enum_ms:.1f} ms): re-capture"})
    else:
        roof.update({"achieved": None, "frac": None, "traffic": None,
                     "note": "no ncu counters committed for this workload (profiles/ncu_traffic.json)"})
    return roof


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""bench.py — Atos hot path on B200 (BASELINE.json metric, configs[2]).

Workload (BASELINE.json configs[2]): RMAT scale 24, edge
factor 16, Graph500 (a,b,c) = (.57,.19,.19), seed 1, directed, unpermuted
(vertex 0 is the hub).  One step = one pass of the whole hot path (§8a):
  BFS from vertex 0 (speculative, persistent CTA workers) and
  PageRank alpha=0.85 eps=1e-6 (asynchronous push, persistent CTA workers),
each including its timed init (a2).  Inputs are resident in HBM before the
timed region; the RMAT-24 CSR (1.2 GB) exceeds L2, and L2 is additionally
flushed (512 MB write) between timed steps, outside the events.

value = whole-job GTEPS_norm = (E_bfs + W_pr) / (t_bfs + t_pr), with
  E_bfs = sum of out-degrees of vertices BFS reached (Graph500 style),
  W_pr  = the edge pushes of our own BSP push PageRank run (Alg. 3) on the same
          graph at the same alpha/eps, measured once untimed (SURVEY 8d
          GTEPS_norm, the tbl:extrawork normalisation P:818): a fixed work
          count, so value is proportional to 1/time.  The actual edge pushes
          are reported as pagerank.gteps_raw.
roofline: the dominant kernel (the persistent PageRank kernel) against
MEASURED_PEAKS.json hbm_gbs with algorithmic bytes 8 B / edge push + 32 B /
pop, plus the same for BFS (8 B / reached edge + 28 B / vertex),
and the sector model (32 B per random 4-B access) beside it.

--impl reference: the CPU oracle (oracle/, plain C) on this host on the same
workload, in the same unit: serial BFS + the all-cores fp64 pull-Jacobi
PageRank time-to-answer (bounded sample; the only other place bench.py runs it).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "GTEPS (BFS, PageRank) and time-to-colour at 1/2/4/8 B200; % of HBM roofline"
ALPHA, EPS = 0.85, 1e-6


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="atos", choices=["atos", "reference"])
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--edge-factor", type=int, default=16)
    ap.add_argument("--fetch", type=int, default=128, help="BFS FETCH_SIZE")
    ap.add_argument("--threads", type=int, default=256, help="BFS cta_threads")
    ap.add_argument("--pr-fetch", type=int, default=128, help="PageRank FETCH_SIZE")
    ap.add_argument("--pr-threads", type=int, default=1024, help="PageRank cta_threads")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-color", action="store_true", help="skip the time-to-colour leg (symmetrised graph)")
    ap.add_argument("--dist-kernel-bfs", default="persistent", choices=["persistent", "discrete"],
                    help="N > 1, BFS: per-round local strategy (persistent = drain to local quiescence)")
    ap.add_argument("--dist-kernel-pr", default="discrete", choices=["persistent", "discrete"],
                    help="N > 1, PageRank: per-round local strategy (discrete = one superstep per exchange; "
                         "draining to local quiescence re-activates every remotely-fed vertex each round: 9x the "
                         "edge pushes on RMAT-20 at N=2)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: host-staged exchange, for 1-GPU smoke tests)")
    return ap.parse_args()


# returning f32 atomicAdd on random addresses of a 64 MB array, all SMs, any in-flight depth 1-16 and
# 16-64 warps/SM (profiles/r02_ubench_sweep.md: 101.7-102.6 skewed, 125.9-127.3 uniform)
ATOM_SKEWED_GOPS = 102.6
ATOM_UNIFORM_GOPS = 127.3
RED_SKEWED_GOPS = 145.9  # red.add.f64, skew 12 (the hub pushes of R35)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.rows.append([x.strip() for x in ln.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], None, set()
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for nm, v in zip(names, r[2:6]):
                    if v.lower() == "active":
                        reasons.add(nm)
            except Exception:
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def atomic_ceiling(e_pr, kms, args):
    """Edge pushes per second against the L2 atomic ceiling for THIS graph's target distribution:
    tools/atomic_trace.py replays RMAT-24's column array through the product's push (R35/R38:
    red.add.f64 into one of four replicas at hubs, returning f32 atomicAdd elsewhere),
    profiles/r02_atomic_ceiling.json.  The random-address ceilings of tools/ubench.cu are beside it."""
    ach = statistics.mean(e / (k * 1e-3) / 1e9 for e, k in zip(e_pr, kms))
    out = {"achieved_gops": ach, "atom_uniform_gops": ATOM_UNIFORM_GOPS, "atom_skewed_gops": ATOM_SKEWED_GOPS,
           "red_f64_skewed_gops": RED_SKEWED_GOPS}
    try:
        with open(os.path.join(ROOT, "profiles", "r02_atomic_ceiling.json")) as f:
            c = json.load(f)[f"rmat{args.scale}_ef{args.edge_factor}_s1"]
        out.update(peak_gops=c["product_gops"], frac=ach / c["product_gops"], source=c["source"])
    except Exception:
        out.update(peak_gops=ATOM_SKEWED_GOPS, frac=ach / ATOM_SKEWED_GOPS,
                   source="profiles/r02_ubench_sweep.md (no graph-trace ceiling for this workload)")
    return out


def ncu_traffic(key):
    """Per-launch DRAM traffic of a kernel from the committed ncu capture (profiles/), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as f:
            return json.load(f)[key]["bytes"]
    except Exception:
        return None


def make_graph(args):
    import graphgen as gg
    t = time.time()
    g = gg.rmat(args.scale, args.edge_factor, seed=1)
    return g, time.time() - t


# ------------------------------------------------------------------ reference
# PageRank work constant: edge pushes of our BSP push run (Alg. 3) on this workload (GTEPS_norm's
# numerator), written by the GPU arm (pr_work_bsp) so the reference arm, which must not run
# the CUDA path, reports in the same unit.  Not an oracle input or expected value: a unit conversion.
WORK_FILE = os.path.join(ROOT, "profiles", "work_constants.json")


def work_key(args):
    return f"rmat{args.scale}_ef{args.edge_factor}_s1_a{ALPHA}_e{EPS}"


def read_work(args):
    try:
        with open(WORK_FILE) as f:
            return int(json.load(f)[work_key(args)])
    except Exception:
        return None


def write_work(args, w):
    try:
        d = {}
        if os.path.exists(WORK_FILE):
            with open(WORK_FILE) as f:
                d = json.load(f)
        if d.get(work_key(args)) != w:
            d[work_key(args)] = w
            with open(WORK_FILE, "w") as f:
                json.dump(d, f, indent=1, sort_keys=True)
    except OSError:
        pass


def jacobi_sweeps_to_answer(tol=1e-10, alpha=ALPHA):
    """Sweeps the oracle's Jacobi needs for ||x_k+1 - x_k||_1 <= tol ||x_k+1||_1: the iteration
    contracts the L1 error by alpha per sweep (P column-substochastic), so ceil(log tol / log alpha)."""
    import math
    return math.ceil(math.log(tol) / math.log(alpha))


def oracle_pagerank_answer(g, threads):
    """Time-to-answer of the oracle's all-cores pull-Jacobi (oracle/oracle.c or_pagerank_jacobi, tol 1e-10)
    on the full graph, from a bounded sample: calls with 2 and 10 sweeps give the per-call setup (in-edge
    transpose) T and the per-sweep time s; answer = T + K s with K = jacobi_sweeps_to_answer()."""
    import oracle
    t = []
    for k in (2, 10):
        t0 = time.perf_counter()
        oracle.pagerank(g, ALPHA, tol=0.0, max_iter=k, threads=threads)
        t.append(time.perf_counter() - t0)
    s = max((t[1] - t[0]) / 8, 1e-9)
    T = max(t[0] - 2 * s, 0.0)
    K = jacobi_sweeps_to_answer()
    return T + K * s, T, s, K


def run_reference(args, rank, world):
    """The oracle (plain C, oracle/) on this host, as it stands: serial FIFO BFS from 0 and the all-cores
    fp64 pull-Jacobi PageRank, on the full workload; value in the GPU arm's unit (GTEPS_norm)."""
    if rank != 0:
        return
    import oracle
    g, _ = make_graph(args)
    cores = os.cpu_count() or 1
    deg = g.degrees()
    w_pr = read_work(args)
    # PageRank time-to-answer: measured once (bounded sample, see oracle_pagerank_answer)
    t_pr, T, s_sweep, K = oracle_pagerank_answer(g, cores)
    times, edges = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        d = oracle.bfs(g, 0)
        t1 = time.perf_counter()
        if i >= args.warmup:
            e_bfs = int(deg[d != oracle.UNREACHED].sum())
            times.append(t1 - t0 + t_pr)
            edges.append(e_bfs + (w_pr if w_pr is not None else K * g.m))
    tot_t, tot_e = sum(times), sum(edges)
    v = tot_e / tot_t / 1e9
    sample = (f"per step: serial FIFO BFS from 0 on the full RMAT-{args.scale} (1 thread, timed every step) + "
              f"the all-cores ({cores} threads) fp64 pull-Jacobi time-to-answer (tol 1e-10) on the full graph, "
              f"measured once: in-edge transpose {T:.2f} s + {K} sweeps x {s_sweep:.3f} s (sweep time from calls "
              f"of 2 and 10 sweeps; {K} = ceil(log 1e-10 / log alpha), the contraction bound); PageRank work = "
              + (f"our BSP push count {w_pr} (GTEPS_norm, profiles/work_constants.json)" if w_pr is not None
                 else f"{K} x m (work constant missing)"))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_t / len(times) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"rmat{args.scale}_ef{args.edge_factor}_bfs0+pagerank", "scale": args.scale,
                   "edge_factor": args.edge_factor, "n": g.n, "m": g.m},
        "cpu_baseline": {"value": v, "unit": "GTEPS", "cores": cores, "kind": "oracle", "sample": sample,
                         "pagerank_time_to_answer_s": t_pr, "bfs_s": statistics.mean(x - t_pr for x in times)},
        "e2e": {"value": v, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def cpu_baseline(g, depth_gpu, w_pr, gs=None, colors_gpu=None):
    """The oracle on this host, same workload and unit as `value`: serial BFS (1 thread) + all-cores
    Jacobi time-to-answer (bounded sample, oracle_pagerank_answer)."""
    import oracle
    deg = g.degrees()
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    d = oracle.bfs(g, 0)
    t_bfs = time.perf_counter() - t0
    t_pr, T, s_sweep, K = oracle_pagerank_answer(g, cores)
    e = int(deg[d != oracle.UNREACHED].sum()) + w_pr
    out = {"value": e / (t_bfs + t_pr) / 1e9, "unit": "GTEPS", "cores": cores, "kind": "oracle",
           "sample": f"serial FIFO BFS from 0 on the full graph, 1 thread ({t_bfs:.2f} s) + fp64 pull-Jacobi "
                     f"PageRank time-to-answer with {cores} threads ({t_pr:.1f} s = transpose {T:.2f} s + {K} "
                     f"sweeps x {s_sweep:.3f} s, sweep time measured from calls of 2 and 10 sweeps; {K} = "
                     f"ceil(log 1e-10 / log alpha)); work counted as in `value` (GTEPS_norm)",
           "bfs_s": t_bfs, "pagerank_time_to_answer_s": t_pr, "pagerank_threads": cores,
           "bfs_matches_gpu": bool(np.array_equal(d, depth_gpu))}
    if gs is not None:
        t3 = time.perf_counter()
        _, k = oracle.greedy_color(gs)
        t4 = time.perf_counter()
        bad, kg = oracle.check_coloring(gs, colors_gpu)
        out["color"] = {"time_to_color_ms": (t4 - t3) * 1e3, "colors": k, "kind": "serial id-order first fit",
                        "gpu_monochromatic_edges": bad, "gpu_colors": kg}
    return out


# ------------------------------------------------------------------ atos
def pr_work_bsp(atos, G):
    """PageRank work for `value` (SURVEY 8d GTEPS_norm, the tbl:extrawork normalisation P:818):
    the edge pushes of our own BSP push run (Alg. 3) at the same alpha/eps on the same graph,
    measured once, untimed.  A fixed work count makes `value` proportional to 1/time:
    raw edge pushes would reward a schedule for doing more pushes."""
    _, st = atos.pagerank(G, ALPHA, EPS, kernel="bsp", worker="cta", fetch_size=128, cta_threads=256,
                          timeout_s=300)
    return int(st["edges_processed"])


def run_atos(args, rank, world, local_rank):
    import torch
    import paper_2112_00132_b200 as atos

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    g, gen_s = make_graph(args)
    stream = torch.cuda.current_stream()
    cfg_bfs = atos.Config(kernel="persistent", worker="cta", fetch_size=args.fetch, cta_threads=args.threads,
                          timeout_s=120)
    cfg_pr = atos.Config(kernel="persistent", worker="cta", fetch_size=args.pr_fetch, cta_threads=args.pr_threads,
                         timeout_s=120)
    G = atos.Graph(g.off, g.col)
    depth = torch.empty(g.n, dtype=torch.int32, device=dev)
    rank_out = torch.empty(g.n, dtype=torch.float32, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    deg = g.degrees()
    w_pr = pr_work_bsp(atos, G)
    if rank == 0:
        write_work(args, w_pr)

    def step():
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(stream)
        _, sb = atos.bfs(G, 0, cfg_bfs, out=depth)
        ev[1].record(stream)
        _, sp = atos.pagerank(G, ALPHA, EPS, cfg_pr, out=rank_out)
        ev[2].record(stream)
        return ev, sb, sp

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    records = []
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)  # L2 flush, outside the events
            torch.cuda.synchronize()
            ev, sb, sp = step()
            torch.cuda.synchronize()
            records.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), sb, sp))
    if world > 1:
        torch.distributed.barrier()
    d_host = depth.cpu().numpy().view(np.uint32)
    e_bfs = int(deg[d_host != atos.UNREACHED].sum())
    v_bfs = int((d_host != atos.UNREACHED).sum())
    # vertices a work-efficient run pops: dangling ones are never pushed (R29), the source always is
    v_exp = int(((d_host != atos.UNREACHED) & (deg > 0)).sum()) + int(deg[0] == 0)
    t_bfs = [r[0] for r in records]
    t_pr = [r[1] for r in records]
    e_pr = [r[3]["edges_processed"] for r in records]
    pops_pr = [r[3]["tasks_popped"] for r in records]
    step_ms = [a + b for a, b in zip(t_bfs, t_pr)]
    # max over ranks of the per-step device time (replicas: identical work per rank)
    tot_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([tot_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tot_ms = float(t.item())
    tot_edges = (e_bfs + w_pr) * len(records) * world
    value = tot_edges / (tot_ms * 1e-3) / 1e9
    hbm, peak_kind = peaks()
    # dominant kernel: PageRank persistent kernel (hot-path kernel_ms from the library's events)
    pr_kms = statistics.mean(r[3]["kernel_ms"] for r in records)
    pr_bytes = statistics.mean(8.0 * e + 32.0 * p for e, p in zip(e_pr, pops_pr))
    pr_ach = pr_bytes / (pr_kms * 1e-3) / 1e9
    pr_sec = statistics.mean(36.0 * e + 104.0 * p for e, p in zip(e_pr, pops_pr))
    bfs_kms = statistics.mean(r[2]["kernel_ms"] for r in records)
    bfs_bytes = 8.0 * e_bfs + 28.0 * v_bfs
    bfs_ach = bfs_bytes / (bfs_kms * 1e-3) / 1e9
    launches = sum(r[2]["kernel_launches"] + r[3]["kernel_launches"] for r in records) // len(records)
    out = {
        "metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms / len(records), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32+f32", "data": "synthetic",
        "config": {"workload": f"rmat{args.scale}_ef{args.edge_factor}_bfs0+pagerank", "scale": args.scale,
                   "edge_factor": args.edge_factor, "n": g.n, "m": g.m, "kernel": "persistent", "worker": "cta",
                   "fetch_size": args.fetch, "pr_fetch_size": args.pr_fetch, "cta_threads": args.threads,
                   "pr_cta_threads": args.pr_threads, "sink_defer": True, "pr_hub_check": cfg_pr.pr_hub_check,
                   "pr_hubs": "in-degree >= 2048, fp64 residues in 4 replicas, sweep-activated (R34/R35/R38)",
                   "alpha": ALPHA, "eps": EPS, "l2": "flushed (512 MB write) between steps; inputs 1.2 GB > L2",
                   "parallelism": "replicas" if world > 1 else "single"},
        "roofline": {"bound": "hbm", "achieved": pr_ach, "peak": hbm, "unit": "GB/s", "frac": pr_ach / hbm,
                     "traffic": ncu_traffic("pagerank_persistent_cta"),
                     "traffic_source": "profiles/r02_traffic.json (ncu --set full, same config)",
                     "algorithmic_bytes": pr_bytes, "kernel": "k_persistent<PrAppT<float, true>, CTA>",
                     "bytes_model": "8 B/edge push + 32 B/pop", "peak_kind": peak_kind,
                     # SURVEY 8d sector model (diagnostic): every random 4-8 B access costs a 32-B sector
                     "sector_model": {"bytes": pr_sec, "achieved": pr_sec / (pr_kms * 1e-3) / 1e9,
                                      "frac": pr_sec / (pr_kms * 1e-3) / 1e9 / hbm,
                                      "bytes_model": "36 B/edge push (col 4 + residue sector 32) + 104 B/pop "
                                                     "(off sector 32 + slot 8 + exch sector 32 + rank sector 32)"}},
        # PageRank's edge push is one L2 atomic on an RMAT-skewed address: a returning fp32 atomicAdd
        # (threshold crossing) or, for hub targets (R35), a fire-and-forget red.add.f64
        "atomic_ceiling": atomic_ceiling(e_pr, [r[3]["kernel_ms"] for r in records], args),
        "bfs": {"gteps": e_bfs / (statistics.mean(t_bfs) * 1e-3) / 1e9, "ms": statistics.mean(t_bfs),
                "kernel_ms": bfs_kms, "edges": e_bfs, "reached": v_bfs,
                "roofline_frac": bfs_ach / hbm, "achieved_gbs": bfs_ach,
                "sector_model_frac": (36.0 * e_bfs + 72.0 * v_bfs) / (bfs_kms * 1e-3) / 1e9 / hbm,
                "overwork": statistics.mean(r[2]["tasks_popped"] for r in records) / max(v_exp, 1),
                "overwork_def": "pops / reached vertices with out-degree > 0 (dangling ones are not pushed, R29)"},
        "value_def": "(BFS reached out-edges + PageRank BSP-equivalent edge pushes) / device time (GTEPS_norm, SURVEY 8d)",
        "pagerank": {"gteps_raw": statistics.mean(e / (t * 1e-3) / 1e9 for e, t in zip(e_pr, t_pr)),
                     "work_bsp_pushes": w_pr,
                     "gteps_norm": statistics.mean(w_pr / (t * 1e-3) / 1e9 for t in t_pr),
                     "ms": statistics.mean(t_pr), "kernel_ms": pr_kms, "edge_pushes": statistics.mean(e_pr),
                     "pops": statistics.mean(pops_pr), "max_residue": max(r[3]["max_residue"] for r in records)},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "graph_gen_s": gen_s,
    }
    if not args.no_e2e:
        out["e2e"] = e2e(args, g, atos, stream, cfg_bfs, cfg_pr, world, w_pr)
    gs = colors = None
    if not args.no_color:
        gs, colors, out["color"] = color_leg(args, atos, dev, flush)
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        out["cpu_baseline"] = cpu_baseline(g, d_host, w_pr, gs, colors)
    if rank == 0:
        print(json.dumps(out), flush=True)


def color_leg(args, atos, dev, flush):
    """Time-to-colour (the metric's third part): speculative greedy colouring
    (Alg. 6, persistent CTA workers) of the symmetrised RMAT graph, device time
    of the library call (init + run) with L2 flushed before each run."""
    import torch
    import graphgen as gg
    t = time.time()
    gs = gg.rmat(args.scale, args.edge_factor, seed=1, symmetrize=True)
    gen_s = time.time() - t
    S = atos.Graph(gs.off, gs.col, symmetric=True)
    cfg = atos.Config(kernel="persistent", worker="cta", fetch_size=128, cta_threads=256, timeout_s=120)
    out = torch.empty(gs.n, dtype=torch.int32, device=dev)
    atos.color(S, cfg, out=out)  # warm-up
    ms, k = [], 0
    for _ in range(3):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        _, k, st = atos.color(S, cfg, out=out)
        ms.append(st["ms"])
    S.close()
    return gs, out.cpu().numpy(), {
        "time_to_color_ms": statistics.median(ms), "ms_all": ms, "colors": k, "overwork": st["tasks_popped"] / (2 * gs.n),
        "graph": f"rmat{args.scale}_ef{args.edge_factor} symmetrised (n={gs.n}, m={gs.m})", "graph_gen_s": gen_s,
        "kernel": "persistent", "worker": "cta", "fetch_size": 128, "cta_threads": 256}


def e2e(args, g, atos, stream, cfg_bfs, cfg_pr, world, w_pr):
    """Same metric through the public API from pinned host buffers: graph upload
    (atos_graph_create H2D), BFS + PageRank, results read back to host."""
    import torch
    off = torch.from_numpy(g.off).pin_memory()
    col = torch.from_numpy(g.col).pin_memory()
    depth = torch.empty(g.n, dtype=torch.int32).pin_memory()
    rk = torch.empty(g.n, dtype=torch.float32).pin_memory()
    deg = g.degrees()
    times, edges = [], []
    for i in range(2 + max(3, args.steps)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        G = atos.Graph(off.numpy(), col.numpy())
        _, sb = atos.bfs(G, 0, cfg_bfs, out=depth.numpy().view(np.uint32))
        _, sp = atos.pagerank(G, ALPHA, EPS, cfg_pr, out=rk.numpy())
        t1 = time.perf_counter()
        G.close()
        if i >= 2:
            d = depth.numpy().view(np.uint32)
            edges.append(int(deg[d != atos.UNREACHED].sum()) + w_pr)
            times.append(t1 - t0)
    h2d = g.off.nbytes + g.col.nbytes
    d2h = g.n * 8
    return {"value": sum(edges) * world / sum(times) / 1e9, "unit": "GTEPS", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": statistics.mean(times) * 1e3}


def run_atos_multi(args, rank, world, local_rank):
    """N > 1: the 1-D partitioned path.  RMAT-24 relabelled by a
    seeded permutation (a block split is 3.4x edge-imbalanced otherwise), each
    rank owns n/N vertices; rounds exchange remote activations with NCCL
    all-to-all.  Strong scaling (total work fixed).  Device time per step =
    CUDA events on the compute stream around BFS + PageRank (all rounds, NCCL
    included), max over ranks."""
    import torch
    import torch.distributed as dist
    import graphgen as gg
    import paper_2112_00132_b200 as atos
    from paper_2112_00132_b200 import dist as adist

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    g0, gen_s = make_graph(args)
    g, fwd = gg.permute(g0, 12345)
    src = int(fwd[0])
    del g0
    Gw = atos.Graph(g.off, g.col)
    w_pr = pr_work_bsp(atos, Gw)  # fixed PageRank work of this (permuted) graph, as at N = 1
    Gw.close()
    del Gw
    comm = adist.Comm.auto()  # NCCL over NVLink/NVSwitch (host callbacks for a gloo group)
    pg = adist.PartGraph.from_global(g, comm)
    cfg = atos.Config(kernel=args.dist_kernel_bfs, worker="cta", fetch_size=args.fetch, cta_threads=args.threads,
                      timeout_s=300)
    cfg_pr = atos.Config(kernel=args.dist_kernel_pr, worker="cta", fetch_size=args.fetch, cta_threads=args.threads,
                         timeout_s=300)
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    deg = g.degrees()
    vb, ve = pg.v_begin, pg.v_end

    def step():
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        d, sb = adist.bfs(pg, src, cfg)
        e[1].record(stream)
        r, sp = adist.pagerank(pg, ALPHA, EPS, cfg_pr)
        e[2].record(stream)
        return e, d, sb, sp

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    recs = []
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            dist.barrier()
            e, d, sb, sp = step()
            torch.cuda.synchronize()
            recs.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), d, sb, sp))
    dist.barrier()
    t = torch.tensor([sum(r[0] + r[1] for r in recs), sum(r[0] for r in recs), sum(r[1] for r in recs)], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    d_local = recs[-1][2]
    e_bfs_local = int(deg[vb:ve][d_local != atos.UNREACHED].sum())
    loc = torch.tensor([e_bfs_local, sum(r[4]["edges_processed"] for r in recs), recs[-1][3]["rounds"],
                        recs[-1][4]["rounds"], sum(r[3]["bytes_sent"] + r[4]["bytes_sent"] for r in recs)],
                       dtype=torch.float64, device=dev)
    dist.all_reduce(loc)
    # this rank's kernel launches per step (the library counts every launch it makes)
    launches = sum(r[3]["kernel_launches"] + r[4]["kernel_launches"] for r in recs) // len(recs)
    e_bfs, e_pr = int(loc[0].item()), float(loc[1].item())
    tot_ms = float(t[0].item())
    value = (e_bfs + w_pr) * len(recs) / (tot_ms * 1e-3) / 1e9
    hbm, peak_kind = peaks()
    out = {
        "metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms / len(recs), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32+f32", "data": "synthetic",
        "config": {"workload": f"rmat{args.scale}_ef{args.edge_factor}_bfs0+pagerank", "scale": args.scale,
                   "edge_factor": args.edge_factor, "n": g.n, "m": g.m,
                   "kernel": {"bfs": args.dist_kernel_bfs, "pagerank": args.dist_kernel_pr},
                   "worker": "cta", "fetch_size": args.fetch, "cta_threads": args.threads, "alpha": ALPHA,
                   "eps": EPS, "backend": args.backend,
                   "parallelism": f"1d-partition x{world} (permuted ids, all-to-all per round)",
                   "l2": "flushed (512 MB write) between steps; inputs > L2"},
        "bfs": {"gteps": e_bfs / (float(t[1].item()) / len(recs) * 1e-3) / 1e9, "ms": float(t[1].item()) / len(recs),
                "rounds": int(loc[2].item()) // world},
        "value_def": "(BFS reached out-edges + PageRank BSP-equivalent edge pushes) / device time (GTEPS_norm, SURVEY 8d)",
        "pagerank": {"ms": float(t[2].item()) / len(recs), "edge_pushes": e_pr / len(recs), "work_bsp_pushes": w_pr,
                     "rounds": int(loc[3].item()) // world},
        "bytes_exchanged_per_step": float(loc[4].item()) / len(recs),
        "roofline": {"bound": "hbm", "achieved": (8.0 * e_pr / len(recs)) / (float(t[2].item()) / len(recs) * 1e-3) / 1e9 / world,
                     "peak": hbm, "unit": "GB/s", "frac": None, "traffic": None, "peak_kind": peak_kind,
                     "note": "per-GPU average of the PageRank edge-push bytes over the whole multi-round step"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    out["roofline"]["frac"] = out["roofline"]["achieved"] / hbm
    if not args.no_color:
        out["color"] = color_leg_multi(args, rank, world, dev, flush)
    if rank == 0:
        print(json.dumps(out), flush=True)


def color_leg_multi(args, rank, world, dev, flush):
    """Time-to-colour on N GPUs: partitioned speculative colouring of
    the symmetrised, permuted RMAT graph; device time = CUDA events around the
    whole multi-round call (exchanges included), max over ranks."""
    import torch
    import torch.distributed as dist
    import graphgen as gg
    from paper_2112_00132_b200 import dist as adist
    gs, _ = gg.permute(gg.rmat(args.scale, args.edge_factor, seed=1, symmetrize=True), 12345)
    pg = adist.PartGraph.from_global(gs, adist.Comm.auto())
    stream = torch.cuda.current_stream()
    ms, k, st = [], 0, {}
    for i in range(4):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        c, st = adist.color(pg, timeout_s=300)
        e1.record(stream)
        torch.cuda.synchronize()
        if i:
            ms.append(e0.elapsed_time(e1))
    t = torch.tensor(ms, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    pg.close()
    return {"time_to_color_ms": float(t.median().item()), "colors": st["num_colors"], "rounds": st["rounds"],
            "graph": f"rmat{args.scale}_ef{args.edge_factor} symmetrised + permuted (n={gs.n}, m={gs.m})",
            "parallelism": f"1d-partition x{world}", "kernel": "persistent", "worker": "cta"}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        local_rank = local_rank % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(local_rank)
        if args.backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            torch.distributed.init_process_group("gloo")
        run_atos_multi(args, rank, world, local_rank)
    else:
        run_atos(args, rank, world, local_rank)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()

"""C5 (BASELINE configs[4]) on ONE B200: RMAT-27 (134M vertices, ~2.1B arcs), seeded vertex
permutation, BFS from permuted(0) and PageRank (alpha=0.85, eps=1e-6) through the
C ABI.  BFS is checked bit-exact against the serial oracle; PageRank variants against the
deterministic multithreaded pull-Jacobi (time-boxed).  The oracle is test infrastructure.
Prints one JSON line.  Not part of the product path."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import graphgen as gg
import paper_2112_00132_b200 as atos

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=27)
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--no-oracle", action="store_true")
ap.add_argument("--permute", type=int, default=1, help="seeded vertex permutation (SURVEY 8d C5); 0 = off")
ap.add_argument("--jacobi-threads", type=int, default=0, help="oracle pull-Jacobi threads (0 = all host cores)")
ap.add_argument("--jacobi-max-s", type=float, default=900.0, help="skip PR parity if the solve would take longer")
ap.add_argument("--pr-variants", default='{"default": {}}', help="JSON {name: Config kwargs}")
a = ap.parse_args()
t = time.time()
g = gg.rmat(a.scale, 16, seed=1)
src = 0
if a.permute:
    g, fwd = gg.permute(g, a.permute)
    src = int(fwd[0])  # BFS from permuted(0): the hub keeps its role
gen_s = time.time() - t
print(f"generated n={g.n} m={g.m} in {gen_s:.1f}s", flush=True)
G = atos.Graph(g.off, g.col)
dev = torch.device("cuda", 0)
depth = torch.empty(g.n, dtype=torch.int32, device=dev)
rank_out = torch.empty(g.n, dtype=torch.float32, device=dev)
cfg_bfs = atos.Config(fetch_size=128, cta_threads=256, timeout_s=300)
flush = torch.empty(512 << 18, dtype=torch.float32, device=dev)
bfs_ms = []
for i in range(a.runs + 1):
    flush.fill_(1.0); torch.cuda.synchronize()
    _, st = atos.bfs(G, src, cfg_bfs, out=depth)
    if i: bfs_ms.append(st["ms"])
d = depth.cpu().numpy().view(np.uint32)
deg = g.degrees()
reached = d != atos.UNREACHED
e_bfs = int(deg[reached].sum())
v_exp = int((reached & (deg > 0)).sum()) + int(deg[src] == 0)
out = {"workload": f"rmat{a.scale}_ef16 single GPU (C5 at N=1)", "n": g.n, "m": g.m, "gen_s": round(gen_s, 1),
       "permute_seed": a.permute, "src": src, "host_cores": os.cpu_count(),
       "bfs": {"ms_median": float(np.median(bfs_ms)), "ms_all": bfs_ms, "edges": e_bfs, "reached": int(reached.sum()),
               "gteps": e_bfs / (np.median(bfs_ms) * 1e-3) / 1e9, "pops": st["tasks_popped"],
               "overwork": st["tasks_popped"] / max(1, v_exp)}, "pagerank": {}}
ranks = {}
for name, kw in json.loads(a.pr_variants).items():
    cfg_pr = atos.Config(fetch_size=128, cta_threads=1024, timeout_s=600, **kw)
    flush.fill_(1.0); torch.cuda.synchronize()
    _, sp = atos.pagerank(G, 0.85, 1e-6, cfg_pr, out=rank_out)
    ranks[name] = rank_out.cpu().numpy().astype(np.float64)
    out["pagerank"][name] = {"config": kw, "ms": sp["ms"], "edge_pushes": sp["edges_processed"],
                             "gteps_raw": sp["edges_processed"] / (sp["ms"] * 1e-3) / 1e9,
                             "max_residue": sp["max_residue"], "pops": sp["tasks_popped"]}
    print(name, out["pagerank"][name], flush=True)
if not a.no_oracle:
    import oracle
    t = time.time()
    ref = oracle.bfs(g, src)
    out["bfs"]["oracle_s"] = round(time.time() - t, 1)
    out["bfs"]["bit_exact_vs_oracle"] = bool(np.array_equal(ref, d))
    # PageRank parity vs the deterministic multithreaded pull-Jacobi, time-boxed:
    # 1 and 3 sweeps are timed first (the difference excludes the serial transpose) and the
    # full solve (~130 sweeps) runs only if it fits the budget.
    t = time.time()
    oracle.pagerank(g, 0.85, tol=1e-300, max_iter=1, threads=a.jacobi_threads)
    t1 = time.time() - t
    t = time.time()
    oracle.pagerank(g, 0.85, tol=1e-300, max_iter=3, threads=a.jacobi_threads)
    sweep_s = max(0.0, (time.time() - t - t1) / 2)
    out["jacobi"] = {"setup_s": round(t1 - sweep_s, 1), "sweep_s": round(sweep_s, 2)}
    if t1 + sweep_s * 150 <= a.jacobi_max_s:
        t = time.time()
        x, it = oracle.pagerank(g, 0.85, threads=a.jacobi_threads)
        out["jacobi"].update(s=round(time.time() - t, 1), iters=int(it), x_max=float(x.max()))
        indeg = np.bincount(g.col, minlength=g.n)
        for name, rk in ranks.items():
            err = np.abs(rk - x)
            i = int(np.argmax(err))
            out["pagerank"][name].update({
                "linf_rel": float(err[i] / x.max()), "within_1e-4": bool(err[i] / x.max() <= 1e-4),
                "worst": {"v": i, "x": float(x[i]), "rank": float(rk[i]), "outdeg": int(deg[i]),
                          "indeg": int(indeg[i])},
                "n_over_1e-4": int(np.sum(err > 1e-4 * x.max()))})
print(json.dumps(out), flush=True)

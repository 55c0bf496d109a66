"""Round experiments (configs of BASELINE.json beyond the bench line), markdown to stdout.

  heatmap   BFS worker size x FETCH_SIZE sweep on the 4899x4899 grid (configs[3]; the
            paper's fig:heatmap analog) and on RMAT-20
  kernels   persistent vs discrete vs BSP on RMAT-24 for BFS and PageRank (configs[2])
  color     greedy colouring on RMAT-16 (configs[1]): time-to-colour, colours vs the
            oracle, overwork; permuted vs unpermuted ids; all kernels/workers
  grid      BFS on the 24M-vertex grid and the road-like variant: ms, per-hop latency
  timeline  cumulative work vs time for BFS/PR on RMAT-24, colouring on RMAT-22
  colorq    colour count vs concurrency (workers in flight), RMAT-20, plain and permuted ids
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_2112_00132_b200 as atos  # noqa: E402


def timed(fn, reps=3):
    out = [fn() for _ in range(reps)]
    return out[-1], statistics.median(o[-1]["ms"] for o in out)


def heatmap():
    sizes = [(8, "thread", 256), (32, "warp", 256), (64, "cta", 64), (128, "cta", 128), (256, "cta", 256),
             (512, "cta", 512), (1024, "cta", 1024)]
    fetches = [1, 4, 16, 64, 256, 1024]
    for gname, g in [("grid 4899x4899 (24.0M vertices, 96.0M arcs, ecc. 9,796)", gg.grid(4899, 4899)),
                     ("RMAT-20 (1.05M vertices, 16.1M arcs)", gg.rmat(20, 16, seed=1))]:
        G = atos.Graph.from_csr(g)
        print(f"\n### BFS from 0 on {gname}: ms (overwork = pops / reached)\n")
        print("| worker (threads) | " + " | ".join(f"F={f}" for f in fetches) + " |")
        print("|---|" + "---|" * len(fetches))
        for _, w, t in sizes:
            row = []
            for f in fetches:
                try:
                    (d, st), ms = timed(lambda: atos.bfs(G, 0, worker=w, cta_threads=t, fetch_size=f, timeout_s=120), 2)
                    reached = int(np.sum(d != atos.UNREACHED))
                    row.append(f"{ms:.2f} ({st['tasks_popped'] / reached:.2f})")
                except atos.AtosError as e:
                    row.append(e.name)
            label = f"{w} ({t})"
            print(f"| {label} | " + " | ".join(row) + " |", flush=True)
        del G


def kernels():
    """Persistent vs discrete vs BSP for the three apps (configs[2]; the paper's strategy comparison,
    P:1025-1027) in the bench configuration, with the work of each schedule relative to BSP's (the
    tbl:extrawork overwork lens): BFS pops / BSP pops, PageRank edge pushes / BSP edge
    pushes, colouring tasks / 2n."""
    g = gg.rmat(24, 16, seed=1)
    G = atos.Graph.from_csr(g)
    deg = g.degrees()
    print("\n### RMAT-24: persistent vs discrete vs BSP (CTA workers, bench configuration)\n")
    print("| app | kernel | ms | launches | rounds | pops | edges | work / BSP | GTEPS |")
    print("|---|---|---|---|---|---|---|---|---|")
    rows = []
    for kern, dl in [("persistent", False), ("discrete", False), ("discrete", True), ("bsp", False)]:
        (d, st), ms = timed(lambda: atos.bfs(G, 0, kernel=kern, device_loop=dl, fetch_size=128, cta_threads=256,
                                             timeout_s=300), 3)
        rows.append(("BFS", kern + (" (device loop)" if dl else ""), ms, st, int(deg[d != atos.UNREACHED].sum())))
    bsp_pops = rows[-1][3]["tasks_popped"]
    for app, name, ms, st, e in rows:
        print(f"| {app} | {name} | {ms:.2f} | {st['kernel_launches']} | {st['rounds']} | {st['tasks_popped']} | "
              f"{st['edges_processed']} | {st['tasks_popped'] / bsp_pops:.3f} (pops) | {e / ms / 1e6:.1f} |", flush=True)
    rows = []
    for kern, dl in [("persistent", False), ("discrete", False), ("discrete", True), ("bsp", False)]:
        (r, st), ms = timed(lambda: atos.pagerank(G, 0.85, 1e-6, kernel=kern, device_loop=dl, fetch_size=128,
                                                  cta_threads=1024 if kern == "persistent" else 256,
                                                  timeout_s=300), 2)
        rows.append(("PageRank", kern + (" (device loop)" if dl else ""), ms, st))
    (r, st), ms = timed(lambda: atos.pagerank(G, 0.85, 1e-6, pr_activation=1, check_size=8, fetch_size=128,
                                              cta_threads=512, timeout_s=300), 1)
    rows.append(("PageRank (Check_Size=8 window, f1)", "persistent", ms, st))
    bsp_e = rows[3][3]["edges_processed"]
    for app, name, ms, st in rows:
        print(f"| {app} | {name} | {ms:.1f} | {st['kernel_launches']} | {st['rounds']} | {st['tasks_popped']} | "
              f"{st['edges_processed']} | {st['edges_processed'] / bsp_e:.3f} (edge pushes) | "
              f"{bsp_e / ms / 1e6:.1f} (norm) |", flush=True)
    s = gg.rmat(22, 16, seed=1, symmetrize=True)
    S = atos.Graph.from_csr(s, symmetric=True)
    for kern, w, f in [("persistent", "cta", 128), ("persistent", "warp", 128), ("discrete", "warp", 32),
                       ("discrete", "cta", 32), ("bsp", "warp", 32), ("bsp", "cta", 32)]:
        (c, k, st), ms = timed3(lambda: atos.color(S, kernel=kern, worker=w, fetch_size=f, cta_threads=256,
                                                   timeout_s=300), 2)
        print(f"| colouring RMAT-22 sym ({k} colours) | {kern} {w} F={f} | {ms:.1f} | {st['kernel_launches']} | "
              f"{st['rounds']} | {st['tasks_popped']} | {st['edges_processed']} | "
              f"{st['tasks_popped'] / (2 * s.n):.3f} (tasks / 2n) | - |", flush=True)


def timed3(fn, reps=3):
    out = [fn() for _ in range(reps)]
    return out[-1], statistics.median(o[-1]["ms"] for o in out)


def color():
    import oracle
    print("\n### Colouring: time-to-colour, colours (GPU vs serial first-fit oracle), overwork = tasks / 2n\n")
    print("| graph | kernel | worker | ms | colours | oracle colours | overwork |")
    print("|---|---|---|---|---|---|---|")
    for gname, g in [("RMAT-16 sym", gg.rmat(16, 16, seed=1, symmetrize=True)),
                     ("RMAT-16 sym, permuted ids", gg.rmat(16, 16, seed=1, symmetrize=True, perm_seed=7)),
                     ("RMAT-22 sym", gg.rmat(22, 16, seed=1, symmetrize=True)),
                     ("RMAT-22 sym, permuted ids", gg.rmat(22, 16, seed=1, symmetrize=True, perm_seed=7)),
                     ("grid 1024x1024", gg.grid(1024, 1024))]:
        G = atos.Graph.from_csr(g, symmetric=True)
        _, k_or = oracle.greedy_color(g)
        for kern, w in [("persistent", "warp"), ("persistent", "cta"), ("discrete", "warp"), ("discrete", "cta"),
                        ("bsp", "cta")]:
            (c, k, st), ms = timed(lambda: atos.color(G, kernel=kern, worker=w, fetch_size=32 if w == "warp" else 256,
                                                      timeout_s=300), 3)
            bad, _ = oracle.check_coloring(g, c)
            assert bad == 0
            print(f"| {gname} | {kern} | {w} | {ms:.2f} | {k} | {k_or} | {st['tasks_popped'] / (2 * g.n):.2f} |",
                  flush=True)


def grid():
    print("\n### High-diameter BFS (configs[3])\n")
    print("| graph | worker | F | ms | per-hop us | pops/reached |")
    print("|---|---|---|---|---|---|")
    center = 2449 * 4899 + 2449
    for gname, g, src in [("grid 4899x4899, src corner", gg.grid(4899, 4899), 0),
                          ("road-like 4899x4899 (40% edges dropped), src centre", gg.grid(4899, 4899, drop_prob=0.4, seed=3),
                           center)]:
        G = atos.Graph.from_csr(g)
        for w, t, f, k in [("cta", 256, 128, "persistent"), ("cta", 64, 16, "persistent"), ("warp", 256, 4, "persistent"),
                           ("thread", 256, 256, "persistent"), ("cta", 256, 128, "discrete"),
                           ("cta", 256, 128, "discrete+device-loop"), ("cta", 256, 128, "bsp")]:
            kern = k.split("+")[0]
            (d, st), ms = timed(lambda: atos.bfs(G, src, worker=w, cta_threads=t, fetch_size=f, kernel=kern,
                                                 device_loop="device-loop" in k, timeout_s=300), 2)
            label = f"{w} {k}"
            reached = d != atos.UNREACHED
            e = int(d[reached].max())
            print(f"| {gname} | {label} ({t}) | {f} | {ms:.1f} | {ms * 1e3 / e:.2f} (ecc {e}, reached "
                  f"{int(reached.sum())}) | {st['tasks_popped'] / reached.sum():.3f} |", flush=True)


def colorq():
    """Colour count vs concurrency (855 colours vs the oracle's 464 on RMAT-24):
    speculative colouring picks the smallest colour free among the neighbours' colours as they are
    at that moment; with thousands of tasks in flight a vertex often sees neighbours still uncoloured
    or about to change, and conflicts re-colour the larger id with a larger colour.  Fewer concurrent
    workers should approach the serial id-order greedy count."""
    import oracle
    for perm in (0, 7):
        s = gg.rmat(20, 16, seed=1, symmetrize=True, perm_seed=perm)
        S = atos.Graph.from_csr(s, symmetric=True)
        _, k_or = oracle.greedy_color(s)
        print(f"\n### Colours vs concurrency, RMAT-20 symmetrised{' (permuted ids)' if perm else ''}: "
              f"oracle id-order greedy = {k_or}\n")
        print("| worker | CTAs (num_blocks) | threads | F | tasks in flight (max) | ms | colours | colours / oracle | tasks / 2n |")
        print("|---|---|---|---|---|---|---|---|---|")
        for w, blocks, t, f in [("thread", 1, 32, 1), ("warp", 1, 32, 1), ("cta", 1, 128, 32), ("cta", 8, 128, 32),
                                ("cta", 32, 128, 32), ("cta", 148, 256, 32), ("cta", 0, 256, 32),
                                ("cta", 0, 256, 128)]:
            (c, k, st), ms = timed3(lambda: atos.color(S, worker=w, num_blocks=blocks, cta_threads=t, fetch_size=f,
                                                      timeout_s=300), 2)
            flight = "all resident" if blocks == 0 else str(blocks * (f if w == "cta" else (t // 32) * f * (32 if w == "thread" else 1)))
            print(f"| {w} | {blocks or 'max'} | {t} | {f} | {flight} | {ms:.1f} | {k} | {k / k_or:.2f} | "
                  f"{st['tasks_popped'] / (2 * s.n):.2f} |", flush=True)


def timeline():
    """Cumulative work vs time (the paper's throughput-over-time figures) for the three apps
    in the bench configuration; colouring on the symmetrised RMAT-22."""
    g = gg.rmat(24, 16, seed=1)
    G = atos.Graph.from_csr(g)
    s = gg.rmat(22, 16, seed=1, symmetrize=True)
    S = atos.Graph.from_csr(s, symmetric=True)
    tr = atos.Trace(1 << 23)
    for app in ["bfs", "pr", "color"]:
        if app == "bfs":
            atos.bfs(G, 0, fetch_size=128)
            _, st = atos.bfs(G, 0, fetch_size=128, trace=tr)
        elif app == "pr":
            _, st = atos.pagerank(G, 0.85, 1e-6, fetch_size=128, cta_threads=1024, trace=tr)
        else:
            atos.color(S, fetch_size=128)
            _, _, st = atos.color(S, fetch_size=128, trace=tr)
        r = tr.records(st)
        t = (r["t_ns"] - r["t_ns"][0]) / 1e3
        nb = 20
        edges = np.linspace(0, t[-1] + 1e-9, nb + 1)
        idx = np.clip(np.searchsorted(edges, t, side="right") - 1, 0, nb - 1)
        tot = r["edges"].astype(np.int64).sum()
        gname = "RMAT-22 symmetrised" if app == "color" else "RMAT-24"
        print(f"\n### Timeline: {app.upper()} {gname} ({st['ms']:.2f} ms, {len(r)} batches)\n")
        print("| t (us) | batches | items | edges | cum. edges % | SMs active |")
        print("|---|---|---|---|---|---|")
        cum = 0
        for b in range(nb):
            m = idx == b
            eb = int(r["edges"][m].astype(np.int64).sum())
            cum += eb
            print(f"| {edges[b]:.0f} | {int(m.sum())} | {int(r['items'][m].sum())} | {eb} | {100 * cum / tot:.1f} | "
                  f"{len(np.unique(r['sm'][m]))} |")


if __name__ == "__main__":
    for name in sys.argv[1:]:
        t0 = time.time()
        globals()[name]()
        print(f"\n_({name}: {time.time() - t0:.0f} s)_", flush=True)

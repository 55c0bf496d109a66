import numpy as np, graphgen as gg, oracle, paper_2112_00132_b200 as atos
g = gg.rmat(16, 16, seed=1)
x, _ = oracle.pagerank(g, 0.85)
G = atos.Graph.from_csr(g)
for rep in range(3):
  for k in ["persistent", "discrete"]:
    for f in [1, 32, 256]:
        for w in ["thread", "warp", "cta"]:
            r, st = atos.pagerank(G, 0.85, 1e-6, kernel=k, worker=w, fetch_size=f)
            err = np.max(np.abs(r - x)) / x.max()
            bad = np.argmax(np.abs(r - x))
            print(rep, k, w, f, f"err={err:.2e} maxres={st['max_residue']:.2e} pops={st['tasks_popped']} pushes={st['tasks_pushed']} edges={st['edges_processed']} hw={st['queue_high_water']} ms={st['ms']:.2f} bad={bad} r={r[bad]:.5f} x={x[bad]:.5f}", flush=True)

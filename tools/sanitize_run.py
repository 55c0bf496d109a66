"""Small runs of every app x worker x kernel strategy, for the bounds-checked
library build (-DATOS_CHECKED, loaded through ATOS_LIB; tests/test_queue_stress.py)
or a memory checker.  Results are checked with plain invariants
(BFS grid depth = i + j, valid colouring, PageRank residues <= eps) so this
script needs no oracle.  usage: python tools/sanitize_run.py [tool]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen as gg  # noqa: E402
import paper_2112_00132_b200 as atos  # noqa: E402


def main():
    tool = sys.argv[1] if len(sys.argv) > 1 else "memcheck"
    grid = gg.grid(16, 16)
    rm = gg.rmat(9, 8, seed=1)
    rms = gg.rmat(9, 8, seed=1, symmetrize=True)
    hub = gg.hub_graph(5000, extra=40)
    G, R, S, H = (atos.Graph.from_csr(grid), atos.Graph.from_csr(rm), atos.Graph.from_csr(rms, symmetric=True),
                  atos.Graph.from_csr(hub))
    i, j = np.divmod(np.arange(256), 16)
    kernels = ["persistent", "discrete", "bsp"]
    # racecheck serialises shared-memory accesses and is slow: fewer combinations
    fetches = [32] if tool == "racecheck" else [1, 32]
    for kernel in kernels:
        for worker in ["thread", "warp", "cta"]:
            # racecheck does not model flag / mbarrier producer-consumer handoffs (tools/rc_probe.cu: a
            # textbook mbarrier pipeline is reported as tens of thousands of hazards), so the
            # warp-specialised persistent CTA kernel (BFS, PageRank) is left to memcheck / synccheck
            ws = kernel == "persistent" and worker == "cta"
            for f in fetches:
                kw = dict(kernel=kernel, worker=worker, fetch_size=f, cta_threads=128, timeout_s=600, num_blocks=4)
                if not (ws and tool == "racecheck"):
                    d, _ = atos.bfs(G, 0, **kw)
                    assert np.array_equal(d, (i + j).astype(np.uint32)), (kernel, worker, f)
                    atos.bfs(H, 0, **kw)
                    r, st = atos.pagerank(R, 0.85, 1e-5, **kw)
                    assert st["max_residue"] <= 1e-5
                c, k, _ = atos.color(S, **kw)
                e = np.repeat(np.arange(rms.n), np.diff(rms.off))
                assert not np.any((c[e] == c[rms.col]) & (e != rms.col)), (kernel, worker, f)
    # warp-specialised persistent CTA worker at its bench shape (queue agent + LBS warps, hub chunks)
    for th, f in ([] if tool == "racecheck" else [(256, 128), (1024, 128)]):
        atos.bfs(H, 0, fetch_size=f, cta_threads=th, timeout_s=600)
        atos.pagerank(R, 0.85, 1e-5, fetch_size=f, cta_threads=th, timeout_s=600)
        atos.bfs(R, 0, fetch_size=f, cta_threads=th, queue_capacity=256, timeout_s=600)
    print("sanitize_run ok", tool, flush=True)


if __name__ == "__main__":
    main()

"""Run tools/atomic_trace.cu on RMAT-<scale>'s column array (the targets of one
full sweep of edge pushes), tagged like the library tags it (HUB_TAG bit 31 for
in-degree >= HUB, R34; --hub, default the library's 2048): the L2 atomic ceiling for this graph's own target
distribution.  usage: python tools/atomic_trace.py [--scale 24]"""
import argparse
import os
import subprocess
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import graphgen as gg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--hub", type=int, default=2048)
a = ap.parse_args()
g = gg.rmat(a.scale, 16, seed=1)
indeg = np.bincount(g.col, minlength=g.n)
col = g.col.astype(np.uint32)
col[indeg[g.col] >= a.hub] |= np.uint32(0x80000000)
d = tempfile.mkdtemp()
path = os.path.join(d, "cols.bin")
col.tofile(path)
exe = os.path.join(d, "atomic_trace")
here = os.path.dirname(os.path.abspath(__file__))
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe,
                       os.path.join(here, "atomic_trace.cu")])
print(f"RMAT-{a.scale}: n={g.n} m={g.m}, hub targets: "
      f"{100 * float(np.mean(indeg[g.col] >= a.hub)):.1f}% of edges (threshold {a.hub})\n", flush=True)
subprocess.check_call([exe, path, str(g.n)])

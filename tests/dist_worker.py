"""Worker for multi-process partitioned tests (spawned by tests; one process per rank).

Runs the CUDA partitioned BFS / PageRank (mode "gpu") or the orchestration with
a numpy stand-in for the device library (mode "fake", CPU-only), over gloo on
127.0.0.1, and writes this rank's result slice to <outdir>/rank<r>.npz."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


class FakeLib:
    """CPU stand-in for the atos_part_* entry points (BFS and colouring), used to
    test the Python orchestration (message grouping, all-to-all splits,
    termination) and the cross-rank colouring protocol without a GPU.  Test
    infrastructure — not the product path."""

    def __init__(self):
        self.g = {}

    def _get(self, h):
        return self.g[h.value if hasattr(h, "value") else h]

    def atos_graph_create_partitioned(self, N, world, rank, bounds_p, off_p, col_p, m, flags, out):
        import ctypes
        b = np.ctypeslib.as_array(ctypes.cast(bounds_p, ctypes.POINTER(ctypes.c_int64)), (world + 1,)).copy()
        n = int(b[rank + 1] - b[rank])
        off = np.ctypeslib.as_array(ctypes.cast(off_p, ctypes.POINTER(ctypes.c_int64)), (n + 1,)).copy()
        col = (np.ctypeslib.as_array(ctypes.cast(col_p, ctypes.POINTER(ctypes.c_int32)), (m,)).copy()
               if m else np.zeros(0, np.int32))
        key = len(self.g) + 1
        self.g[key] = dict(N=N, world=world, rank=rank, b=b, off=off, col=col, n=n)
        out._obj.value = key
        return 0

    def atos_part_begin(self, h, app, src, alpha, eps, cfg):
        s = self._get(h)
        s["app"] = app
        vb = s["b"][s["rank"]]
        if app == 2:  # colouring: replica of all colours, every vertex's ASSIGN queued
            s["color"] = np.full(s["N"], -1, np.int64)
            s["pend"] = np.ones(s["n"], bool)
            s["chg"] = np.zeros(s["n"], bool)
            s["q"] = [(v, 0) for v in range(s["n"])]
            return 0
        s["dist"] = np.full(s["n"], 0xFFFFFFFF, np.uint64)
        s["sent"] = np.full(s["N"], 0xFFFFFFFF, np.uint64)
        s["q"] = []
        if vb <= src < s["b"][s["rank"] + 1]:
            s["dist"][src - vb] = 0
            s["q"].append(src - vb)
        return 0

    def _gc_run(self, s, out):
        vb, ve, b, col, off, color = int(s["b"][s["rank"]]), int(s["b"][s["rank"] + 1]), s["b"], s["col"], s["off"], s["color"]
        while s["q"]:
            v, kind = s["q"].pop(0)
            vg = vb + v
            adj = [int(u) for u in col[off[v]:off[v + 1]] if int(u) != vg]
            if kind == 0:  # ASSIGN: first fit against the replica
                s["pend"][v] = False
                used = {int(color[u]) for u in adj}
                c = 0
                while c in used:
                    c += 1
                color[vg] = c
                s["chg"][v] = True
                s["q"].append((v, 1))
            else:  # CHECK: the larger endpoint of a conflict recolours; a remote one is its owner's
                self_c = False
                for u in adj:
                    if color[u] == color[vg]:
                        if u < vg:
                            self_c = True
                        elif vb <= u < ve and not s["pend"][u - vb]:
                            s["pend"][u - vb] = True
                            s["q"].append((u - vb, 0))
                if self_c and not s["pend"][v]:
                    s["pend"][v] = True
                    s["q"].append((v, 0))
        for v in np.nonzero(s["chg"])[0]:
            s["chg"][v] = False
            owners = {int(np.searchsorted(b, int(u), side="right") - 1) for u in col[off[v]:off[v + 1]]}
            for r in sorted(owners - {s["rank"]}):
                out[r].append(((vb + int(v)) << 32) | int(color[vb + v]))

    def atos_part_run(self, h, flush_all, counts_p):
        import ctypes
        s = self._get(h)
        vb, ve, b = s["b"][s["rank"]], s["b"][s["rank"] + 1], s["b"]
        out = [[] for _ in range(s["world"])]
        if s["app"] == 2:
            self._gc_run(s, out)
        while s["app"] != 2 and s["q"]:
            v = s["q"].pop(0)
            d = s["dist"][v] + 1
            for w in s["col"][s["off"][v]:s["off"][v + 1]]:
                w = int(w)
                if vb <= w < ve:
                    if d < s["dist"][w - vb]:
                        s["dist"][w - vb] = d
                        s["q"].append(w - vb)
                elif d < s["sent"][w]:
                    s["sent"][w] = d
                    r = int(np.searchsorted(b, w, side="right") - 1)
                    out[r].append(((w - int(b[r])) << 32) | int(d))
        s["out"] = out
        c = np.ctypeslib.as_array(ctypes.cast(counts_p, ctypes.POINTER(ctypes.c_int64)), (s["world"] + 1,))
        c[:] = [len(o) for o in out] + [0]
        return 0

    def atos_part_pack(self, h, dst, cap):
        import ctypes
        s = self._get(h)
        flat = [m for o in s["out"] for m in o]
        a = np.ctypeslib.as_array(ctypes.cast(dst, ctypes.POINTER(ctypes.c_uint64)), (max(cap, 1),))
        a[:len(flat)] = flat
        return 0

    def atos_part_apply(self, h, msgs, count):
        import ctypes
        s = self._get(h)
        if count and s["app"] == 2:
            a = np.ctypeslib.as_array(ctypes.cast(msgs, ctypes.POINTER(ctypes.c_uint64)), (count,))
            vb = int(s["b"][s["rank"]])
            changed = set()
            for m in a:
                u, c = int(m) >> 32, int(m) & 0xFFFFFFFF
                s["color"][u] = c
                changed.add(u)
            for v in range(s["n"]):
                vg = vb + v
                hit = any(int(u) in changed and int(u) < vg and s["color"][int(u)] == s["color"][vg]
                          for u in s["col"][s["off"][v]:s["off"][v + 1]])
                if hit and not s["pend"][v]:
                    s["pend"][v] = True
                    s["q"].append((v, 0))
        elif count:
            a = np.ctypeslib.as_array(ctypes.cast(msgs, ctypes.POINTER(ctypes.c_uint64)), (count,))
            for m in a:
                l, d = int(m) >> 32, int(m) & 0xFFFFFFFF
                if d < s["dist"][l]:
                    s["dist"][l] = d
                    s["q"].append(l)
        return 0

    def atos_part_finish(self, h, out, st):
        import ctypes
        s = self._get(h)
        if s["app"] == 2:
            a = np.ctypeslib.as_array(ctypes.cast(out, ctypes.POINTER(ctypes.c_int32)), (s["n"],))
            vb = int(s["b"][s["rank"]])
            a[:] = s["color"][vb:vb + s["n"]].astype(np.int32)
            return 0
        a = np.ctypeslib.as_array(ctypes.cast(out, ctypes.POINTER(ctypes.c_uint32)), (s["n"],))
        a[:] = s["dist"].astype(np.uint32)
        return 0

    def atos_graph_destroy(self, h):
        return 0

    def atos_config_default(self, cfg):
        return None


def main():
    rank, world, port, mode, app, outdir = (int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4],
                                            int(sys.argv[5]), sys.argv[6])
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
    import torch
    import torch.distributed as dist
    import graphgen as gg
    import paper_2112_00132_b200 as atos
    from paper_2112_00132_b200 import dist as adist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    if mode == "fake":
        fake = FakeLib()
        atos._lib = fake
        adist.lib = lambda: fake
        atos.lib = lambda: fake
    else:  # "gpu" / "gpu-discrete": every rank on cuda:0
        torch.cuda.set_device(0)
    g, fwd = gg.permute(gg.rmat(12, 8, seed=3, symmetrize=(app == 2)), 7)
    src = int(fwd[0])
    pg = adist.PartGraph.from_global(g, world, rank)
    kern = "discrete" if mode == "gpu-discrete" else "persistent"
    worker = os.environ.get("ATOS_TEST_WORKER", "cta")
    if app == 2:
        res, st = (adist.color(pg, timeout_s=60, kernel=kern, worker=worker) if mode != "fake"
                   else adist.color(pg))
    elif app == 0:
        res, st = adist.bfs(pg, src, timeout_s=60, kernel=kern) if mode != "fake" else adist.bfs(pg, src)
    else:
        res, st = adist.pagerank(pg, 0.85, 1e-6, timeout_s=60, kernel=kern)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), res=res, rounds=st.get("rounds", 0),
             bytes=st.get("bytes_sent", 0), src=src, num_colors=st.get("num_colors", 0))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

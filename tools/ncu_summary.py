"""Summarise an ncu report (raw metrics + stall reasons + top SASS stall sites) as markdown."""
import csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "lts__t_sectors_srcunit_tex_op_atom.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
        "lts__t_sectors_srcunit_tex_op_atom_evict_last_lookup_hit.sum",
        "lts__t_sectors_srcunit_tex_op_atom_evict_last_lookup_miss.sum"]


def run(rep, page, extra=()):
    return subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout


def main(rep, title):
    raw = list(csv.reader(io.StringIO(run(rep, "raw"))))
    h, u, v = raw[0], raw[1], raw[2]
    print(f"# {title}\n\nSource: `{rep}` (ncu --set full --clock-control none; one launch)\n")
    name_i = h.index("Kernel Name") if "Kernel Name" in h else None
    if name_i is not None:
        print(f"Kernel: `{v[name_i][:160]}`\n")
    print("| metric | value | unit |\n|---|---|---|")
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"| {k} | {v[i]} | {u[i]} |")
    st = [(n, float(v[i])) for i, n in enumerate(h)
          if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued") and v[i]]
    tot = sum(x for _, x in st) or 1
    print("\n## Warp stall sampling\n\n| reason | share |\n|---|---|")
    for n, x in sorted(st, key=lambda t: -t[1])[:8]:
        print(f"| {n.replace('smsp__pcsamp_warps_issue_stalled_', '')} | {x / tot * 100:.1f}% |")
    src = list(csv.reader(io.StringIO(run(rep, "source", ["--print-source", "sass"]))))
    hh = src[1]
    data = src[2:]
    iS = hh.index("Warp Stall Sampling (All Samples)")
    iSrc = hh.index("Source")
    tot = sum(float(r[iS] or 0) for r in data) or 1
    print("\n## Top SASS stall sites (sample share; the stalled instruction and the one before it)\n")
    print("| share | instruction | previous |\n|---|---|---|")
    for i in sorted(range(1, len(data)), key=lambda i: -float(data[i][iS] or 0))[:12]:
        print(f"| {float(data[i][iS]) / tot * 100:.1f}% | `{data[i][iSrc].strip()[:60]}` | `{data[i - 1][iSrc].strip()[:60]}` |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])

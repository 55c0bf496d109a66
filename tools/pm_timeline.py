"""SM occupancy and pipe/memory activity over time from an ncu report captured
with the PmSampling + PmSampling_WarpStates sections ("PM-sampling
section for occupancy over time").  Per time bin (a fraction of the kernel's
duration): resident warps per SM sub-partition as % of its 16-warp maximum
(the sum of the sampled warp-state counts over the interval's active cycles),
the share of those warp-cycles stalled on long_scoreboard (L2/DRAM loads and
atomics) and sleeping/wait (backoff, fixed-latency waits), L2 and DRAM
throughput, and instruction issue.  usage: pm_timeline.py REP [bins]"""
import csv
import io
import subprocess
import sys


def series(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-metric-instances", "values"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, v = rows[0], rows[2]
    res = {}
    for i, name in enumerate(h):
        if "TriageCompute." not in name and not name.startswith("pmsampling:"):
            continue
        val = v[i]
        if "(" not in val:
            continue
        try:
            xs = [float(x) for x in val[val.index("(") + 1:val.rindex(")")].split(";") if x.strip()]
        except ValueError:
            continue
        key = name.split("TriageCompute.", 1)[1] if "TriageCompute." in name else name.split(":", 1)[1]
        res[key] = xs
    return res


def trim(xs):
    """drop the leading/trailing idle samples (before launch / after exit)"""
    lo = next((i for i, x in enumerate(xs) if x > 0), 0)
    hi = len(xs) - next((i for i, x in enumerate(reversed(xs)) if x > 0), 0)
    return xs[lo:hi]


def binned(xs, bins):
    n = len(xs)
    return [sum(xs[b * n // bins:max(b * n // bins + 1, (b + 1) * n // bins)]) /
            max(1, len(xs[b * n // bins:max(b * n // bins + 1, (b + 1) * n // bins)])) for b in range(bins)]


def main(rep, bins=16):
    s = series(rep)
    states = {k: v for k, v in s.items() if k.startswith("smsp__warps_issue_stalled_")}
    m = min(len(v) for v in states.values())
    tot_raw = [sum(v[i] for v in states.values()) for i in range(m)]
    act = [i for i, t in enumerate(tot_raw) if t > 0]
    lo, hi = act[0], act[-1] + 1
    tot = tot_raw[lo:hi]
    pick = lambda k: states.get(k, [0.0] * m)[lo:hi]
    ls = pick("smsp__warps_issue_stalled_long_scoreboard.avg")
    slp = [a + b for a, b in zip(pick("smsp__warps_issue_stalled_sleeping.avg"), pick("smsp__warps_issue_stalled_wait.avg"))]
    # warp-state counts are warp-cycles per SM sub-partition per sampling interval; the interval of this
    # pass group is not reported, so resident warps are shown relative to the run's median sample
    # (the absolute mean is sm__warps_active in the --set full capture)
    med = sorted(tot)[len(tot) // 2] or 1.0
    occ_b = binned([t / med for t in tot], bins)
    ls_b = binned([a / max(t, 1.0) * 100 for a, t in zip(ls, tot)], bins)
    sl_b = binned([a / max(t, 1.0) * 100 for a, t in zip(slp, tot)], bins)
    cols = [("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 thr. %"),
            ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM thr. %"),
            ("sm__inst_executed_realtime.avg.pct_of_peak_sustained_elapsed", "issue %")]
    extra = [(lab, binned(trim(s[k]), bins)) for k, lab in cols if k in s]
    print(f"{len(tot)} warp-state samples over the kernel; {bins} bins of equal duration\n")
    print("| bin (of the run) | warps resident (/ median sample) | long_scoreboard % | sleeping+wait % | " +
          " | ".join(lab for lab, _ in extra) + " |")
    print("|---|---|---|---|" + "---|" * len(extra))
    for b in range(bins):
        print(f"| {b}/{bins} | {occ_b[b]:.2f} | {ls_b[b]:.1f} | {sl_b[b]:.1f} | " +
              " | ".join(f"{vals[b]:.1f}" for _, vals in extra) + " |")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 16)

"""Top source lines by warp-stall samples from an ncu report (--import-source,
-lineinfo build).  usage: ncu_source_hot.py REP [top]"""
import csv
import io
import subprocess
import sys


def main(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, tot, res = None, 0.0, []
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or not r[0].isdigit():
            continue
        try:
            s = float(r[4])
        except ValueError:
            continue
        tot += s
        res.append((s, f"{cur}:{r[0]}", r[1].strip()[:100]))
    res.sort(reverse=True)
    print("| share | line | source |\n|---|---|---|")
    for s, loc, src in res[:top]:
        print(f"| {100 * s / tot:.1f}% | {loc} | `{src}` |")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)

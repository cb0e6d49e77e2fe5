"""Per-source-line instruction and stall totals of one kernel in an ncu report
(needs -lineinfo + --import-source).  usage: ncu_lines.py REPORT LAUNCH_INDEX [top]"""
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "--launch-skip", idx, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
acc = {}
tot_e = tot_s = 0
for block in txt.split('"File Path"')[1:]:
    lines = block.splitlines()
    fname = lines[0].strip(',"').split("/")[-1]
    body = [l for l in lines[1:] if not l.startswith('"Function Name"')]
    rows = list(csv.reader(io.StringIO("\n".join(body))))
    hdr = rows[0]
    E = hdr.index("Instructions Executed")
    S = hdr.index("Warp Stall Sampling (All Samples)")
    cur = None
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        if r[0]:  # a source line
            cur = (f"{fname}:{r[0]}", r[1].strip()[:80])
            continue
        if cur is None or r[E] in ("", "-"):
            continue
        e, s_ = int(r[E]), int(r[S] or 0)
        tot_e += e
        tot_s += s_
        a = acc.setdefault(cur, [0, 0])
        a[0] += e
        a[1] += s_
print(f"total warp-instructions {tot_e}, stall samples {tot_s}")
for (loc, src), (e, s_) in sorted(acc.items(), key=lambda t: -t[1][0])[:top]:
    print(f"{e:>11} {100*e/max(tot_e,1):5.1f}%  stall {100*s_/max(tot_s,1):5.1f}%  {loc:22s} {src}")

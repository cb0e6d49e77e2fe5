"""Summarise an ncu report's SASS source page: hottest instructions by warp
stall samples (usage: python tools/ncu_hot.py REPORT [launch-index] [top])."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"]
if kre:
    cmd += ["--launch-skip", kre]
txt = subprocess.run(cmd, capture_output=True, text=True).stdout
lines = txt.splitlines()
# the page may hold several kernels; take the first table
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('"Kernel Name"')),
           len(lines))
print(lines[start - 1][:200])
rows = list(csv.reader(io.StringIO("\n".join(lines[start:end]))))
hdr = rows[0]
S = hdr.index("Warp Stall Sampling (All Samples)")
E = hdr.index("Instructions Executed")
tot = sum(int(r[S] or 0) for r in rows[1:])
print("total samples", tot)
best = sorted(rows[1:], key=lambda r: -int(r[S] or 0))[:top]
for r in best:
    print(f"{int(r[S]):7d} {100*int(r[S])/tot:5.1f}%  exec={r[E]:>10}  {r[0][-5:]}  {r[1].strip()}")

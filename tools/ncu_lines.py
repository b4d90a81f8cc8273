"""Per-CUDA-source-line warp-stall samples from an ncu report
(python tools/ncu_lines.py report.ncu-rep [kernel-regex] [topN])."""
import csv, io, subprocess, sys
rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if kre:
    cmd += ["-k", "regex:" + kre]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res = []
cur = None
for r in rows:
    if len(r) > 6 and r[0].isdigit():
        try:
            res.append((int(r[4]), int(r[0]), r[1][:110]))
        except ValueError:
            pass
tot = sum(x[0] for x in res) or 1
for s, ln, src in sorted(res, reverse=True)[:top]:
    print(f"{s:7d} {s/tot:6.1%}  L{ln:<5d} {src}")

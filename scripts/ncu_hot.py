"""Top SASS instructions by warp-stall samples from an ncu report (source page).
   python scripts/ncu_hot.py <report.ncu-rep> [N] [kernel-index]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = [b for b in out.split('"Kernel Name"') if b.strip()]
k = int(sys.argv[3]) if len(sys.argv) > 3 else 0
lines = ('"Kernel Name"' + blocks[k]).splitlines()
print(lines[0][:120])
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
si = h.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[si] or 0) for r in rows[1:] if len(r) > si)
rows = sorted(rows[1:], key=lambda r: -float(r[si] or 0))
for r in rows[:N]:
    print(f"{float(r[si])/tot*100:5.1f}%  {r[0][-5:]}  {r[1].strip()[:90]}")

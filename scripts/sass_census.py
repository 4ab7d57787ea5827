"""SASS instruction census of libkfac.so: per kernel, the instructions that prove which engine runs
(tcgen05 MMA / TMEM loads / TMA, fp64 DMMA, integer tensor MMA, warp MMA, cluster barriers, DSMEM)
plus register and shared-memory usage from cuobjdump's resource summary.

  python scripts/sass_census.py [libkfac.so] > profiles/rNN_sass_census.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2007_00784_b200", "libkfac.so")
CUOBJDUMP = os.environ.get("CUOBJDUMP", "/usr/local/cuda/bin/cuobjdump")

# opcode prefix -> column label
KEYS = [("UTCHMMA", "UTCHMMA (tcgen05 f16/tf32)"), ("UTCIMMA", "UTCIMMA (tcgen05 int8)"),
        ("UTCQMMA", "UTCQMMA"), ("UTMALDG", "UTMALDG (TMA load)"), ("UTMASTG", "UTMASTG"),
        ("LDTM", "LDTM (TMEM load)"), ("DMMA", "DMMA (fp64 MMA)"), ("HMMA", "HMMA"), ("IMMA", "IMMA"),
        ("LDGSTS", "LDGSTS (cp.async)"), ("SYNCS", "SYNCS (mbarrier)"), ("UCGABAR", "UCGABAR (cluster bar)"),
        ("MEMBAR", "MEMBAR"), ("DFMA", "DFMA"), ("FFMA", "FFMA")]

sass = subprocess.run([CUOBJDUMP, "-sass", lib], capture_output=True, text=True).stdout
res = subprocess.run([CUOBJDUMP, "-res-usage", lib], capture_output=True, text=True).stdout

counts = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m:
        op = m.group(2)
        for k, _ in KEYS:
            if op.startswith(k):
                counts[cur][k] += 1
                break

usage = {}
fn = None
for line in res.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r"REG:(\d+).*SHARED:(\d+)", line)
    if m and fn:
        usage[fn] = (int(m.group(1)), int(m.group(2)))


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return [re.sub(r"\(.*", "", o.replace("(anonymous namespace)::", "")) for o in out]


names = list(counts)
pretty = demangle(names)
used = [k for k, _ in KEYS if any(counts[n][k] for n in names)]
print(f"# SASS census: `{os.path.basename(lib)}` (cuobjdump -sass, sm_100a)\n")
print("Static instruction counts per kernel (occurrences in the SASS, not executions).\n")
print("| kernel | regs | static smem B | " + " | ".join(dict(KEYS)[k] for k in used) + " |")
print("|---|---|---|" + "---|" * len(used))
for n, p in sorted(zip(names, pretty), key=lambda t: t[1]):
    r, sm = usage.get(n, ("", ""))
    print(f"| `{p}` | {r} | {sm} | " + " | ".join(str(counts[n][k] or "") for k in used) + " |")

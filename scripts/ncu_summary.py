"""Summarise ncu outputs into profiles/ (committed evidence).

  python scripts/ncu_summary.py launches <launches.csv> <out.md>   # per-kernel time share
  python scripts/ncu_summary.py full <report.ncu-rep> <out.md>     # key metrics of a --set full capture
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tc pipe active %"),
    ("sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active", "UMMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall mio_throttle"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math_pipe_throttle"),
]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    t, c = collections.defaultdict(float), collections.defaultdict(int)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
        name = r[ki].split("(")[0].replace("kfac::<unnamed>::", "kfac::")[:70]
        t[name] += v * scale
        c[name] += 1
    tot = sum(t.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list: {path}\n\n")
        f.write("Per-launch gpu__time_duration.sum (cold-cache, serialised replay; compare shares).\n\n")
        f.write(f"Total {tot:.3f} ms over {sum(c.values())} launches.\n\n")
        f.write("| kernel | launches | total ms | share | avg us |\n|---|---|---|---|---|\n")
        for k, v in sorted(t.items(), key=lambda x: -x[1]):
            f.write(f"| `{k}` | {c[k]} | {v:.3f} | {100 * v / tot:.1f}% | {1000 * v / c[k]:.1f} |\n")
    print(open(out).read())


def full(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary: {path}\n\n")
        for r in rows[2:] if len(rows) > 2 and rows[1][0] == "" else rows[1:]:
            d = dict(zip(h, r))
            name = d.get("Kernel Name", "?").split("(")[0]
            f.write(f"## `{name}`\n\n| metric | value |\n|---|---|\n")
            for k, label in KEYS:
                if k in d and d[k] not in ("", "n/a"):
                    f.write(f"| {label} (`{k}`) | {d[k]} |\n")
            f.write("\n")
    print(open(out).read())


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])

"""Summarise an ncu report (or a launch-list CSV) into the text kept under
profiles/. Usage:
    python paper_1505_07368_b200/tools/ncu_summary.py report.ncu-rep > profiles/x.txt
    python paper_1505_07368_b200/tools/ncu_summary.py --launches launches.csv > profiles/y.txt
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarise(rep):
    hdr, units, data = raw(rep)
    for row in data:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        print(f"== kernel: {d.get('Kernel Name', '?')}")
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]:>16s} {u.get(k, '')}")
        stalls = [(float(d[k].replace(',', '') or 0), k) for k in hdr
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("not_issued") and d[k] not in ("", "0")]
        tot = sum(v for v, _ in stalls) or 1
        print("  warp-state samples (share):")
        for v, k in sorted(stalls, reverse=True)[:8]:
            print(f"    {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {v / tot:6.1%}")


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    per = collections.defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) > iv and r[iv]:
            v = float(r[iv].replace(",", ""))
            if r[iu] in ("usecond", "us"):
                v *= 1e3
            elif r[iu] in ("msecond", "ms"):
                v *= 1e6
            per[r[ik][:90]].append(v)
    tot = sum(sum(v) for v in per.values())
    print(f"{'kernel':90s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:90s} {len(v):8d} {sum(v) / 1e6:10.3f} {sum(v) / tot:7.1%}")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        summarise(sys.argv[1])

"""Key metrics of an ncu --set full report (+ top SASS stall lines)."""
import csv
import io
import subprocess
import sys

KEEP = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'Executed Ipc Active',
        'Issue Slots Busy', 'Warp Cycles Per Issued Instruction', 'Registers Per Thread', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Executed Instructions', 'Grid Size', 'Dynamic Shared Memory Per Block',
        'Eligible Warps Per Scheduler', 'Active Warps Per Scheduler', 'L1/TEX Cache Throughput', 'L2 Cache Throughput',
        'Compute (SM) Throughput', 'Block Limit Registers', 'Block Limit Shared Mem']


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def dram_bytes(rep):
    """dram__bytes_read.sum + dram__bytes_write.sum of the first captured launch, in bytes."""
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hh, units, vals = raw[0], raw[1], raw[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hh.index(k)
        tot += float(vals[i].replace(",", "")) * scale[units[i]]
    return tot


def record_traffic(rep, out, kernel, workload):
    """Merges {kernel: {workload, dram_bytes_per_launch, report}} into `out` (read by bench.py)."""
    import json
    import os
    d = json.load(open(out)) if os.path.exists(out) else {}
    d[kernel] = {"workload": workload, "dram_bytes_per_launch": dram_bytes(rep), "report": os.path.basename(rep)}
    json.dump(d, open(out, "w"), indent=1)


def l1tex_util(rep):
    """L1/TEX cache throughput (% of peak) and hit rate of the first captured launch: the
    ceiling of the OFA kernels, whose V gathers and table reads all go through L1/shared."""
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    h = rows[0]
    out = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d["Metric Name"] in ("L1/TEX Cache Throughput", "L1/TEX Hit Rate", "Duration", "Issue Slots Busy",
                                "Achieved Occupancy"):
            out.setdefault(d["Metric Name"], float(d["Metric Value"].replace(",", "")))
    return out


def record_l1tex(rep, out, kernel, workload):
    """Merges {kernel: {workload, l1tex_pct_of_peak, ...}} into `out` (read by bench.py)."""
    import json
    import os
    d = json.load(open(out)) if os.path.exists(out) else {}
    u = l1tex_util(rep)
    d[kernel] = {"workload": workload, "l1tex_pct_of_peak": u.get("L1/TEX Cache Throughput"),
                 "l1tex_hit_rate_pct": u.get("L1/TEX Hit Rate"), "issue_slots_busy_pct": u.get("Issue Slots Busy"),
                 "achieved_occupancy_pct": u.get("Achieved Occupancy"), "report": os.path.basename(rep)}
    json.dump(d, open(out, "w"), indent=1)


def main(rep, top=25):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    h = rows[0]
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d["Metric Name"] in KEEP:
            print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    if len(raw) > 2:
        hh = raw[0]
        vals = raw[2]
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if k in hh:
                print(f"{k:40s} {vals[hh.index(k)]} {raw[1][hh.index(k)]}")
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    hs = src[1]
    data = [dict(zip(hs, r)) for r in src[2:] if len(r) == len(hs)]
    tot = sum(int(d["Warp Stall Sampling (All Samples)"]) for d in data) or 1
    exs = sum(int(d["Instructions Executed"]) for d in data) or 1
    print("--- top stall lines")
    for d in sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"]))[:top]:
        print(f"{int(d['Warp Stall Sampling (All Samples)']) / tot * 100:5.1f}% "
              f"ex={int(d['Instructions Executed']) / exs * 100:5.2f}%  {d['Source'][:80]}")


if __name__ == "__main__":
    # ncu_summary.py REPORT [TOP]  |  ncu_summary.py --traffic OUT.json KERNEL WORKLOAD REPORT
    if sys.argv[1] == "--traffic":
        record_traffic(sys.argv[5], sys.argv[2], sys.argv[3], sys.argv[4])
    elif sys.argv[1] == "--l1tex":
        record_l1tex(sys.argv[5], sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)

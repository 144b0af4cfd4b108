"""Compact per-kernel text summary of an `ncu --set full` report (.ncu-rep), for profiles/.
usage: ncu_summary.py report.ncu-rep [kernel-regex]

Per kernel launch: duration, DRAM bytes read / written and the resulting bandwidth, warp
instructions, issue-slot utilisation, achieved occupancy, registers, and the top warp-stall
reasons (pc-sampling, share of samples)."""
import csv
import io
import re
import subprocess
import sys

STALL = "smsp__pcsamp_warps_issue_stalled_"


def raw(report, kregex=None):
    cmd = ["ncu", "-i", report, "--page", "raw", "--csv"]
    if kregex:
        cmd += ["-k", f"regex:{kregex}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def num(row, h, key, scale=1.0):
    try:
        return float(row[h.index(key)].replace(",", "")) * scale
    except (ValueError, IndexError):
        return float("nan")


def unit_scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
            "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "us": 1.0, "ns": 1e-3, "ms": 1e3}.get(u, 1.0)


def main():
    report = sys.argv[1]
    h, units, rows = raw(report, sys.argv[2] if len(sys.argv) > 2 else None)
    U = dict(zip(h, units))
    for r in rows:
        name = re.sub(r"\(.*", "", r[h.index("Kernel Name")]).replace("vks::<unnamed>::", "")
        t_us = num(r, h, "gpu__time_duration.sum", unit_scale(U.get("gpu__time_duration.sum")))
        rd = num(r, h, "dram__bytes_read.sum", unit_scale(U.get("dram__bytes_read.sum")))
        wr = num(r, h, "dram__bytes_write.sum", unit_scale(U.get("dram__bytes_write.sum")))
        inst = num(r, h, "smsp__inst_executed.sum")
        issue = num(r, h, "smsp__issue_active.avg.pct_of_peak_sustained_active")
        occ = num(r, h, "sm__warps_active.avg.pct_of_peak_sustained_active")
        regs = num(r, h, "launch__registers_per_thread")
        grid = r[h.index("Grid Size")] if "Grid Size" in h else "?"
        block = r[h.index("Block Size")] if "Block Size" in h else "?"
        stalls = {k[len(STALL):]: num(r, h, k) for k in h if k.startswith(STALL) and not k.endswith("not_issued")}
        tot = sum(v for v in stalls.values() if v == v) or 1.0
        top = sorted(stalls.items(), key=lambda kv: -(kv[1] if kv[1] == kv[1] else 0))[:4]
        bw = (rd + wr) / (t_us * 1e-6) / 1e9 if t_us == t_us and t_us > 0 else float("nan")
        print(f"{name}  grid {grid} block {block} regs {regs:.0f}")
        print(f"    {t_us:9.1f} us   dram rd {rd / 1e6:8.1f} MB  wr {wr / 1e6:8.1f} MB  -> {bw:7.0f} GB/s   "
              f"inst {inst / 1e6:7.1f} M  issue {issue:5.1f}%  occupancy {occ:5.1f}%")
        print("    stalls: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))


if __name__ == "__main__":
    main()

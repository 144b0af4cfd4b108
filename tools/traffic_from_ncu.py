"""Write profiles/rNN_traffic.json: DRAM bytes (read + write), issue-slot utilisation and warp
instructions per launch of each hot-path stage's dominant kernel, from one `ncu --set full`
capture (bench.py reports them as roofline.traffic / roofline.issue).
usage: traffic_from_ncu.py report.ncu-rep [out.json]"""
import csv
import io
import json
import re
import subprocess
import sys

STAGES = {  # bench stage -> kernel-name regex of its dominant kernel
    "raster_bwd": r"raster_bwd_kernel",
    "raster_fwd": r"raster_fwd_kernel",
    "project_fwd": r"project_fwd_batch_kernel",  # per launch = one batch of 8 views
    "project_bwd": r"project_bwd_batch_kernel",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep = sys.argv[1]
    out = sys.argv[2] if len(sys.argv) > 2 else "profiles/r1_traffic.json"
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                          "smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        for stage, rx in STAGES.items():
            if re.search(rx, name) and stage not in res:
                rd = float(r[h.index("dram__bytes_read.sum")]) * SCALE[units[h.index("dram__bytes_read.sum")]]
                wr = float(r[h.index("dram__bytes_write.sum")]) * SCALE[units[h.index("dram__bytes_write.sum")]]
                iss = float(r[h.index("smsp__issue_active.avg.pct_of_peak_sustained_active")]) / 100.0
                ui = units[h.index("smsp__inst_executed.sum")]
                inst = float(r[h.index("smsp__inst_executed.sum")].replace(",", "")) * {"inst": 1, "Kinst": 1e3,
                                                                                      "Minst": 1e6, "Ginst": 1e9}.get(ui, 1)
                res[stage] = dict(kernel=re.sub(r"\(.*", "", name), dram_bytes_read=rd, dram_bytes_write=wr,
                                  dram_bytes_per_launch=rd + wr, issue_active=round(iss, 4),
                                  warp_instructions_per_launch=inst)
    json.dump(dict(source=rep.split("/")[-1], note="one ncu --set full capture of tools/profile_bench_step.py "
                   "(bicycle: batched projection of 8 views, view 0's raster passes); per launch", kernels=res), open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

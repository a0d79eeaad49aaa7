"""Raw counters of the round's `ncu --set full` captures -> profiles/<tag>_ncu_full_raw.csv
(byte counters normalised to GB, times to ms).   python tools/ncu_raw_csv.py r02"""
import csv
import glob
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COLS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active", "lts__t_sector_hit_rate.pct", "launch__registers_per_thread"]
STALL = ["barrier", "long_scoreboard", "short_scoreboard", "wait", "branch_resolving", "math_pipe_throttle"]
SCALE = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6, "s": 1e3, "second": 1e3}

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
out = open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full_raw.csv"), "w", newline="")
w = csv.writer(out)
w.writerow(["kernel"] + COLS + ["smsp__pcsamp_warps_issue_stalled_" + s for s in STALL])
for rep in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", f"{tag}_full_*.ncu-rep"))):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, unit = rows[0], rows[1]
    for r in rows[2:]:
        def val(c):
            if c not in hdr:
                return ""
            i = hdr.index(c)
            v = float(r[i].replace(",", "") or 0)
            return f"{v * SCALE.get(unit[i], 1.0):.6f}" if unit[i] in SCALE else r[i]
        w.writerow([r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")] + [val(c) for c in COLS] +
                   [val("smsp__pcsamp_warps_issue_stalled_" + s) for s in STALL])
out.close()
print(open(out.name).read())

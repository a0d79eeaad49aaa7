"""Summarise ncu outputs (launch list CSV + full report) into profiles/ (tracked)."""
import csv, collections, json, subprocess, sys, os

def launches(path, out_csv):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per = {}
    for r in data:
        if len(r) < len(hdr):
            continue
        per.setdefault(int(r[ii]), {"k": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    ids = sorted(per)
    half = ids[len(ids) // 2:]  # bench --steps 1 --warmup 1: second half = the timed step
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    with open(out_csv, "w") as f:
        f.write("id,kernel,time_ns,dram_read_bytes,dram_write_bytes\n")
        for i in ids:
            d = per[i]
            name = d["k"].split("(")[0].replace("void ", "").split("::")[-1]
            f.write(f"{i},{name},{d.get('gpu__time_duration.sum', 0):.0f},{d.get('dram__bytes_read.sum', 0):.0f},"
                    f"{d.get('dram__bytes_write.sum', 0):.0f}\n")
    for i in half:
        d = per[i]
        name = d["k"].split("(")[0].replace("void ", "").split("::")[-1]
        a = agg[name]
        a[0] += 1; a[1] += d.get("gpu__time_duration.sum", 0); a[2] += d.get("dram__bytes_read.sum", 0); a[3] += d.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    lines = ["| kernel | launches | time (ms) | share | DRAM read (GB) | DRAM write (GB) |", "|---|---|---|---|---|---|"]
    for n, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        if a[1] / tot < 0.001:
            continue
        lines.append(f"| `{n}` | {a[0]} | {a[1]/1e6:.2f} | {a[1]/tot*100:.1f}% | {a[2]/1e9:.2f} | {a[3]/1e9:.2f} |")
    return "\n".join(lines), tot

def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(out.splitlines()); hdr = next(r)
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Issue Slots Busy",
            "Achieved Occupancy", "Registers Per Thread", "L2 Hit Rate", "L1/TEX Hit Rate", "Eligible Warps Per Scheduler"]
    rows = {}
    for row in r:
        if row[mi] in want:
            rows.setdefault((int(row[ii]), row[ki].split("(")[0].replace("void ", "").split("::")[-1]), {})[row[mi]] = row[vi]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines())); rh = rr[0]
    traffic = {}
    for row in rr[2:]:
        try:
            traffic[int(row[rh.index("ID")])] = (float(row[rh.index("dram__bytes_read.sum")]), float(row[rh.index("dram__bytes_write.sum")]),
                                                 rh and row[rh.index("dram__bytes_read.sum")])
        except (ValueError, IndexError):
            pass
    lines = ["| id | kernel | " + " | ".join(want) + " | dram read+write |", "|" + "---|" * (len(want) + 3)]
    for (i, k), v in sorted(rows.items()):
        t = traffic.get(i)
        lines.append(f"| {i} | `{k}` | " + " | ".join(v.get(w, "") for w in want) + f" | {t[0]+t[1] if t else ''} |")
    return "\n".join(lines)

CLASS = {"tile_scatter_kernel": "part_scatter", "tile_hist_kernel": "part_hist", "bucket_unique_kernel": "bucket_unique",
         "bucket_compact_kernel": "pack", "group_off_kernel": "pack", "owner_bounds_kernel": "pack",
         "gen_kernel": "gen", "merge_tile_kernel": "merge_tile", "merge_split_kernel": "merge_split",
         "scatter1_kernel": "part_scatter", "tile_scatter_atomic_kernel": "part_scatter",
         "sparse_copy_kernel": "merge_tile", "sparse_place_kernel": "merge_tile",
         "sparse_locate_kernel": "merge_split", "sparse_bounds_kernel": "merge_split",
         "copy_check_kernel": "sorted_check", "check_sorted_kernel": "sorted_check",
         "run_bounds_kernel": "pack", "run_offsets_kernel": "pack"}


def traffic_json(path, out_json, meta=None):
    """per profiler class: DRAM bytes per launch from the launch list (timed step)."""
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per = {}
    for r in data:
        if len(r) < len(hdr):
            continue
        per.setdefault(int(r[ii]), {"k": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    ids = sorted(per)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i in ids[len(ids) // 2:]:
        d = per[i]
        name = d["k"].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
        c = CLASS.get(name)
        if c:
            a = agg[c]
            a[0] += 1
            a[1] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
            a[2] += d.get("gpu__time_duration.sum", 0)
    out = {c: {"launches": a[0], "dram_bytes_per_launch": a[1] / a[0], "ncu_ms_per_launch": a[2] / a[0] / 1e6}
           for c, a in agg.items() if a[0]}
    json.dump({"source": path, **(meta or {}), "classes": out}, open(out_json, "w"), indent=1)
    return out


if __name__ == "__main__":
    # python tools/summarize_ncu.py TAG [WORKLOAD PARENTS EPS]
    tag = sys.argv[1]
    wl = sys.argv[2] if len(sys.argv) > 2 else "n2"
    meta = {"workload": wl, "parents": int(sys.argv[3]) if len(sys.argv) > 3 else 1_000_000,
            "eps": float(sys.argv[4]) if len(sys.argv) > 4 else 0.0}
    print(json.dumps(traffic_json(f"gpurun_out/{tag}_launches.csv", f"profiles/{tag}_{wl}_traffic.json", meta), indent=1))
    tbl, tot = launches(f"gpurun_out/{tag}_launches.csv", f"profiles/{tag}_launches.csv")
    print(tbl)
    import glob
    for rep in sorted(glob.glob(f"gpurun_out/{tag}_full*.ncu-rep")):
        print()
        print(f"### {os.path.basename(rep)}")
        print(full(rep))

"""Refresh the measured numbers in profiles/README.md from profiles/r01_bench.json,
the ncu launch list and the --set full captures of gpurun_out/ (run after
tools/summarize_ncu.py r01).  Text outside the generated blocks is kept."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import summarize_ncu as S  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
d = json.load(open(os.path.join(ROOT, "profiles", f"{tag}_bench.json")))
kr, km = d["kernel_roofline"], d["kernel_ms_per_step"]
p = os.path.join(ROOT, "profiles", "README.md")
s = open(p).read()


def between(s, a, b, new):
    i, j = s.index(a), s.index(b)
    return s[:i] + new + s[j:]


hist = s[s.index("* Round history:"):s.index("\n", s.index("* Round history:"))]
old = hist.split("→")[-1].replace("ms/step now.", "").strip()
now = f"{d['ms_per_step']:.1f}"
if now != old:
    hist = hist.replace(f"{old} ms/step now.", f"{old} → {now} ms/step now.")
s = between(s, "* **", "* clocks:",
            f"* **{d['value']:.3g} coupled configs/s** ({d['ms_per_step']:.1f} ms/step, {d['config']['records_per_step']:,} records/step),\n"
            f"  **{d['unique_configs_per_s']:.3g} unique configs/s** ({d['config']['unique_per_step']:,} unique; redundancy {d['redundancy']:.3f});\n"
            f"  e2e through host parents (pinned H2D + D2H inside the region): {d['e2e']['value']:.3g}/s ({d['e2e']['ms_per_step']:.1f} ms/step).\n"
            + hist + "\n")
f2, s3 = d["f2_regular_sampling"], d["stage3_contract"]
t1 = f2["table1_P8"]
s = between(s, "* cpu_baseline", "| kernel class",
            f"* cpu_baseline (the oracle, 1 host thread, first 1,000 parents): {d['cpu_baseline']['value']:.3g} coupled configs/s; oracle-MT (the same\n"
            f"  oracle sharded over the box's {d['cpu_baseline_mt']['cores']} host threads): {d['cpu_baseline_mt']['value']:.3g} coupled configs/s (`cpu_baseline_mt`).\n"
            f"* Stage-3 contraction (f1, not in the step): {s3['records_per_s']:.3g} records/s over the same records ({s3['ms_per_step']:.0f} ms for the 2 batches).\n"
            f"* Regular-sampling dedup (f2, not in the step), one batch of {f2['records']:,} records: `dedup_sorted`\n"
            f"  {f2['dedup_sorted_ms']:.1f} ms vs the hash `dedup_global` {f2['dedup_global_ms']:.1f} ms.  Paper Table-1 metrics for P = 8 virtual\n"
            f"  ranks: regular sampling (S = 1024) max/min {t1['regular_sampling']['max_over_min']:.3f}, CV {t1['regular_sampling']['cv']:.3f};\n"
            f"  hash owner max/min {t1['hash_owner']['max_over_min']:.4f}, CV {t1['hash_owner']['cv']:.1e}.\n\n")
rows = "".join(f"| {k if k != 'merge' else 'merge (merge_split + merge_tile + copy/check: every merge_space kernel)'} | "
               f"{v['ms_per_step']:.1f} | {v['achieved_GBs']:,.0f} | {v['frac']:.2f} |\n"
               for k, v in sorted(kr.items(), key=lambda kv: -kv[1]["ms_per_step"]))
i = s.index("| kernel class")
i = s.index("\n", s.index("\n", i) + 1) + 1
j = s.index("\n", s.index("| pack + scan")) + 1
s = s[:i] + rows + f"| pack + scan | {km.get('pack', 0) + km.get('scan', 0):.1f} | | |\n" + s[j:]
tbl, _ = S.launches(os.path.join(ROOT, "gpurun_out", f"{tag}_launches.csv"), os.path.join(ROOT, "profiles", f"{tag}_launches.csv"))
s = between(s, "| kernel | launches |", "The shares agree", tbl + "\n\n")
# full captures: update the rows of the kernels captured this time
full = S.full(os.path.join(ROOT, "gpurun_out", f"{tag}_full.ncu-rep")).splitlines()[2:]
for line in full:
    c = [x.strip() for x in line.strip("|").split("|")]
    name = c[1]
    vals = dict(dur=c[2], dram=c[3], issue=c[6], occ=c[7], regs=c[8], l2=c[9], elig=c[11], tr=float(c[12]))
    k0 = s.index("## Full captures")
    head, tail = s[:k0], s[k0:]
    for row in tail.splitlines():
        if row.startswith(f"| {name}") and "Duration" not in row:
            cells = [x.strip() for x in row.strip("|").split("|")]
            cells[1:] = [f"{float(vals['dur']):.2f}", f"{float(vals['dram']):.1f}", f"{float(vals['issue']):.1f}",
                         f"{float(vals['occ']):.1f}", vals["regs"], f"{float(vals['l2']):.1f}", f"{float(vals['elig']):.2f}",
                         f"{vals['tr']:.2f}"]
            tail = tail.replace(row, "| " + " | ".join(cells) + " |")
            break
    s = head + tail
s = s.replace(s[s.index("fraction against HBM ("):s.index(")", s.index("fraction against HBM (")) + 1],
              f"fraction against HBM ({kr['bucket_unique']['frac']:.2f})")
open(p, "w").write(s)
print("updated", p)

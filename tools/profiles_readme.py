"""Write the round section of profiles/README.md from profiles/<tag>_bench.json, the ncu
launch list (gpurun_out/<tag>_launches.csv), profiles/<tag>_ncu_full_raw.csv and the side
benches; the older rounds' sections below it are kept.   python tools/profiles_readme.py r02"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import summarize_ncu as S  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
P = lambda *a: os.path.join(ROOT, *a)  # noqa: E731
d = json.load(open(P("profiles", f"{tag}_bench.json")))
kr = d["kernel_roofline"]
dd, f2, s3, f3, f4 = d["dedup_roofline"], d["f2_regular_sampling"], d["stage3_contract"], d["f3_streaming"], d["f4_sci_growth"]
t1 = f2["table1_P8"]
rf = d["roofline"]
L = [f"## Round {int(tag[1:])}\n",
     f"Produced by `tools/round_profile.sh {tag}` (build → `pytest -m gpu` → smoke → `bench.py` → ncu launch list of\n"
     "`bench.py --steps 1 --warmup 1` → one `ncu --set full` capture per top kernel), summarised by `tools/summarize_ncu.py`\n"
     f"and `tools/profiles_readme.py`; side configurations by `tools/side_benches.sh`; sanitizers by `tools/sanitize.sh`.\n",
     f"* `{tag}_bench.json`: the bench line (CUDA events, {d['steps']} timed steps after {d['warmup']} warm-up, clocks sampled during the run).",
     f"* `{tag}_launches.csv`, `{tag}_n2_traffic.json`: every launch of the ncu-profiled step (time, DRAM bytes) and DRAM bytes per\n  launch per kernel class (read by `bench.py` as `traffic`).",
     f"* `{tag}_ncu_full_raw.csv`: raw counters of the five `--set full` captures (gen, both partition passes, bucket_unique, merge_tile).",
     f"* `{tag}_sanitizer_{{memcheck,racecheck,synccheck,memcheck_large}}.log`: compute-sanitizer over every kernel path (mid-round-2 code, see Reading): 0 errors, 0 hazards.",
     f"* `{tag}_gpu_tests.log`, `{tag}_smoke.log`: the GPU test suite and the smoke run.",
     f"* `{tag}_{{eps,m120,c2h4,h2o}}_bench.json`: the other BASELINE configurations.\n",
     "### Bench line (N2 cc-pVDZ-like: 56 spin orbitals, 14 electrons, 10^6 parents, eps = 0)\n",
     f"* **{d['value']:.3g} coupled configs/s** ({d['ms_per_step']:.1f} ms/step, {d['config']['records_per_step']:,} records/step),",
     f"  **{d['unique_configs_per_s']:.3g} unique configs/s** ({d['config']['unique_per_step']:,} unique; redundancy {d['redundancy']:.3f});",
     f"  e2e through `stream_generate` from pinned host parents: {d['e2e']['value']:.3g}/s ({d['e2e']['ms_per_step']:.1f} ms/step).",
     f"* Round history: 171.4 (round-1 start) → 105.2 (round-1 end) → 96.1 (round-2 start) → 92.4 (mid round 2) → {d['ms_per_step']:.1f} ms/step.",
     f"* `roofline` (headline): `{rf['kernel']}` at {rf['frac']:.3f} of the {rf['peak']:,.0f} GB/s measured copy peak ({rf['achieved']:,.0f} GB/s of algorithmic bytes;\n"
     f"  DRAM traffic {rf['traffic']/1e9:.2f} GB per launch vs {rf['alg_bytes_per_launch']/1e9:.2f} GB algorithmic).",
     f"* clocks {d['clocks']['sm_mhz']:.0f} MHz median under load (max {d['clocks']['sm_max_mhz']:.0f}), throttle reasons {d['clocks']['reasons']}; {d['gpu_launches']} library launches in the timed region.",
     f"* cpu_baseline (the oracle, 1 thread, 1,000 parents): {d['cpu_baseline']['value']:.3g} coupled configs/s; oracle-MT ({d['cpu_baseline_mt']['cores']} threads): {d['cpu_baseline_mt']['value']:.3g}/s.",
     f"* dedup as a whole (SURVEY 8(d): read N keys, write U): {dd['ms_per_step']:.1f} ms/step, {dd['frac']:.3f} of the copy peak, DRAM-traffic\n  amplification {dd['traffic_amplification']:.2f} (the partition passes' own reads and writes).",
     f"* f1 contraction (not in the step): {s3['records_per_s']:.3g} records/s ({s3['ms_per_step']:.0f} ms for the step's 3.9e9 records).",
     f"* f2 (not in the step), one batch of {f2['records']:,} records: `dedup_sorted` {f2['dedup_sorted_ms']:.1f} ms vs `dedup_global` {f2['dedup_global_ms']:.1f} ms;\n"
     f"  Table-1 for P = 8 virtual ranks: regular sampling max/min {t1['regular_sampling']['max_over_min']:.3f} (CV {t1['regular_sampling']['cv']:.3f}), hash owner {t1['hash_owner']['max_over_min']:.4f} (CV {t1['hash_owner']['cv']:.1e})."]
s1, r3, g3 = f3["stage1_offload"], f3["stage3_reload"], f3["stage3_regenerate"]
L.append(f"* f3 (not in the step), {f3['parents']:,} parents in {f3['batches']} mini-batches, {f3['records']:,} records ({f3['record_bytes']} B each) offloaded:\n"
         f"  Stage 1 wall {s1['ms_wall']:.0f} ms with the D2H stream busy {s1['ms_d2h']:.0f} ms of it ({s1['d2h_GBs']:.1f} GB/s, overlapped with compute), peak device\n"
         f"  {s1['peak_device_bytes']/1e9:.1f} GB; Stage 3 reload {r3['ms_wall']:.0f} ms (H2D-bound) vs regenerate {g3['ms_wall']:.1f} ms, e identical: {f3['stage3_identical']}.")
L.append("* f4 growth from 2,000 parents (K = 4|S|): " + "; ".join(
    f"|S| {i['space_before']:,} → {i['records']:,} records, {i['unique']:,} unique (redundancy {i['redundancy']:.2f})" for i in f4["iterations"]) + ".\n")
L += ["| kernel class | ms/step | algorithmic GB/s | fraction of the measured copy peak |", "|---|---|---|---|"]
for k, v in sorted(kr.items(), key=lambda kv: -kv[1]["ms_per_step"]):
    nm = {"merge": "merge (merge_split + merge_tile + copy/check)",
          "part_scatter": "part_scatter (pass bytes: implementation overhead)"}.get(k, k)
    L.append(f"| {nm} | {v['ms_per_step']:.1f} | {v['achieved_GBs']:,.0f} | {v['frac']:.2f} |")
L.append("\n### Launch list (ncu `--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none`; the timed step; cold-cache, serialised)\n")
tbl, _ = S.launches(P("gpurun_out", f"{tag}_launches.csv"), P("profiles", f"{tag}_launches.csv"))
L.append(tbl + "\n")
L.append("### Full captures (`ncu --set full --clock-control none`, one full-size launch each)\n")
L += ["| kernel | duration (ms) | DRAM read+write (GB) | warp-instr | issue active % | warps active % | eligible / sched | L2 hit % | regs | top stalls (samples) |",
      "|---|---|---|---|---|---|---|---|---|---|"]
for r in csv.DictReader(open(P("profiles", f"{tag}_ncu_full_raw.csv"))):
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v) for k, v in r.items() if "stalled" in k and v}
    top = ", ".join(f"{k} {int(v / 1000)}k" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
    L.append(f"| `{r['kernel'].replace('unnamed>::', '')}` | {float(r['gpu__time_duration.sum']):.2f} | "
             f"{float(r['dram__bytes_read.sum']) + float(r['dram__bytes_write.sum']):.1f} | {float(r['smsp__inst_executed.sum']):.3g} | "
             f"{float(r['smsp__issue_active.avg.pct_of_peak_sustained_active']):.1f} | {float(r['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f} | "
             f"{float(r['smsp__warps_eligible.avg.per_cycle_active']):.2f} | {float(r['lts__t_sector_hit_rate.pct']):.1f} | {r['launch__registers_per_thread']} | {top} |")
body = "\n".join(L) + "\n"
p = P("profiles", "README.md")
s = open(p).read()
i = s.index(f"## Round {int(tag[1:])}\n")
j = s.index("### Reading", i)
open(p, "w").write(s[:i] + body + "\n" + s[j:])
print("updated", p)

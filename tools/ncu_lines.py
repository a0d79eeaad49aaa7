"""Per-source-line instruction / stall-sample breakdown of an ncu report
(--import-source on, -lineinfo): python tools/ncu_lines.py REPORT [kernel-regex] [N] [skip]."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
skip = int(sys.argv[4]) if len(sys.argv) > 4 else 0  # matching launches to skip
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", "--kernel-name",
                      f"regex:{kre}", "--launch-skip", str(skip), "--launch-count", "1"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
hdr = rows[hi]
ie = hdr.index("Instructions Executed")
ws = hdr.index("Warp Stall Sampling (All Samples)")
cur, agg, src = None, {}, {}
for r in rows[hi + 1:]:
    if len(r) < len(hdr) or r[0] == "Line No":
        continue
    if r[0] != "":
        cur = int(r[0])
        src[cur] = r[1]
    if r[2] in ("", "..."):
        continue
    try:
        n, s = int(r[ie]), int(r[ws])
    except ValueError:
        continue
    a = agg.setdefault(cur, [0, 0])
    a[0] += n
    a[1] += s
tot = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instructions {tot:.4g}, stall samples {ts}")
for l, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{l:5d} {n / tot * 100:5.1f}% inst {s / ts * 100:5.1f}% stall  {src.get(l, '').strip()[:100]}")

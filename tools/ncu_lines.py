"""Per-source-line totals (stall samples, warp instructions) from an ncu report."""
import csv, subprocess, sys, io
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
hdr = rows[hi]
si, ii = 4, 7
def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
lines = []
for r in rows[hi + 1:]:
    if len(r) < 8 or not r[0].isdigit():
        continue
    lines.append(r)
tot = sum(f(r[si]) for r in lines); toti = sum(f(r[ii]) for r in lines)
print(f"samples {tot:.0f} instr {toti:.3e}")
for r in sorted(lines, key=lambda r: -f(r[si]))[:top]:
    st = sorted(((f(r[c]), hdr[c]) for c in stall_cols if c < len(r) and r[c] not in ("", "-")), reverse=True)[:3]
    print(f"L{r[0]:>4} {f(r[si])/tot*100:5.1f}% ins={f(r[ii])/toti*100:5.1f}% {r[1].strip()[:70]:70s} " + " ".join(f"{h[6:]}={v/tot*100:.1f}" for v, h in st if v))

"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv, subprocess, sys, io
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = [r for r in rows[2:] if len(r) == len(hdr)]
si = hdr.index("Warp Stall Sampling (All Samples)"); ii = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
tot = sum(float(r[si] or 0) for r in data)
print(f"total samples {tot:.0f}, instructions executed {sum(float(r[ii] or 0) for r in data):.3e}")
idx = {r[0]: n for n, r in enumerate(data)}
for n, r in sorted(enumerate(data), key=lambda x: -float(x[1][si] or 0))[:top]:
    st = sorted(((float(r[c] or 0), hdr[c]) for c in stall_cols), reverse=True)[:3]
    print(f"{n:5d} {float(r[si])/tot*100:5.1f}% ex={r[ii]:>10} {r[1].strip()[:60]:60s} " + " ".join(f"{h[6:]}={v:.0f}" for v, h in st if v))

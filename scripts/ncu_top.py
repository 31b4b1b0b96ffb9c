"""Summarise an ncu report's source page: top SASS lines by stall samples (dev helper)."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
S = hdr.index("Warp Stall Sampling (All Samples)")
I = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
tot = sum(float(r[S] or 0) for r in data)
tot_i = sum(float(r[I] or 0) for r in data)
print(f"total samples {tot:.0f}, warp instructions {tot_i:.3e}")
agg = {}
for r in data:
    for i in stall_cols:
        agg[hdr[i]] = agg.get(hdr[i], 0) + float(r[i] or 0)
print("stalls:", ", ".join(f"{k[6:]}={v/tot*100:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
for k, r in sorted(enumerate(data), key=lambda x: -float(x[1][S] or 0))[:n]:
    top_stall = max(stall_cols, key=lambda i: float(r[i] or 0))
    print(f"{float(r[S])/tot*100:5.1f}% inst={float(r[I]):9.0f} #{k:5d} {hdr[top_stall][6:]:>14} | {r[1].strip()[:80]}")
